"""Drop-in under the reference's module name (`afpipe`, /root/reference/pkg/pyproject.toml:6).

1. Without the reference installed, `import afpipe` serves the config API (this repo's
   mirror), the hot path (afpipe.moe / afpipe.runtime / afpipe.kernels / afpipe.profile),
   and refuses control-plane names with a clear message.
2. With the reference installed next to it (AFPIPE_REFERENCE_SRC, here /root/reference),
   the reference's control-plane modules join the package and run on THIS package's
   config objects: `afpipe.report.run_schedule` / `allocate` give results identical to
   the unmodified reference package on the same documents.
Each case runs in a fresh interpreter (the package extends its __path__ at import)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg/src")
TOY = Path("/root/reference/pkg/configs/toy.yaml")
DEEPSEEK = Path("/root/reference/pkg/configs/deepseek_moe.yaml")


def _py(code: str, env_extra: dict, pythonpath: list[str]):
    env = {k: v for k, v in os.environ.items() if k not in ("AFPIPE_REFERENCE_SRC", "PYTHONPATH")}
    env.update(env_extra)
    env["PYTHONPATH"] = os.pathsep.join(pythonpath)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd="/tmp",
                         timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    return res.stdout


def test_afpipe_serves_config_and_hot_path_without_reference():
    out = _py("""
import json, afpipe, afpipe.config, afpipe.moe, afpipe.runtime, afpipe.profile
import paper_2605_11005_b200.config as mine
assert afpipe.parse_experiment is mine.parse_experiment and afpipe.config.Experiment is mine.Experiment
assert callable(afpipe.moe.moe) and afpipe.MoEShape is afpipe.moe.MoEShape
assert afpipe.runtime.AFPipeRank and afpipe.runtime.LoopbackWorld and afpipe.profile.measured_profile
try:
    afpipe.simulate
    raise SystemExit("control-plane name resolved without the reference")
except AttributeError as e:
    assert "AFPIPE_REFERENCE_SRC" in str(e)
print(json.dumps({"ref": afpipe.reference_available()}))
""", {}, [str(ROOT)])
    assert json.loads(out.strip().splitlines()[-1]) == {"ref": False}


_SCRIPT = """
import json, sys
import afpipe
from afpipe.config import load_experiment
from afpipe.allocator import default_allocation
from afpipe.report import run_schedule
out = {"config_module": afpipe.config.__name__ if hasattr(afpipe, "config") else None}
for path in sys.argv[1:]:
    exp = load_experiment(path)
    alloc = default_allocation(exp)
    r = {"alloc": [alloc.attn_nodes, alloc.ffn_nodes, alloc.attn_nics, alloc.ffn_nics]}
    for kind in afpipe.ScheduleKind:
        trace, res = run_schedule(exp, kind, alloc)
        r[kind.value] = [res.iteration_time, res.exposed_comm, res.mfu, res.bubble_fraction]
    out[path] = r
print(json.dumps(out))
"""


@pytest.mark.skipif(not (REF_SRC / "afpipe" / "sim.py").exists(), reason="reference sources not present")
def test_reference_control_plane_runs_on_our_config_identically():
    args = [str(TOY), str(DEEPSEEK)]
    code = _SCRIPT.replace("sys.argv[1:]", repr(args))
    ours = _py(code + "\nimport paper_2605_11005_b200.config as m; assert afpipe.config.Experiment is m.Experiment"
                      "\nassert afpipe.reference_available()",
               {"AFPIPE_REFERENCE_SRC": str(REF_SRC / "afpipe")}, [str(ROOT)])
    ref = _py(code, {}, [str(REF_SRC)])
    a = json.loads(ours.strip().splitlines()[-1])
    b = json.loads(ref.strip().splitlines()[-1])
    for path in args:
        assert a[path] == b[path], (path, a[path], b[path])


@pytest.mark.skipif(not (REF_SRC / "afpipe" / "sim.py").exists(), reason="reference sources not present")
def test_reference_names_reexported_lazily():
    out = _py("""
import json, afpipe
print(json.dumps({"simulate": afpipe.simulate.__module__, "phase3": afpipe.phase3_refine.__module__,
                  "config": afpipe.parse_experiment.__module__}))
""", {"AFPIPE_REFERENCE_SRC": str(REF_SRC / "afpipe")}, [str(ROOT)])
    d = json.loads(out.strip().splitlines()[-1])
    assert d == {"simulate": "afpipe.sim", "phase3": "afpipe.allocator", "config": "paper_2605_11005_b200.config"}
