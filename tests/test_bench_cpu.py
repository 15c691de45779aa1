"""bench.py contract on CPU: the reference arm (`--impl reference`, the oracle port on the
host cores) prints one JSON line with the keys the driver reads, and non-zero ranks of a
torchrun launch exit 0 without work."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(extra_env=None, *args):
    env = {**os.environ, **(extra_env or {})}
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                           "--config", str(ROOT / "configs" / "tiny.yaml"), *args],
                          capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    res = _run(None, "--steps", "2", "--warmup", "1")
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["warmup"] >= 3          # W >= 3 is enforced
    assert line["steps"] == 2
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_reference_arm_other_ranks_exit_quietly():
    res = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--gpus", "2")
    assert res.returncode == 0, res.stderr[-2000:]
    assert not [ln for ln in res.stdout.splitlines() if ln.startswith("{")]


def test_reference_arm_time_is_measured_not_extrapolated():
    """ms_per_step is the measured time of the step's own sample: steps x ms_per_step fits
    inside the arm's wall time, and value x ms_per_step recovers the sampled token count."""
    res = _run(None, "--steps", "2", "--warmup", "1")
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    c = line["consistency"]
    assert line["steps"] * line["ms_per_step"] / 1e3 <= c["timed_s"] * 1.01 + 1e-3
    assert c["timed_s"] <= c["run_s"]
    assert abs(line["value"] * line["ms_per_step"] / 1e3 - line["config"]["tokens_per_step"]) < 0.01 * line["config"]["tokens_per_step"]
    assert "no extrapolation" in line["cpu_baseline"]["sample"]


def test_gpus_must_match_world_size():
    env = {**os.environ, "RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config",
                          str(ROOT / "configs" / "tiny.yaml")], capture_output=True, text=True, timeout=600,
                         env=env, cwd=ROOT)
    assert res.returncode != 0
    assert "WORLD_SIZE" in res.stderr


def test_schedule_model_reproduces_a_serial_chain():
    """bench._schedule_model: the restated reference schedule on measured task times — for one
    micro-batch the chain is serial, so the prediction is the sum of the task times + W."""
    import bench

    ivs = [("A_f", 0, "compute", 0.0, 1.0, 0), ("M2N", 0, "send", 1.0, 1.2, 8), ("F_f", 0, "compute", 1.2, 3.0, 0),
           ("N2M", 0, "send", 3.0, 3.2, 8), ("A_t", 0, "compute", 3.2, 3.6, 0), ("M2N_b", 0, "send", 3.6, 3.8, 8),
           ("F_b", 0, "compute", 3.8, 7.0, 0), ("N2M_b", 0, "send", 7.0, 7.2, 8), ("A_b", 0, "compute", 7.2, 7.5, 0),
           ("W", -1, "compute", 7.5, 9.0, 0)]
    m = bench._schedule_model([{"ivs": ivs}], 1, 1, 1, 9.0)
    assert abs(m["predicted_iteration_ms"] - 9.0) < 1e-3
    assert m["measured_over_predicted"] == 1.0
