"""afpipe — the reference package's module name, with the MoE hot path on B200.

Drop-in for arxiv/paper_2605_11005's `afpipe` (/root/reference/pkg/pyproject.toml:6,
export surface pkg/src/afpipe/__init__.py:1-71) on the path BASELINE.json's north
star names: the config API is this repo's mirror (`afpipe.config`, same schema,
defaults, errors and messages — tests/golden/config_cases.json), and the hot path the
reference only costs is real here:

    afpipe.moe        moe() autograd op, MoELayer / MoEStack (fused single GPU), MoEShape
    afpipe.runtime    AFPipeRank / Topology (A:F groups over NCCL), LoopbackWorld (1 GPU)
    afpipe.kernels    thin torch wrappers over the sm_100a C ABI (include/dm_moe.h)
    afpipe.profile    measured_profile (Algorithm 1 Phase 3's Profile), measured traces

The reference's control plane (costs, placement, taskgraph, sim, allocator, report,
trace_io, cli) is not rebuilt (out of scope). When the reference package
is installed next to this one, its modules join this package: its directory (found on
sys.path, or named by AFPIPE_REFERENCE_SRC) is appended to `afpipe.__path__`, so
`afpipe.sim`, `afpipe.allocator`, ... import from the reference and — because
`afpipe.config` resolves here first — run on this package's config objects; their
public names (simulate, allocate, phase3_refine, ...) are re-exported lazily.
"""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path

from paper_2605_11005_b200.config import (  # noqa: F401
    ClusterConfig,
    ConfigError,
    Experiment,
    InvalidValue,
    MissingField,
    ModelConfig,
    ScheduleKind,
    SchemaViolation,
    Workload,
    load_experiment,
    parse_experiment,
    serialize_experiment,
    validate,
)

__version__ = "0.1.0"

_HERE = Path(__file__).resolve().parent

# reference control-plane modules and the public names each contributes to `afpipe`
# (pkg/src/afpipe/__init__.py:1-71)
_REFERENCE_EXPORTS = {
    "allocator": ("Allocation", "AllocationReport", "AllocatorParams", "NoFeasible", "SearchSpaceTooLarge",
                  "allocate", "brute_force_oracle", "enumerate_feasible", "phase1_min_bottleneck",
                  "phase2_tiebreak", "phase3_refine"),
    "costs": ("CostBreakdown", "LayerCosts", "StageTimes", "arithmetic_intensities", "attention_flops",
              "backward_scale", "cost_breakdown", "ep_a2a_bytes_per_gpu", "ffn_flops", "layer_costs",
              "m2n_comm_bytes", "roofline_attainable", "stage_times", "turning_points"),
    "placement": ("InvalidDepth", "MemoryEstimate", "PlacementPlan", "assign_layers", "memory_estimate",
                  "oom_check", "validate_partition"),
    "sim": ("CycleDetected", "NegativeDuration", "ScheduleTrace", "SimResult", "chunked_overlap_exposed",
            "chunked_overlap_layer_time", "exposed_comm", "simulate", "warmup_bubble_analytic"),
    "taskgraph": ("GraphConstructionError", "Task", "TaskGraph", "TaskKind", "build_task_graph"),
    "trace_io": ("SerializationError", "export_trace", "export_trace_json", "write_trace"),
}
_NAME_TO_MODULE = {n: m for m, names in _REFERENCE_EXPORTS.items() for n in names}
# this package's own hot-path names
_OWN = {
    "moe": "afpipe.moe", "MoEFunction": "afpipe.moe", "MoELayer": "afpipe.moe", "MoEShape": "afpipe.moe",
    "MoEStack": "afpipe.moe", "AFPipeRank": "afpipe.runtime", "Topology": "afpipe.runtime",
    "LoopbackWorld": "afpipe.runtime", "measured_profile": "afpipe.profile", "MeasuredStages": "afpipe.profile",
}


def _reference_dirs() -> list[str]:
    """Directories of an installed reference `afpipe` (its sim.py marks it)."""
    found = []
    env = os.environ.get("AFPIPE_REFERENCE_SRC")
    cands = [Path(env)] if env else []
    cands += [Path(p) / "afpipe" for p in sys.path if p]
    for c in cands:
        try:
            c = c.resolve()
        except OSError:
            continue
        if c != _HERE and (c / "sim.py").is_file() and str(c) not in found:
            found.append(str(c))
    return found[:1]


REFERENCE_DIR = None
for _d in _reference_dirs():
    __path__.append(_d)   # after this package's own directory: afpipe.config stays ours
    REFERENCE_DIR = _d


def reference_available() -> bool:
    """True when the reference's control-plane modules are importable as afpipe.*."""
    return REFERENCE_DIR is not None


def __getattr__(name):
    if name in _OWN:
        return getattr(importlib.import_module(_OWN[name]), name)
    mod = _NAME_TO_MODULE.get(name)
    if mod is not None:
        if REFERENCE_DIR is None:
            raise AttributeError(f"afpipe.{name} belongs to the reference's afpipe.{mod} (control plane), which "
                                 "is not installed; set AFPIPE_REFERENCE_SRC to its package directory")
        return getattr(importlib.import_module(f"afpipe.{mod}"), name)
    raise AttributeError(name)
