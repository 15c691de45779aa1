"""paper_2605_11005_b200 — B200-native (sm_100a) DisagMoE MoE hot path.

Drop-in for the hot path of the reference package `afpipe`
(arxiv/paper_2605_11005): top-k gating + permutation (dispatch), per-expert
SwiGLU FFN fwd/bwd on tcgen05 tensor cores, gate-weighted combine, scheduled
with AF-Pipe's issue order. The reference's config API is mirrored in
`.config`; the kernels sit behind the C ABI in include/dm_moe.h.
"""

from .config import (  # noqa: F401
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


def __getattr__(name):
    # torch-dependent modules load lazily so config-only users need no GPU stack.
    if name in ("MoELayer", "MoEShape", "moe", "MoEFunction"):
        from . import moe as _moe

        return getattr(_moe, name)
    raise AttributeError(name)
