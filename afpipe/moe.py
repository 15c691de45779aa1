"""afpipe.moe — the MoE layer hot path on B200 (dispatch, SwiGLU experts, combine; fwd +
bwd) that the reference models as costs (costs.py:90-103) and F-side tasks
(taskgraph.py:333-347). Re-exports paper_2605_11005_b200.moe."""

from paper_2605_11005_b200.moe import (  # noqa: F401
    ActivationSlab,
    ExpertParams,
    MicroBatchBuffers,
    MoEFunction,
    MoELayer,
    MoEShape,
    MoEStack,
    RouterParams,
    interleave_w13,
    moe,
    split_w13,
)
