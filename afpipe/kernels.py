"""afpipe.kernels — torch wrappers over the sm_100a C ABI (include/dm_moe.h).
Re-exports paper_2605_11005_b200.kernels."""

from paper_2605_11005_b200.kernels import *  # noqa: F401,F403
