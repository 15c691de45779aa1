"""afpipe.profile — measured stage times as Algorithm 1's Profile(M, M_a) (allocator.py:205-237)
and measured runtime traces in the reference trace schema (trace_io.py:33-67).
Re-exports paper_2605_11005_b200.profile."""

from paper_2605_11005_b200.profile import *  # noqa: F401,F403
from paper_2605_11005_b200.profile import MeasuredStages, export_trace, measured_profile  # noqa: F401
