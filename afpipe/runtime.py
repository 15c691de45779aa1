"""afpipe.runtime — the AF-Pipe runtime the reference simulates (_build_afpipe,
taskgraph.py:307-356; simulate, sim.py:101-216): A and F rank groups exchanging
micro-batches over NCCL (one process per GPU) or the single-GPU loopback transport.
Re-exports paper_2605_11005_b200.runtime / .transport."""

from paper_2605_11005_b200.runtime import AFPipeRank, GpuStages, Topology, balanced_blocks, trace_intervals  # noqa: F401
from paper_2605_11005_b200.transport import LoopbackTransport, LoopbackWorld, NcclTransport  # noqa: F401
