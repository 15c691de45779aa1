"""cProfile the host side of one AF-Pipe rank (tiny config, N=2) to find runtime overheads.
Run under torchrun; rank 0 writes gpurun_out/host_profile.txt."""
import cProfile
import io
import os
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_11005_b200.config import load_experiment  # noqa: E402
from paper_2605_11005_b200.moe import MoEShape  # noqa: E402
from paper_2605_11005_b200.runtime import AFPipeRank, Topology  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
exp = load_experiment(sys.argv[1] if len(sys.argv) > 1 else "configs/tiny.yaml")
shape = MoEShape.from_experiment(exp)
r = AFPipeRank(shape, Topology.default(world, shape.E), rank, exp.workload.num_microbatches, dev,
               layers=exp.model.layers)
r.init_groups()
for _ in range(5):
    r.run_iteration()
torch.cuda.synchronize()
dist.barrier()
pr = cProfile.Profile()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pr.enable()
for _ in range(20):
    r.run_iteration()
pr.disable()
e1.record()
torch.cuda.synchronize()
if rank in (0, world - 1):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/host_profile_r{rank}.txt").write_text(f"ms/iter {e0.elapsed_time(e1) / 20:.3f}\n" + s.getvalue())
dist.barrier()
dist.destroy_process_group()
