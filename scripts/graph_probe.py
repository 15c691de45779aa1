"""torchrun --nproc-per-node 2: capture one AF-Pipe iteration (1A:1F) as a CUDA graph and
replay it; prints progress per rank (diagnostic for AFPipeRank.capture)."""
import os
import sys
import time
import traceback
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2605_11005_b200.moe import MoEShape
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology

    T = int(os.environ.get("GP_T", "512"))
    r = AFPipeRank(MoEShape(T, 256, 8, 2, 256), Topology(world, 1, 8, 1), rank, 2, dev, layers=2)
    r.init_groups()
    if r.role == "A":
        for i in range(2):
            r.input(i).normal_()
            r.out_bufs[i].dy.normal_()
    print(f"[{rank}] built", flush=True)
    try:
        t0 = time.time()
        g = r.capture()
        print(f"[{rank}] captured in {time.time() - t0:.2f}s", flush=True)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        print(f"[{rank}] replayed", flush=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms_g = e0.elapsed_time(e1) / 20
        dist.barrier()
        e0.record()
        for _ in range(20):
            r.run_iteration()
        e1.record()
        torch.cuda.synchronize()
        ms_e = e0.elapsed_time(e1) / 20
        print(f"[{rank}] graph {ms_g:.3f} ms/iter, eager {ms_e:.3f} ms/iter", flush=True)
    except Exception:
        traceback.print_exc()
        sys.stdout.flush()
        os._exit(1)
    del g
    torch.cuda.synchronize()
    dist.barrier()
    print(f"[{rank}] final barrier passed", flush=True)
    dist.destroy_process_group()
    print(f"[{rank}] destroyed", flush=True)


if __name__ == "__main__":
    main()
