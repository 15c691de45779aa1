"""One warm-up + N profiled steps of the fused MoE layer (for ncu launch lists).

The measured steps are bracketed by cudaProfilerStart/Stop, so run ncu with
`--profile-from-start off` to capture exactly one iteration's launches."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200.config import load_experiment  # noqa: E402
from paper_2605_11005_b200.moe import MoELayer, MoEShape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="configs/mixtral_layer.yaml")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
a = ap.parse_args()
exp = load_experiment(a.config)
shape = MoEShape.from_experiment(exp)
mb = exp.workload.num_microbatches
layer = MoELayer.random(shape, device="cuda", seed=1, num_buffers=mb)
for b in layer.buffers:
    b.x.normal_()
    b.dy.normal_()
for _ in range(a.warmup):
    layer.iteration(mb)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    layer.iteration(mb)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
