"""Each A-side stage of the Mixtral layer once, inside cudaProfilerStart/Stop (after a
warm-up pass), for `ncu --profile-from-start off --set full` captures of dispatch,
combine fwd/bwd, permute bwd and the router weight gradient."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200.moe import MoELayer, MoEShape  # noqa: E402

shape = MoEShape(4096, 4096, 8, 2, 14336)
layer = MoELayer.random(shape, device="cuda", seed=1)
b = layer.buffers[0]
b.x.normal_()
b.dy.normal_()
layer.forward_backward(b)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stages = [lambda: layer.stage_dispatch(b), lambda: layer.stage_combine(b), lambda: layer.stage_combine_bwd(b),
          lambda: layer.stage_permute_bwd(b), lambda: layer.stage_router_wgrad(b, False)]
torch.cuda.profiler.start()
for fn in stages:
    flush.zero_()   # cold L2, as in bench.isolated_stage_ms
    fn()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
