"""Cold-L2 time of each A-side stage of the Mixtral layer (bench.isolated_stage_ms), for
quick A/B runs of the HBM-bound kernels."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_11005_b200.moe import MoELayer, MoEShape  # noqa: E402

shape = MoEShape(4096, 4096, 8, 2, 14336)
layer = MoELayer.random(shape, device="cuda", seed=1)
b = layer.buffers[0]
b.x.normal_()
b.dy.normal_()
layer.forward_backward(b)
torch.cuda.synchronize()
fns = {"dispatch": lambda: layer.stage_dispatch(b), "combine_fwd": lambda: layer.stage_combine(b),
       "combine_bwd": lambda: layer.stage_combine_bwd(b), "permute_bwd": lambda: layer.stage_permute_bwd(b),
       "router_wgrad": lambda: layer.stage_router_wgrad(b, False)}
hb = shape.hbm_bytes()
hb["router_wgrad"] = shape.T * shape.H * 2 + shape.T * shape.k * 8
iso = bench.isolated_stage_ms(fns, torch.device("cuda"))
print(json.dumps({k: {"us": round(v * 1e3, 1), "frac": round(hb[k] / (v / 1e3) / 6547.5e9, 3)} for k, v in iso.items()}))
