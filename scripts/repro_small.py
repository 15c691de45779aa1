import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2605_11005_b200.moe import MoELayer, MoEShape
from paper_2605_11005_b200 import kernels as K
T, H, E, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
layer = MoELayer.random(MoEShape(T=T, H=H, E=E, k=k, De=256), device="cuda")
buf = layer.buffers[0]
buf.x.normal_()
layer.stage_dispatch(buf)
torch.cuda.synchronize()
print("dispatch ok", buf.pad_off.tolist())
layer.forward_backward(buf)
torch.cuda.synchronize()
print("fwd_bwd ok")
