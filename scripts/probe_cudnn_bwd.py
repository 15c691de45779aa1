"""Can torch's cuDNN SDPA backward consume (O, LSE) from dm_attention_fwd? Compares its
dq/dk/dv against autograd through torch SDPA on the same inputs."""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import kernels as K  # noqa: E402

D = 128
dev = torch.device("cuda", 0)
b, s, nh, nkv = 2, 1024, 8, 2
qkv = torch.randn(b * s, (nh + 2 * nkv) * D, device=dev).to(torch.bfloat16)
x = qkv.view(b, s, nh + 2 * nkv, D).transpose(1, 2)
q, k, v = (t.contiguous().requires_grad_(True) for t in (x[:, :nh], x[:, nh:nh + nkv], x[:, nh + nkv:]))
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    o_ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
do = torch.randn_like(o_ref)
o_ref.backward(do)
# cuDNN fwd outputs for reference (lse layout)
kr, vr = k.detach().repeat_interleave(nh // nkv, 1), v.detach().repeat_interleave(nh // nkv, 1)
res = torch.ops.aten._scaled_dot_product_cudnn_attention(q.detach(), kr, vr, None, True, 0.0, True, False)
print("cudnn lse", res[1].shape, res[1].dtype, res[1].stride(), "philox", res[6], res[7])
out = torch.empty(b * s, nh * D, dtype=torch.bfloat16, device=dev)
lse = torch.empty(b, nh, s, dtype=torch.float32, device=dev)
K.attention_fwd(qkv, s, nh, nkv, out, lse)
o_own = out.view(b, s, nh, D).transpose(1, 2)
print("lse diff vs cudnn", (lse - res[1].view(b, nh, s)).abs().max().item())
lse_in = lse.view_as(res[1]) if res[1].numel() == lse.numel() else lse
g = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
    do, q.detach(), kr, vr, o_own, lse_in, res[6], res[7], None,
    res[2], res[3], s, s, 0.0, True)
dq, dk, dv = g
dk = dk.view(b, nkv, nh // nkv, s, D).sum(2)
dv = dv.view(b, nkv, nh // nkv, s, D).sum(2)
for name, a, r in (("dq", dq, q.grad), ("dk", dk, k.grad), ("dv", dv, v.grad)):
    print(name, (a.float() - r.float()).abs().max().item() / r.float().abs().max().item())
