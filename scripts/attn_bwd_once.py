"""One dm_attention_bwd call (s = 4096, 32 heads / 8 KV heads, 16K tokens) for ncu captures."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import kernels as K  # noqa: E402

s, nh, nkv, T = 4096, 32, 8, 16384
D = 128
qkv = torch.randn(T, (nh + 2 * nkv) * D, device="cuda").to(torch.bfloat16)
dout = torch.randn(T, nh * D, device="cuda").to(torch.bfloat16)
out = torch.empty(T, nh * D, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(T // s, nh, s, dtype=torch.float32, device="cuda")
K.attention_fwd(qkv, s, nh, nkv, out, lse)
dqkv = torch.empty_like(qkv)
for _ in range(2):
    K.attention_bwd(qkv, out, dout, lse, s, nh, nkv, dqkv)
torch.cuda.synchronize()
print("ok")
