"""Own attention backward (dm_attention_bwd) vs cuDNN's SDPA backward on the same (O, LSE):
time per call (CUDA events, median of 10) and TFLOP/s (causal bwd = 2.5 x 2 s^2 H per seq)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import kernels as K  # noqa: E402

D = 128


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for s in (2048, 4096, 8192):
    nh, nkv, T = 32, 8, 16384
    b = T // s
    qkv = torch.randn(T, (nh + 2 * nkv) * D, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, nh * D, device="cuda").to(torch.bfloat16)
    out = torch.empty(T, nh * D, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(b, nh, s, dtype=torch.float32, device="cuda")
    K.attention_fwd(qkv, s, nh, nkv, out, lse)
    dqkv = torch.empty_like(qkv)
    dl = torch.empty(2, b, nh, s, dtype=torch.float32, device="cuda")
    own = t(lambda: K.attention_bwd(qkv, out, dout, lse, s, nh, nkv, dqkv, dl))
    x = qkv.view(b, s, nh + 2 * nkv, D).transpose(1, 2)
    q, k, v = x[:, :nh], x[:, nh:nh + nkv], x[:, nh + nkv:]
    o = out.view(b, s, nh, D).transpose(1, 2)
    do = dout.view(b, s, nh, D).transpose(1, 2)
    zero = torch.zeros((), dtype=torch.int64, device="cuda")
    lib = t(lambda: torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
        do, q, k, v, o, lse.unsqueeze(-1), zero, zero, None, None, None, s, s, 0.0, True))
    fl = 2.5 * 2 * s * s * nh * D * b
    print(json.dumps({"seq_len": s, "own_ms": round(own, 3), "cudnn_ms": round(lib, 3),
                      "own_TFLOPs": round(fl / own / 1e9, 1), "cudnn_TFLOPs": round(fl / lib / 1e9, 1),
                      "own_vs_cudnn": round(lib / own, 3)}))
