"""Own causal GQA flash-attention forward (dm_attention_fwd) vs torch SDPA (cuDNN) forward on
the same B200: CUDA-event time per call and causal TFLOP/s (2·2·s²·D·nh/2 per sequence)."""

import json
import sys
from pathlib import Path

import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import kernels as K  # noqa: E402

D = 128


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda", 0)
    for s, b in ((2048, 8), (4096, 4), (8192, 2), (16384, 1)):
        nh, nkv = 32, 8
        qkv = torch.randn(b * s, (nh + 2 * nkv) * D, device=dev).to(torch.bfloat16)
        out = torch.empty(b * s, nh * D, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(b, nh, s, dtype=torch.float32, device=dev)
        x = qkv.view(b, s, nh + 2 * nkv, D).transpose(1, 2)
        q, k, v = x[:, :nh].contiguous(), x[:, nh:nh + nkv].contiguous(), x[:, nh + nkv:].contiguous()
        own = timeit(lambda: K.attention_fwd(qkv, s, nh, nkv, out, lse))
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            lib = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True,
                                                                                  enable_gqa=True))
        flops = 2 * 2 * s * s * D * nh * b / 2
        print(json.dumps({"seq": s, "batch": b, "heads": nh, "kv_heads": nkv, "own_ms": round(own, 3),
                          "own_TFLOP/s": round(flops / own / 1e9, 1), "cudnn_ms": round(lib, 3),
                          "cudnn_TFLOP/s": round(flops / lib / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
