"""Probe which torch SDPA backends run fwd+bwd on this GPU and how fast (A-side attention stopgap)."""
import time

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

dev = torch.device("cuda")
for S in (4096, 16384):
    B, NH, NKV, D = 1, 32, 8, 128
    q = torch.randn(B, NH, S, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
    k = torch.randn(B, NKV, S, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
    v = torch.randn(B, NKV, S, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel([be]):
                def run():
                    o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
                    o.backward(torch.ones_like(o))
                run()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    run()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 5
                flops = 4 * B * NH * S * S * D / 2 * 3.5  # causal fwd (x1) + bwd (x2.5)
                print(f"S={S} {be.name}: {ms:.3f} ms fwd+bwd, {flops / ms / 1e9:.0f} TFLOP/s", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(f"S={S} {be.name}: unavailable ({type(ex).__name__}: {str(ex)[:120]})", flush=True)
