"""Isolated timing of the Mixtral-shape grouped GEMMs (CUDA events, 10 reps). Run twice,
once with DM_GEMM_DIAG=1 (A tile loaded only for the first stages of each tile, results
invalid): if the mainloop is operand-supply bound the time drops with the bytes."""

import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import kernels as K  # noqa: E402


def main(E=8, rows_per=1024, H=4096, De=14336):
    dev = "cuda"
    off = [i * rows_per for i in range(E + 1)]
    cap = off[-1]
    po = torch.tensor(off, dtype=torch.int32, device=dev)
    x = torch.randn(cap, H, device=dev).to(torch.bfloat16)
    w13 = (torch.randn(E, 2 * De, H, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn(E, H, De, device=dev) * 0.02).to(torch.bfloat16)
    h13 = torch.empty(cap, 2 * De, dtype=torch.bfloat16, device=dev)
    act = torch.empty(cap, De, dtype=torch.bfloat16, device=dev)
    y = torch.empty(cap, H, dtype=torch.bfloat16, device=dev)
    dh13 = torch.empty_like(h13)
    dx = torch.empty_like(y)
    flops = 2 * cap * H * De
    so4 = torch.stack([po] * 4)  # 4 micro-batches stacked (deferred wgrad shape)
    x4, act4, y4, dh4 = (t.repeat(4, 1) for t in (x, act, y, dh13))
    dW2 = torch.empty(E, H, De, device=dev)
    dW13 = torch.empty(E, 2 * De, H, device=dev)
    ops = {
        "w13_fwd": (lambda: K.w13_swiglu_fwd(x, w13, po, h13, act), 2 * flops),
        "w2_fwd": (lambda: K.w2_fwd(act, w2, po, y), flops),
        "w2_dgrad": (lambda: K.w2_dgrad_swiglu_bwd(y, w2, h13, po, dh13), flops),
        "w13_dgrad": (lambda: K.w13_dgrad(dh13, w13, po, dx), 2 * flops),
        "wgrad2_x4": (lambda: K.wgrad(y4, act4, so4, dW2), 4 * flops),
        "wgrad13_x4": (lambda: K.wgrad(dh4, x4, so4, dW13), 8 * flops),
    }
    out = {"diag": os.environ.get("DM_GEMM_DIAG", "0"), "dual": os.environ.get("DM_GEMM_DUAL", "1")}
    for name, (fn, fl) in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out[name] = {"ms": round(ms, 4), "TFLOP/s": round(fl / ms / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dsv3":
        main(E=256, rows_per=128, H=7168, De=2048)
    else:
        main()
