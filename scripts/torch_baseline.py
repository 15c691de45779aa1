"""A library baseline for the same MoE layer fwd+bwd: PyTorch ops + torch._grouped_mm (CUTLASS
grouped GEMM) with autograd — router matmul + topk + softmax, stable argsort permutation,
grouped W13 GEMM, SiLU*up, grouped W2 GEMM, weighted index_add combine. Same shapes and
micro-batching as bench.py (Mixtral layer, 4 micro-batches of 4096 tokens); reports tokens/s
so the fused sm_100a path can be compared with what a user gets from the stock libraries."""

import json
import sys

import torch
import torch.nn.functional as F


def moe_torch(x, wg, w13, w2, k):
    T, H = x.shape
    E = wg.shape[0]
    logits = x.float() @ wg.t()
    topv, idx = torch.topk(logits, k, dim=1)
    w = torch.softmax(topv, dim=1)
    flat = idx.reshape(-1)
    order = torch.argsort(flat, stable=True)
    tok = order // k
    counts = torch.bincount(flat, minlength=E)
    offs = torch.cumsum(counts, 0).to(torch.int32)
    xp = x[tok]
    h = torch._grouped_mm(xp, w13.transpose(1, 2), offs=offs)
    De = h.shape[1] // 2
    act = F.silu(h[:, :De]) * h[:, De:]
    yp = torch._grouped_mm(act, w2.transpose(1, 2), offs=offs)
    wt = w.reshape(-1)[order].to(yp.dtype)
    y = torch.zeros_like(x).index_add_(0, tok, yp * wt[:, None])
    return y


def main(T=4096, H=4096, E=8, k=2, De=14336, mb=4, steps=5, warmup=3):
    dev = "cuda"
    wg = (torch.randn(E, H, device=dev) * 0.02).requires_grad_(True)
    w13 = (torch.randn(E, 2 * De, H, device=dev) * 0.02).to(torch.bfloat16).requires_grad_(True)
    w2 = (torch.randn(E, H, De, device=dev) * 0.02).to(torch.bfloat16).requires_grad_(True)
    xs = [torch.randn(T, H, device=dev).to(torch.bfloat16).requires_grad_(True) for _ in range(mb)]
    dys = [torch.randn(T, H, device=dev).to(torch.bfloat16) for _ in range(mb)]

    def step():
        for x, dy in zip(xs, dys):
            moe_torch(x, wg, w13, w2, k).backward(dy)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(json.dumps({"impl": "torch ops + torch._grouped_mm + autograd", "T": T, "H": H, "E": E, "k": k,
                      "D_e": De, "microbatches": mb, "ms_per_step": round(ms, 3),
                      "tokens_per_s": round(mb * T / (ms / 1e3), 1)}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dsv3":
        main(H=7168, E=256, k=8, De=2048)
    else:
        main()
