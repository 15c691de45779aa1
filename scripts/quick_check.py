"""Early GPU smoke of every kernel family against torch fp32 math (dev aid).

    python scripts/quick_check.py [gemm|dispatch|all]
"""

import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2605_11005_b200 import kernels as K  # noqa: E402
from paper_2605_11005_b200 import _lib  # noqa: E402


def rel(a, b):
    a = a.float(); b = b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


def interleave_w13(w1, w3):
    E, De, H = w1.shape
    w = torch.empty(E, 2 * De, H, dtype=w1.dtype, device=w1.device)
    wv = w.view(E, De // 128, 2, 128, H)
    wv[:, :, 0] = w1.view(E, De // 128, 128, H)
    wv[:, :, 1] = w3.view(E, De // 128, 128, H)
    return w


def gemm_check(E=4, H=512, De=256, rows=(256, 0, 384, 128)):
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(0)
    off = [0]
    for r in rows:
        off.append(off[-1] + r)
    cap = off[-1] + 256
    pad_off = torch.tensor(off, dtype=torch.int32, device=dev)
    x = (torch.randn(cap, H, generator=g) ).to(torch.bfloat16).to(dev)
    w1 = (torch.randn(E, De, H, generator=g) * 0.05).to(torch.bfloat16).to(dev)
    w3 = (torch.randn(E, De, H, generator=g) * 0.05).to(torch.bfloat16).to(dev)
    w2 = (torch.randn(E, H, De, generator=g) * 0.05).to(torch.bfloat16).to(dev)
    w13 = interleave_w13(w1, w3)
    h13 = torch.zeros(cap, 2 * De, dtype=torch.bfloat16, device=dev)
    act = torch.zeros(cap, De, dtype=torch.bfloat16, device=dev)
    y = torch.zeros(cap, H, dtype=torch.bfloat16, device=dev)
    K.w13_swiglu_fwd(x, w13, pad_off, h13, act)
    K.w2_fwd(act, w2, pad_off, y)
    dy = torch.randn(cap, H, generator=g).to(torch.bfloat16).to(dev)
    dh13 = torch.zeros_like(h13)
    K.w2_dgrad_swiglu_bwd(dy, w2, h13, pad_off, dh13)
    dx = torch.zeros(cap, H, dtype=torch.bfloat16, device=dev)
    K.w13_dgrad(dh13, w13, pad_off, dx)
    dW2 = torch.zeros(E, H, De, dtype=torch.float32, device=dev)
    dW13 = torch.zeros(E, 2 * De, H, dtype=torch.float32, device=dev)
    K.wgrad(dy, act, pad_off, dW2)
    K.wgrad(dh13, x, pad_off, dW13)
    torch.cuda.synchronize()
    errs = {}
    for e in range(E):
        a, b = off[e], off[e + 1]
        if a == b:
            errs[f"dW2_e{e}_empty"] = dW2[e].abs().max().item()
            continue
        xe = x[a:b].float()
        g_ = xe @ w1[e].float().t(); u_ = xe @ w3[e].float().t()
        act_r = torch.nn.functional.silu(g_) * u_
        errs[f"gate_e{e}"] = rel(h13[a:b].view(-1, De // 128, 2, 128)[:, :, 0].reshape(b - a, De), g_)
        errs[f"up_e{e}"] = rel(h13[a:b].view(-1, De // 128, 2, 128)[:, :, 1].reshape(b - a, De), u_)
        errs[f"act_e{e}"] = rel(act[a:b], act_r)
        y_r = act[a:b].float() @ w2[e].float().t()
        errs[f"y_e{e}"] = rel(y[a:b], y_r)
        dact = dy[a:b].float() @ w2[e].float()
        gb = h13[a:b].view(-1, De // 128, 2, 128)[:, :, 0].reshape(b - a, De).float()
        ub = h13[a:b].view(-1, De // 128, 2, 128)[:, :, 1].reshape(b - a, De).float()
        s = torch.sigmoid(gb)
        dg_r = dact * ub * s * (1 + gb * (1 - s)); du_r = dact * gb * s
        errs[f"dg_e{e}"] = rel(dh13[a:b].view(-1, De // 128, 2, 128)[:, :, 0].reshape(b - a, De), dg_r)
        errs[f"du_e{e}"] = rel(dh13[a:b].view(-1, De // 128, 2, 128)[:, :, 1].reshape(b - a, De), du_r)
        dx_r = dh13[a:b].float() @ w13[e].float()
        errs[f"dx_e{e}"] = rel(dx[a:b], dx_r)
        dW2_r = dy[a:b].float().t() @ act[a:b].float()
        errs[f"dW2_e{e}"] = rel(dW2[e], dW2_r)
        dW13_r = dh13[a:b].float().t() @ x[a:b].float()
        errs[f"dW13_e{e}"] = rel(dW13[e], dW13_r)
    bad = {k: v for k, v in errs.items() if v > 2e-2}
    print("gemm max rel err:", max(errs.values()), "bad:", bad)
    return not bad


def dispatch_check(T=1000, H=512, E=8, k=2):
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(1)
    x = torch.randn(T, H, generator=g).to(torch.bfloat16).to(dev)
    wg = (torch.randn(E, H, generator=g) * 0.02).to(dev)
    cap = _lib.capacity_rows(T, E, k)
    ws = torch.empty(_lib.route_workspace_size(T, H, E, k), dtype=torch.uint8, device=dev)
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    w = torch.empty(T, k, dtype=torch.float32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    pad_off = torch.empty(E + 1, dtype=torch.int32, device=dev)
    row_map = torch.empty(T, k, dtype=torch.int32, device=dev)
    src = torch.empty(cap, dtype=torch.int32, device=dev)
    xp = torch.full((cap, H), float("nan"), dtype=torch.bfloat16, device=dev)
    K.route_and_dispatch(x, wg, k, ws, idx, w, counts, pad_off, row_map, src, xp)
    torch.cuda.synchronize()
    logits_ref = x.float() @ wg.t()
    lg = torch.empty(T, E, device=dev)
    K.router_logits(x, wg, lg)
    print("logits rel err", rel(lg, logits_ref))
    v, i = torch.topk(lg, k, dim=1)
    ok_idx = (i.int() == idx).all().item()
    w_ref = torch.softmax(v, dim=1)
    print("idx match", ok_idx, "w err", rel(w, w_ref))
    cnt_ref = torch.bincount(idx.flatten().long(), minlength=E).int()
    print("counts match", (cnt_ref == counts).all().item(), counts.tolist(), pad_off.tolist())
    # x_perm rows equal source
    rm = row_map.long()
    ok_rows = torch.equal(xp[rm.flatten()], x.repeat_interleave(k, dim=0))
    print("x_perm rows", ok_rows)
    # padding rows zero
    po = pad_off.tolist(); cn = counts.tolist()
    pad_ok = all(torch.all(xp[po[e] + cn[e]:po[e + 1]] == 0).item() for e in range(E))
    print("padding zero", pad_ok)
    # combine fwd/bwd
    y_perm = torch.randn(cap, H, generator=g).to(torch.bfloat16).to(dev)
    y = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    K.combine_fwd(y_perm, row_map, w, y)
    y_ref = (y_perm.float()[rm] * w.unsqueeze(-1)).sum(1)
    print("combine fwd err", rel(y, y_ref))
    dy = torch.randn(T, H, generator=g).to(torch.bfloat16).to(dev)
    dyp = torch.full((cap, H), float("nan"), dtype=torch.bfloat16, device=dev)
    dw = torch.empty(T, k, device=dev); dl = torch.empty(T, k, device=dev)
    K.combine_bwd(dy, y_perm, row_map, w, counts, pad_off, dyp, dw, dl)
    dw_ref = (y_perm.float()[rm] * dy.float().unsqueeze(1)).sum(-1)
    print("dw err", rel(dw, dw_ref))
    dl_ref = w * (dw_ref - (w * dw_ref).sum(1, keepdim=True))
    print("dlogit err", rel(dl, dl_ref))
    dyp_ref = dy.float().unsqueeze(1) * w.unsqueeze(-1)
    print("dy_perm err", rel(dyp[rm], dyp_ref))
    dx = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    K.permute_bwd(dyp, row_map, idx, dl, wg, dx)
    dx_ref = dyp.float()[rm].sum(1) + torch.einsum("tk,tkh->th", dl, wg[idx.long()])
    print("permute_bwd err", rel(dx, dx_ref))
    pws = torch.empty(_lib.router_wgrad_workspace_size(T, H, E) // 4, device=dev)
    dwg = torch.empty(E, H, device=dev)
    K.router_wgrad(x, idx, dl, pws, dwg)
    dense = torch.zeros(T, E, device=dev).scatter_(1, idx.long(), dl)
    print("router wgrad err", rel(dwg, dense.t() @ x.float()))
    torch.cuda.synchronize()


def gemm_bench(E=8, rows_per=1024, H=4096, De=14336):
    dev = "cuda"
    off = [i * rows_per for i in range(E + 1)]
    cap = off[-1]
    pad_off = torch.tensor(off, dtype=torch.int32, device=dev)
    x = torch.randn(cap, H, device=dev).to(torch.bfloat16)
    w13 = (torch.randn(E, 2 * De, H, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn(E, H, De, device=dev) * 0.02).to(torch.bfloat16)
    h13 = torch.empty(cap, 2 * De, dtype=torch.bfloat16, device=dev)
    act = torch.empty(cap, De, dtype=torch.bfloat16, device=dev)
    y = torch.empty(cap, H, dtype=torch.bfloat16, device=dev)
    dh13 = torch.empty_like(h13); dx = torch.empty_like(y)
    dW2 = torch.empty(E, H, De, device=dev); dW13 = torch.empty(E, 2 * De, H, device=dev)
    fl = 2 * cap * H * De
    ops = {
        "w13_fwd": (lambda: K.w13_swiglu_fwd(x, w13, pad_off, h13, act), 2 * fl),
        "w2_fwd": (lambda: K.w2_fwd(act, w2, pad_off, y), fl),
        "w2_dgrad": (lambda: K.w2_dgrad_swiglu_bwd(y, w2, h13, pad_off, dh13), fl),
        "w13_dgrad": (lambda: K.w13_dgrad(dh13, w13, pad_off, dx), 2 * fl),
        "wgrad2": (lambda: K.wgrad(y, act, pad_off, dW2), fl),
        "wgrad13": (lambda: K.wgrad(dh13, x, pad_off, dW13), 2 * fl),
    }
    for name, (fn, flops) in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        n = 10
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        print(f"{name}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
    a = x[:, :].clone()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b = w13[0].clone()
    torch.matmul(a, b.t()); torch.cuda.synchronize()
    s.record()
    for _ in range(5):
        torch.matmul(a, b.t())
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"cublas same-shape dense: {ms:.3f} ms {2 * cap * H * 2 * De / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    print(torch.cuda.get_device_name(), "launches so far", _lib.launch_count())
    t = time.time()
    if what in ("gemm", "all"):
        ok = gemm_check()
        ok &= gemm_check(E=3, H=256, De=256, rows=(128, 512, 0))
        print("GEMM OK" if ok else "GEMM MISMATCH")
    if what in ("dispatch", "all"):
        dispatch_check()
        dispatch_check(T=4096, H=4096, E=8, k=2)
        dispatch_check(T=512, H=7168, E=256, k=8)
    if what in ("bench", "all"):
        gemm_bench()
    print("done in", time.time() - t)
