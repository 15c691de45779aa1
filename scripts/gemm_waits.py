"""Per-role wait-cycle breakdown of the 2-SM grouped GEMMs (dm_debug_gemm_profile).

For each GEMM of the Mixtral layer shape, prints the fraction of the average CTA
lifetime the TMA producer waits on free smem slots, the MMA issuer waits on
data (full) and on the epilogue (tempty), and the epilogue waits on MMA (tfull).
"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import _lib  # noqa: E402
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
    dW2 = torch.empty(E, H, De, device=dev)
    dW13 = torch.empty(E, 2 * De, H, device=dev)
    so4 = torch.stack([po] * 4)  # 4 micro-batches stacked (deferred wgrad shape)
    x4, act4, y4, dh4 = (t.repeat(4, 1) for t in (x, act, y, dh13))
    ops = {
        "w13_fwd": lambda: K.w13_swiglu_fwd(x, w13, po, h13, act),
        "w2_fwd": lambda: K.w2_fwd(act, w2, po, y),
        "w2_dgrad": lambda: K.w2_dgrad_swiglu_bwd(y, w2, h13, po, dh13),
        "w13_dgrad": lambda: K.w13_dgrad(dh13, w13, po, dx),
        "wgrad2_x4": lambda: K.wgrad(y4, act4, so4, dW2),
        "wgrad13_x4": lambda: K.wgrad(dh4, x4, so4, dW13),
    }
    nsm = torch.cuda.get_device_properties(0).multi_processor_count & ~1
    buf = torch.zeros(5, dtype=torch.int64, device=dev)
    for name, fn in ops.items():
        fn()
        torch.cuda.synchronize()
        buf.zero_()
        _lib.load().dm_debug_gemm_profile(buf.data_ptr())
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        _lib.load().dm_debug_gemm_profile(None)
        b = buf.cpu().tolist()
        life = b[4] / nsm
        print(f"{name:12s} {s.elapsed_time(e):7.3f} ms | producer wait(empty) {b[0] / nsm / life:5.1%} | "
              f"MMA wait(full) {b[2] / (nsm // 2) / life:5.1%} | MMA wait(tempty) {b[1] / (nsm // 2) / life:5.1%} | "
              f"epilogue wait(tfull) {b[3] / (4 * nsm) / life:5.1%}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dsv3":   # E=256 experts of ~128 rows, H=7168, D_e=2048
        main(E=256, rows_per=128, H=7168, De=2048)
    else:
        main()
