"""Our grouped GEMMs vs library GEMMs on the same ragged shapes (Mixtral expert layer,
8 experts x 1024 rows): cuBLAS per-expert torch.matmul (bf16, fp32 accumulate) and
torch._grouped_mm when this torch build provides it. Plain-output GEMMs only (w2 fwd:
[rows, D_e] x W2^T; w13 dgrad: [rows, 2 D_e] x W13), so the work is identical."""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import kernels as K  # noqa: E402


def timed(fn, reps=10):
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


def main(E=8, rows=1024, H=4096, De=14336):
    dev = "cuda"
    R = E * rows
    po = torch.tensor([i * rows for i in range(E + 1)], dtype=torch.int32, device=dev)
    act = torch.randn(R, De, device=dev).to(torch.bfloat16)
    w2 = (torch.randn(E, H, De, device=dev) * 0.02).to(torch.bfloat16)
    y = torch.empty(R, H, dtype=torch.bfloat16, device=dev)
    dh13 = torch.randn(R, 2 * De, device=dev).to(torch.bfloat16)
    w13 = (torch.randn(E, 2 * De, H, device=dev) * 0.02).to(torch.bfloat16)
    dx = torch.empty(R, H, dtype=torch.bfloat16, device=dev)
    out = {}
    cases = {
        "w2_fwd": (2 * R * H * De,
                   lambda: K.w2_fwd(act, w2, po, y),
                   lambda: [torch.matmul(act[i * rows:(i + 1) * rows], w2[i].t(), out=y[i * rows:(i + 1) * rows])
                            for i in range(E)],
                   lambda: torch._grouped_mm(act, w2.transpose(1, 2), offs=po[1:])),
        "w13_dgrad": (2 * R * 2 * De * H,
                      lambda: K.w13_dgrad(dh13, w13, po, dx),
                      lambda: [torch.matmul(dh13[i * rows:(i + 1) * rows], w13[i], out=dx[i * rows:(i + 1) * rows])
                               for i in range(E)],
                      lambda: torch._grouped_mm(dh13, w13, offs=po[1:])),
    }
    for name, (fl, ours, cublas, grouped) in cases.items():
        r = {"ours_ms": timed(ours), "cublas_per_expert_ms": timed(cublas)}
        try:
            r["torch_grouped_mm_ms"] = timed(grouped)
            ref = grouped()
            got = y if name == "w2_fwd" else dx
            ours()
            torch.cuda.synchronize()
            r["max_rel_diff_vs_grouped_mm"] = float(((got.float() - ref.float()).abs().max() / ref.float().abs().max()))
        except Exception as ex:  # noqa: BLE001
            r["torch_grouped_mm"] = f"unavailable: {type(ex).__name__}: {str(ex)[:100]}"
        for k in list(r):
            if k.endswith("_ms"):
                r[k.replace("_ms", "_TFLOPs")] = round(fl / r[k] / 1e9, 1)
                r[k] = round(r[k], 4)
        out[name] = r
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
