"""Isolated cold-L2 timing of the dispatch stage (route_and_dispatch) at the Mixtral
shape, plus a hash of its outputs (for A/B comparisons of dispatch-kernel variants)."""

import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200 import _lib  # noqa: E402
from paper_2605_11005_b200 import kernels as K  # noqa: E402


def main(T=4096, H=4096, E=8, k=2, reps=50):
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn(T, H, generator=g).to(torch.bfloat16).to(dev)
    wg = (torch.randn(E, H, generator=g) * 0.02).to(dev)
    cap = _lib.capacity_rows(T, E, k)
    ws = torch.zeros(_lib.route_workspace_size(T, H, E, k), dtype=torch.uint8, device=dev)
    i32 = lambda *s: torch.empty(*s, dtype=torch.int32, device=dev)  # noqa: E731
    idx, rm = i32(T, k), i32(T, k)
    w = torch.empty(T, k, device=dev)
    counts, pad, src = i32(E), i32(E + 1), i32(cap)
    xp = torch.empty(cap, H, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    run = lambda: K.route_and_dispatch(x, wg, k, ws, idx, w, counts, pad, rm, src, xp)  # noqa: E731
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    h = hashlib.sha1()
    for t in (idx, rm, w, counts, pad, xp[: int(pad[-1])]):
        h.update((t.view(torch.int16) if t.dtype == torch.bfloat16 else t).cpu().numpy().tobytes())
    nbytes = T * H * 2 + T * k * H * 2 + 8 * T * k
    med = ts[len(ts) // 2]
    print(json.dumps({"E": E, "median_us": round(med, 1), "min_us": round(ts[0], 1),
                      "GB/s": round(nbytes / med / 1e3, 1), "hash": h.hexdigest()[:12]}))


if __name__ == "__main__":
    main()
    main(E=16)
