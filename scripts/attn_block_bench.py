"""AttentionBlock fwd / bwd time with the own forward kernel vs the all-library block."""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200.attention import AttentionBlock  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    H = 4096
    for s, b, g in ((4096, 1, 1), (32768, 1, 1), (8192, 1, 4)):
        x = torch.randn(b * s, H, device=dev).to(torch.bfloat16)
        dh = torch.randn_like(x)
        row = {"seq": s, "gqa": g}
        for own in (True, False):
            blk = AttentionBlock(H, g, dev, own_kernel=own)
            out, dx = torch.empty_like(x), torch.empty_like(x)
            for _ in range(2):
                blk.forward(0, x, out, s)
                blk.backward(0, dh, dx, False)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            blk.forward(0, x, out, s)
            ev[1].record()
            blk.backward(0, dh, dx, False)
            ev[2].record()
            torch.cuda.synchronize()
            k = "own" if own else "lib"
            row[k + "_fwd_ms"] = round(ev[0].elapsed_time(ev[1]), 3)
            row[k + "_bwd_ms"] = round(ev[1].elapsed_time(ev[2]), 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
