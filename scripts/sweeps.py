"""BASELINE configs #4 (long-context seq sweep) and #5 (A:F allocation x micro-batch
sweep): run bench.py for each point and collect the JSON lines.

    python scripts/sweeps.py alloc   --gpus 4 --out gpurun_out/sweep_alloc.jsonl
    python scripts/sweeps.py seqlen  --gpus 4 --out gpurun_out/sweep_seq.jsonl
"""

import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def run(gpus: int, extra: list[str], port: int, steps: int, warmup: int) -> dict | None:
    if gpus == 1:
        cmd = [sys.executable, str(ROOT / "bench.py")]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py")]
    cmd += ["--gpus", str(gpus), "--steps", str(steps), "--warmup", str(warmup), "--no-cpu-baseline", *extra]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    for line in res.stdout.splitlines()[::-1]:
        if line.startswith("{"):
            return json.loads(line)
    print("FAILED", extra, res.stderr[-2000:], file=sys.stderr)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["alloc", "seqlen", "layers"])
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--attention", action="store_true", help="A-side attention in every layer (bench --attention)")
    ap.add_argument("--with-fused", action="store_true", help="also run each point on 1 GPU (fused path)")
    a = ap.parse_args()
    points = []
    if a.what == "alloc":
        for n_attn in range(1, a.gpus):
            for mb in (2, 4, 8):
                points.append((["--n-attn", str(n_attn), "--microbatches", str(mb)], {"A": n_attn, "F": a.gpus - n_attn, "mb": mb}))
    elif a.what == "layers":   # virtual stages (p = 1): measured memory vs the reference model
        for L in (1, 2, 4):
            points.append((["--layers", str(L)], {"layers": L}))
    else:
        for s in (2048, 4096, 8192, 16384, 32768):
            mb = 4 if s <= 8192 else 2
            points.append((["--seq-len", str(s), "--microbatches", str(mb)], {"seq_len": s, "mb": mb}))
    with open(a.out, "w") as fh:
        for i, (extra, meta) in enumerate(points):
            if a.attention:
                extra = extra + ["--attention"]
            line = run(a.gpus, extra, 29600 + i, a.steps, a.warmup)
            if line is None:
                continue
            row = {**meta, "attention": a.attention, "tokens_per_s": line["value"], "ms_per_step": line["ms_per_step"],
                   "exposed_comm": line.get("exposed_comm"), "gemm_frac": line["roofline"]["frac"],
                   "clocks": line.get("clocks"), "e2e": line["e2e"]["value"], "memory": line.get("memory")}
            if a.with_fused:
                fused = run(1, [x for x in extra if x not in ("--n-attn",)] if "--n-attn" not in extra else
                            extra[:extra.index("--n-attn")] + extra[extra.index("--n-attn") + 2:], 0, a.steps, a.warmup)
                if fused is not None:
                    row["fused_1gpu_tokens_per_s"] = fused["value"]
                    row["fused_attention_ms_per_mb"] = (fused.get("attention") or {}).get("ms_per_microbatch_layer")
                    row["speedup_vs_fused"] = round(line["value"] / fused["value"], 3)
            fh.write(json.dumps(row) + "\n")
            fh.flush()
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
