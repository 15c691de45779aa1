"""Convert an ncu CSV of one iteration's GEMM launches (dram__bytes_read/write.sum,
gpu__time_duration.sum) into profiles/<round>/gemm_traffic_<workload>.json, which
bench.py reports as roofline.traffic (measured DRAM bytes per step vs algorithmic).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        -k regex:grouped_gemm --launch-skip 18 --launch-count 18 --csv --log-file t.csv \\
        python scripts/profile_step.py
    python scripts/gemm_traffic.py t.csv --workload mixtral_layer --out profiles/r01/
"""
import argparse
import csv
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--config", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--kernel-regex", default="grouped_gemm", help="launches to count (a step's full list also "
                    "holds the A-side kernels)")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    launches: dict = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}
    import re

    for r in rows[1:]:
        if not re.search(a.kernel_regex, r[ki]):
            continue
        d = launches.setdefault(r[idi], {"kernel": r[ki].split("(")[0]})
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        d[r[mi]] = v
    out = []
    for d in launches.values():
        out.append({"kernel": d["kernel"], "dram_bytes": int(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)),
                    "ms": round(d.get("gpu__time_duration.sum", 0) * 1e3, 4)})
    from paper_2605_11005_b200.config import load_experiment
    from paper_2605_11005_b200.moe import MoEShape

    cfg = a.config or f"configs/{a.workload}.yaml"
    exp = load_experiment(cfg)
    shape = MoEShape.from_experiment(exp)
    total = sum(o["dram_bytes"] for o in out)
    alg = shape.gemm_hbm_bytes(exp.workload.num_microbatches)
    res = {"workload": a.workload, "launches": out, "bytes_per_iteration": total,
           "algorithmic_bytes_per_iteration": alg, "ratio": round(total / alg, 3),
           "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, one iteration after warm-up"}
    p = Path(a.out) / f"gemm_traffic_{a.workload}.json"
    p.write_text(json.dumps(res, indent=1))
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}))


if __name__ == "__main__":
    main()
