"""Print an `ncu --csv --metrics ...` log as one row per launch: kernel, then each metric
(bytes in GB, durations in us). Usage: python scripts/ncu_csv.py log.csv [log2.csv ...]"""
import csv
import sys

SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def rows(path):
    r = [x for x in csv.reader(open(path)) if len(x) > 10 and not x[0].startswith("==")]
    if not r:
        return []
    h = r[0]
    ki, mi, vi, ui, ii = (h.index(n) for n in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    out = {}
    for x in r[1:]:
        d = out.setdefault(x[ii], {"kernel": x[ki].split("(")[0].replace("void ", "")[:48]})
        try:
            d[x[mi]] = round(float(x[vi].replace(",", "")) * SCALE.get(x[ui], 1.0), 4)
        except ValueError:
            d[x[mi]] = x[vi]
    return list(out.values())


for p in sys.argv[1:]:
    print(f"== {p}")
    for d in rows(p):
        print("  ", "  ".join(f"{k}={v}" for k, v in d.items()))
