"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = collections.OrderedDict()
    for d in data:
        per.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("void ", "")
        if "grouped_gemm_kernel" in name:
            short = name[: name.index("(")].replace("void ", "")
        t = tot[short]
        t[0] += 1
        t[1] += m.get("gpu__time_duration.sum", 0)
        t[2] += m.get("dram__bytes_read.sum", 0)
        t[3] += m.get("dram__bytes_write.sum", 0)
    all_t = sum(v[1] for v in tot.values())
    out = []
    for n, (c, t, r, w) in sorted(tot.items(), key=lambda x: -x[1][1]):
        out.append(f"{n:48s} n={c:3d} total={t/1e3:9.1f}us {100*t/all_t:5.1f}%  per={t/c/1e3:8.1f}us "
                   f"rd={r/c/1e6:8.1f}MB wr={w/c/1e6:8.1f}MB")
    out.append(f"total {all_t/1e3:.1f} us over {len(per)} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
