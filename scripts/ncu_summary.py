"""Summarise an `ncu --set full` report (CSV raw page) into the JSON committed under
profiles/: per launch duration, DRAM bytes, tensor-pipe / smem-tensor activity, L2 hit
rate, occupancy and the top warp-stall reasons.

    ncu -i rep.ncu-rep --page raw --csv > raw.csv; python scripts/ncu_summary.py raw.csv out.json
"""
import csv
import json
import sys

KEYS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smem_tensor_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "regs": "launch__registers_per_thread",
}


def main(src, dst):
    rows = list(csv.reader(open(src)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")][:70]}
        for k, m in KEYS.items():
            if m in h:
                v = r[h.index(m)]
                u = units[h.index(m)]
                try:
                    f = float(v.replace(",", ""))
                    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1, "us": 1,
                             "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3,
                             "Mhz": 1e6, "Ghz": 1e9, "hz": 1}.get(u, 1)
                    d[k] = round(f * scale, 3)
                except ValueError:
                    d[k] = v
        cols = [i for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled")
                and n.endswith("_per_issue_active.ratio")]
        st = sorted(((float(r[i]) if r[i] not in ("", "n/a") else 0.0,
                      h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for i in cols), reverse=True)[:4]
        d["top_stalls_cycles_per_issue"] = [[n, round(v, 2)] for v, n in st]
        out.append(d)
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
