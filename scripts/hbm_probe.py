"""Pure-write vs copy bandwidth on this B200 (context for the permute's write-bound phase)."""
import json
import torch
n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
tw = t(lambda: a.zero_())
tc = t(lambda: b.copy_(a))
ts = t(lambda: a.sum(dtype=torch.int64))
print(json.dumps({"write_GBs": round(n / tw / 1e6, 1), "copy_rw_GBs": round(2 * n / tc / 1e6, 1),
                  "read_GBs": round(n / ts / 1e6, 1)}))
