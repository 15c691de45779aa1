import sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_2605_11005_b200 import _lib
from paper_2605_11005_b200 import kernels as K
T,H,E,k=4096,4096,8,2
dev="cuda"
g=torch.Generator(device="cpu").manual_seed(0)
x=torch.randn(T,H,generator=g).to(torch.bfloat16).to(dev)
wg=(torch.randn(E,H,generator=g)*0.02).to(dev)
cap=_lib.capacity_rows(T,E,k)
ws=torch.zeros(_lib.route_workspace_size(T,H,E,k),dtype=torch.uint8,device=dev)
i32=lambda *s: torch.empty(*s,dtype=torch.int32,device=dev)
idx,rm=i32(T,k),i32(T,k); w=torch.empty(T,k,device=dev); counts,pad,src=i32(E),i32(E+1),i32(cap)
xp=torch.empty(cap,H,dtype=torch.bfloat16,device=dev)
flush=torch.empty(512<<20,dtype=torch.uint8,device=dev)
run=lambda: K.route_and_dispatch(x,wg,k,ws,idx,w,counts,pad,rm,src,xp)
def t(fn, reps=20):
    ts=[]
    for _ in range(reps):
        flush.zero_()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
    ts.sort(); return round(ts[len(ts)//2],1)
for _ in range(3): run()
print(json.dumps({"once": t(run), "twice": t(lambda: (run(), run())), "thrice": t(lambda: (run(), run(), run()))}))
# per-CTA timeline of one launch
NC = 160
prof = torch.zeros(NC * 64, dtype=torch.int64, device=dev)
_lib.load().dm_debug_route_profile(prof.data_ptr())
flush.zero_(); torch.cuda.synchronize()
run(); torch.cuda.synchronize()
_lib.load().dm_debug_route_profile(None)
import numpy as np
p = prof.view(NC, 64).cpu().numpy().astype("int64")
p = p[p[:, 0] > 0]
t0 = p[:, 0].min()
rel = lambda v: (v - t0) / 1e3
names = ["start", "W ready", "units done", "barrier", "permute done"]
for j, n in enumerate(names):
    v = p[:, j]; m = v > 0
    if m.any():
        r = rel(v[m]); print(f"{n:13s} n={m.sum():3d} med {np.median(r):6.2f} max {r.max():6.2f} us")
for i in range(8):
    v = p[:, 16 + i]; m = v > 0
    if m.any():
        r = rel(v[m]); print(f"unit {i} math done med {np.median(r):6.2f} max {r.max():6.2f}")
