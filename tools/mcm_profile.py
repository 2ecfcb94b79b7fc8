"""Task-level profile of the tiled MCM kernel (profiling build).
PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so python tools/mcm_profile.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_01938_b200 as pd
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dims = pd.generate_mcm(n=n, seed=1, dims_min=1, dims_max=100).dims
plan = pd.McmPlan(1, n, dims, pd.MCM_TILED)
size = pd.cell_count(n) + 1
c = torch.empty(size, dtype=torch.int64, device="cuda"); s = torch.empty_like(c)
st = torch.cuda.current_stream()
plan.execute(c.data_ptr(), s.data_ptr(), st.cuda_stream); torch.cuda.synchronize()
pd.profile_read(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); plan.execute(c.data_ptr(), s.data_ptr(), st.cuda_stream); e1.record(st)
torch.cuda.synchronize()
p = pd.profile_read(reset=True)
print(plan.describe(), f"{e0.elapsed_time(e1):.3f} ms")
for kind, nm in enumerate(["diag", "near", "far"]):
    tot, wait, cnt = p[32 + 4 * kind], p[33 + 4 * kind], p[34 + 4 * kind]
    if cnt:
        print(f"  {nm:5s} tasks {cnt:8d}  avg {tot / cnt:10.0f} cyc  avg wait+load {wait / cnt:10.0f} cyc  compute {(tot - wait) / cnt:10.0f} cyc")
if p[42]:
    print(f"  far: flag wait {p[47] / p[42]:.0f} cyc of the wait+load")
if p[38]:
    print(f"  near split: init {p[44]/p[38]:.0f}  wavefront {p[45]/p[38]:.0f}  finish {p[46]/p[38]:.0f} cyc")
if p[38]:
    print("  near wavefront cumulative cycles at steps 15/31/63/95/126:", [round(p[48 + i] / p[38]) for i in range(5)])
t0 = p[63]
lv = [(d, (p[64 + d] - t0) / 1e3) for d in range(64) if p[64 + d]]
print("  level finish (us):", " ".join(f"{d}:{t:.0f}" for d, t in lv[:40]))
