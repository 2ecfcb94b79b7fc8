"""Role-level cycle breakdown of sdp_v2 (profiling build).
PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so python tools/v2_profile.py [log2n] [k] [cap]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_01938_b200 as pd
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
inst = pd.generate_sdp(n=1 << log2n, k=k, seed=1, a1_cap=cap)
plan = pd.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init, "min")
d_init = torch.from_numpy(inst.init).cuda(); d_cells = torch.empty(inst.n, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st.cuda_stream); torch.cuda.synchronize()
pd.profile_read(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st.cuda_stream); e1.record(st)
torch.cuda.synchronize()
p = pd.profile_read(reset=True)
nb = max(p[3], 1)
print(plan.describe(), f"{e0.elapsed_time(e1):.2f} ms", "batches", nb)
names = {0: "chain.wait_mid", 1: "chain.work", 2: "chain.total", 8: "comb.wait_chain", 9: "comb.wait_near",
         10: "comb.wait_remote", 11: "comb.work", 16: "near0.wait", 17: "near0.fold", 18: "nearX.wait(sum)",
         19: "nearX.fold(sum)", 28: "writer.wait_chain", 29: "writer.publish", 24: "prod.wait_pub(warp0)", 25: "prod.fold+combine(warp0)"}
for i, nm in names.items():
    print(f"  {nm:28s} {p[i] / nb:10.1f} cycles/batch (summed over warps)")
