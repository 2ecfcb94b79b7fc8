"""Per-role cycle breakdown of the cluster S-DP pipeline (profiling build).
PIPEDP_SDP_CHUNKED=0 PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so \\
    python tools/cluster_profile.py [log2n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2008_01938_b200 as pd  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
inst = pd.generate_sdp(n=1 << log2n, k=1024, seed=1, a1_cap=4096)
plan = pd.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init, "min")
d_init = torch.from_numpy(inst.init).cuda()
d_cells = torch.empty(inst.n, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
pd.profile_read(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
p = pd.profile_read(reset=True)
nb = max(p[3], 1)
print(plan.describe(), f"{e0.elapsed_time(e1):.2f} ms", "batches", nb,
      f"ns/batch {e0.elapsed_time(e1) * 1e6 / nb:.1f}")
print(f"  chain: wait mid {p[0] / nb:.0f}  wait far-mid {p[1] / nb:.0f}  total {p[2] / nb:.0f} cycles/batch")
for nm, o in (("near A", 8), ("near B", 16), ("far-mid", 12)):
    c = max(p[o + 3], 1)
    print(f"  {nm}: per batch it folds: wait {p[o] / c:.0f}  fold {p[o + 1] / c:.0f}  second wait {p[o + 2] / c:.0f} cycles")
