"""Phase-2 cost probe: the c2 offsets as a batch of G chunk instances."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2008_01938_b200 as pd
inst = pd.generate_sdp(n=1 << 24, k=1024, op="min", seed=1, a1_cap=4096)
a1, k = inst.a1, inst.k
G = int(os.environ.get("G", "256"))
Lc = -(-(inst.n - a1) // G)
Lc = (Lc + 31) // 32 * 32
n_i = a1 + Lc
offs = np.tile(np.asarray(inst.offsets, np.int64), G)
init = np.random.default_rng(0).integers(0, 1000, G * a1).astype(np.int64)
plan = pd.SdpPlan(G, n_i, k, a1, offs, init, "min")
d_init = torch.from_numpy(init).cuda()
d_out = torch.empty(G * n_i, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
plan.execute(d_init.data_ptr(), d_out.data_ptr(), st.cuda_stream); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); plan.execute(d_init.data_ptr(), d_out.data_ptr(), st.cuda_stream); e1.record(st)
torch.cuda.synchronize()
print(os.environ.get("TAG", ""), G, Lc, plan.describe(), f"{e0.elapsed_time(e1):.2f} ms")
