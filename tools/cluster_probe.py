"""Time the cluster S-DP pipeline on a C2-shaped instance (PIPEDP_SDP_CHUNKED=0).
usage: PIPEDP_SDP_CHUNKED=0 python tools/cluster_probe.py [n_log2] [op]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_01938_b200 as pd  # noqa: E402

nl = int(sys.argv[1]) if len(sys.argv) > 1 else 20
op = sys.argv[2] if len(sys.argv) > 2 else "min"
inst = pd.generate_sdp(n=1 << nl, k=1024, op=op, seed=1, a1_cap=4096)
plan = pd.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init, op, device=0)
print(plan.describe(), flush=True)
d_in = torch.from_numpy(inst.init).cuda()
d_out = torch.empty(inst.n, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
plan.execute(d_in.data_ptr(), d_out.data_ptr(), st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
plan.execute(d_in.data_ptr(), d_out.data_ptr(), st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
nb = (inst.n - inst.a1 + 31) // 32
print(f"{ms:.3f} ms, {ms * 1e6 / nb:.1f} ns per 32-cell batch", flush=True)
