"""Run exactly one configuration once (for ncu captures): python tools/one_kernel.py <name>"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_01938_b200 as pd

def sdp(n, k, cap, op="min", batch=1):
    offs, init = [], []
    for b in range(batch):
        i = pd.generate_sdp(n=n, k=k, op=op, seed=(1 if batch == 1 else b), a1_cap=cap)
        offs.append(i.offsets); init.append(i.init)
    a1 = len(init[0]); offs = np.concatenate(offs); init = np.concatenate(init)
    plan = pd.SdpPlan(batch, n, k, a1, offs, init, op)
    d_init = torch.from_numpy(init).cuda(); d_cells = torch.empty(batch * n, dtype=torch.int64, device="cuda")
    for _ in range(2):
        plan.execute(d_init.data_ptr(), d_cells.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()

def mcm(n, kernel, batch=1):
    dims = np.concatenate([pd.generate_mcm(n, seed=b + 1, dims_min=1, dims_max=100).dims for b in range(batch)])
    plan = pd.McmPlan(batch, n, dims, kernel)
    size = batch * (n * (n + 1) // 2 + 1)
    c = torch.empty(size, dtype=torch.int64, device="cuda"); s = torch.empty_like(c)
    for _ in range(2):
        plan.execute(c.data_ptr(), s.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()

cfg = sys.argv[1]
{
    "c2s": lambda: sdp(1 << 20, 1024, 4096),
    "c2": lambda: sdp(1 << 24, 1024, 4096),
    "c1": lambda: sdp(1 << 20, 2, 0, "saturating-add") if False else None,
    "c5b": lambda: sdp(1 << 16, 64, 0, batch=2048),
    "c5a": lambda: mcm(64, 0, batch=8192),
    "c3": lambda: mcm(1024, 1),
    "c4s": lambda: mcm(4096, 1),
}[cfg]()
