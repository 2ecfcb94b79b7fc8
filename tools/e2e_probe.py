"""Breakdown of the c2 end-to-end call (host-buffer C ABI) on the GPU box."""
import time
import numpy as np
import torch
import paper_2008_01938_b200 as pd

inst = pd.generate_sdp(n=1 << 24, k=1024, op="min", seed=1, a1_cap=4096)


def t(f, reps=3):
    f()
    s = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - s) / reps * 1e3


print("validate ms", t(lambda: pd.validate(inst)))
print("np.empty+touch ms", t(lambda: np.empty(inst.n, np.int64).fill(0)))
print("plan create+destroy ms", t(lambda: pd.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init).close()))
plan = pd.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init)
d_init = torch.tensor(np.asarray(inst.init), dtype=torch.int64, device="cuda")
d_cells = torch.empty(inst.n, dtype=torch.int64, device="cuda")
def ex():
    plan.execute(d_init.data_ptr(), d_cells.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
print("execute+sync ms", t(ex))
print("solve_sequential ms", t(lambda: pd.solve_sequential(inst)))
out = np.empty(inst.n, np.int64)
print("d2h pinned-staged (torch to pageable) ms", t(lambda: out.__setitem__(slice(None), d_cells.cpu().numpy())))
