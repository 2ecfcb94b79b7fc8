"""Where an MCM host-buffer solve's time goes (GPU box): the Python call, the
raw C ABI call, and the device plan alone.  usage: python tools/mcm_e2e_breakdown.py [n]"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_01938_b200 as pd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
inst = pd.generate_mcm(n=n, seed=1, dims_min=1, dims_max=100)
dims = np.ascontiguousarray(inst.dims)
L = pd.lib()
size = pd.cell_count(n) + 1


def timeit(f, k=7):
    f()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * sorted(ts)[len(ts) // 2]


p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
cells, split, filled = np.empty(size, np.int64), np.empty(size, np.int64), np.empty(size, np.uint8)
print("python solve_mcm_with_split  min/med ms %.3f %.3f" % timeit(lambda: pd.solve_mcm_with_split(inst, pd.MCM_AUTO)))
print("C ABI, reused outputs        min/med ms %.3f %.3f" % timeit(
    lambda: L.pipedp_mcm_solve(p64(dims), len(dims), 0, p64(cells), filled.ctypes.data_as(C.POINTER(C.c_uint8)), p64(split))))
plan = pd.McmPlan(1, n, dims)
c = torch.empty(size, dtype=torch.int64, device="cuda")
s = torch.empty_like(c)
st = torch.cuda.current_stream()


def dev():
    plan.execute(c.data_ptr(), s.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()


print("device plan + sync           min/med ms %.3f %.3f" % timeit(dev))
