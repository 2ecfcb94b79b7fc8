"""Where C2's end-to-end time goes (GPU box): the Python solve, the raw C-ABI
call into a fresh / a reused output buffer, and the device-only execute.
usage: python tools/e2e_breakdown.py"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_01938_b200 as pd  # noqa: E402

inst = pd.generate_sdp(n=1 << 24, k=1024, op="min", seed=1, a1_cap=4096)
L = pd.lib()
offs, init = np.ascontiguousarray(inst.offsets), np.ascontiguousarray(inst.init)
p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731


def timeit(f, n=5):
    f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * sorted(ts)[len(ts) // 2]


reuse = np.empty(inst.n, np.int64)
print("pd.solve_sequential      min/med ms %.3f %.3f" % timeit(lambda: pd.solve_sequential(inst)))
print("C ABI, fresh output      min/med ms %.3f %.3f" % timeit(
    lambda: L.pipedp_sdp_solve(p64(offs), len(offs), p64(init), len(init), inst.n, 0, p64(np.empty(inst.n, np.int64)), None)))
print("C ABI, reused output     min/med ms %.3f %.3f" % timeit(
    lambda: L.pipedp_sdp_solve(p64(offs), len(offs), p64(init), len(init), inst.n, 0, p64(reuse), None)))
plan = pd.SdpPlan(1, inst.n, inst.k, inst.a1, offs, init, "min", device=0)
d_in = torch.from_numpy(init).cuda()
d_out = torch.empty(inst.n, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()


def dev():
    plan.execute(d_in.data_ptr(), d_out.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()


print("device execute + sync    min/med ms %.3f %.3f" % timeit(dev))
h = torch.empty(inst.n, dtype=torch.int64).pin_memory()
print("D2H 128 MiB pinned       min/med ms %.3f %.3f" % timeit(lambda: (h.copy_(d_out), torch.cuda.synchronize())))
