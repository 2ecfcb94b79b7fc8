cat > /tmp/t.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, time
import paper_2008_01938_b200 as pd
inst = pd.generate_sdp(n=1 << 24, k=1024, op="min", seed=1, a1_cap=4096)
pd.solve_sequential(inst)
ts = []
for i in range(8):
    t0 = time.perf_counter(); pd.solve_sequential(inst); ts.append(1e3 * (time.perf_counter() - t0))
print("fresh  min %.3f med %.3f" % (min(ts), sorted(ts)[4]))
out = np.empty(inst.n, np.int64); fl = np.empty(inst.n, np.uint8)
import ctypes as C
p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
offs, init = inst.offsets, inst.init
ts = []
for i in range(8):
    t0 = time.perf_counter(); pd.lib().pipedp_sdp_solve(p(offs), len(offs), p(init), len(init), inst.n, 0, p(out), fl.ctypes.data_as(C.POINTER(C.c_uint8))); ts.append(1e3 * (time.perf_counter() - t0))
print("reused min %.3f med %.3f" % (min(ts), sorted(ts)[4]))
PY
