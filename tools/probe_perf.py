"""Developer probe: device-resident timings of each kernel family (CUDA events).
Not the bench (bench.py is); used to iterate on kernels."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2008_01938_b200 as pd


def timeit(fn, reps=3):
    st = torch.cuda.current_stream()
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); fn(); e1.record(st); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def sdp(n, k, cap, op="min", batch=1, seeds=None):
    offs, init = [], []
    for b in range(batch):
        i = pd.generate_sdp(n=n, k=k, op=op, seed=(seeds[b] if seeds else 1), a1_cap=cap)
        offs.append(i.offsets); init.append(i.init)
    a1 = len(init[0])
    offs = np.concatenate(offs); init = np.concatenate(init)
    plan = pd.SdpPlan(batch, n, k, a1, offs, init, op)
    d_init = torch.from_numpy(init).cuda()
    d_cells = torch.empty(batch * n, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ms = timeit(lambda: plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st))
    relax = batch * (n - a1) * k
    print(f"SDP n={n} k={k} a1={a1} op={op} batch={batch} {plan.describe()}: {ms:.3f} ms  {relax/ms/1e6:.3e} relax/s", flush=True)
    return d_cells


def sdp_fib(n, op):
    plan = pd.SdpPlan(1, n, 2, 2, [2, 1], [1, 1], op)
    d_init = torch.tensor([1, 1], dtype=torch.int64, device="cuda")
    d_cells = torch.empty(n, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ms = timeit(lambda: plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st))
    print(f"FIB n={n} op={op} {plan.describe()}: {ms:.3f} ms  {(n-2)*2/ms/1e6:.3e} relax/s", flush=True)


def mcm(n, kernel, batch=1):
    dims = np.concatenate([pd.generate_mcm(n, seed=(1 if batch == 1 else b), dims_min=1, dims_max=100).dims for b in range(batch)])
    plan = pd.McmPlan(batch, n, dims, kernel)
    size = batch * (n * (n + 1) // 2 + 1)
    c = torch.empty(size, dtype=torch.int64, device="cuda"); s = torch.empty_like(c)
    st = torch.cuda.current_stream().cuda_stream
    ms = timeit(lambda: plan.execute(c.data_ptr(), s.data_ptr(), st), reps=2 if n >= 4096 else 3)
    relax = batch * (n**3 - n) // 6
    print(f"MCM n={n} batch={batch} kernel={kernel} {plan.describe()}: {ms:.3f} ms  {relax/ms/1e6:.3e} relax/s", flush=True)
    return c, s


if __name__ == "__main__":
    what = sys.argv[1:] or ["all"]
    for op, bits in [("min", 32), ("min", 64), ("saturating-add", 64), ("modular-add", 32)]:
        print("chain step", op, bits, pd.chain_step_ns(op, bits))
    sdp_fib(1 << 20, "saturating-add")
    sdp_fib(1 << 20, "modular-add")
    sdp(1 << 20, 1024, 4096)
    sdp(1 << 24, 1024, 4096)
    sdp(1 << 16, 64, 0, batch=4096, seeds=list(range(4096)))
    mcm(64, 0, batch=8192)
    mcm(1024, 1)
    mcm(1024, 3)
    mcm(2048, 1)
    if "big" in what:
        mcm(8192, 1)
