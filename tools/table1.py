"""Paper Table I on B200: the reference's --paper-scale bench buckets
(commands.cpp:347-379, seed 0, op min; n/k drawn by the reference's bucket
RNG = 29,103/7,168, 73,853/21,722, 493,505/123,928 -- SURVEY.md section 6)
with the reference's four solvers (commands.cpp:480-507):
  sequential  the reference library itself on one host core (oracle/_ref)
  naive       the paper's naive method on the GPU (sdp_naive)
  prefix      the paper's tournament method on the GPU (sdp_tournament)
  pipeline    the pipelined kernels (sdp_v2_multi)
Writes the reference's CSV (bucket,solver,mean_msec,result_digest,steps)
and the published Table I (GTX TITAN Black / Xeon E3-1245 v3)
beside it.  python tools/table1.py [--skip-naive-over N] [--out profiles/table1.csv]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_01938_b200 as pd

BUCKETS = [(29103, 7168, 0), (73853, 21722, 1), (493505, 123928, 2)]
PAPER = {  # ms, PAPER.md:340-347 (bucket regimes)
    0: {"sequential": 274, "naive": 64, "pipeline": 78},
    1: {"sequential": 4288, "naive": 368, "pipeline": 386},
    2: {"sequential": 68453, "naive": 3018, "pipeline": 2408},
}


def gpu_time(inst, method, reps):
    plan = pd.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init, inst.op)
    plan.set_method(method)
    d_init = torch.from_numpy(np.asarray(inst.init, dtype=np.int64)).cuda()
    d_cells = torch.empty(inst.n, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        plan.execute(d_init.data_ptr(), d_cells.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.mean(ts)), pd.table_digest(d_cells.cpu().numpy()), plan.describe()[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--naive-max-k", type=int, default=30000)  # the atomic method is O(nk) serialised
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from oracle import pyoracle  # the CPU reference (sequential) leg, as in bench.py
    ref = pyoracle.load_ref() or pyoracle.load_c()
    rows = ["bucket,solver,mean_msec,result_digest,steps,device,paper_msec"]
    for n, k, seed in BUCKETS:
        inst = pd.generate_sdp(n=n, k=k, op="min", seed=seed)
        label = f"n{n}-k{k}"
        computed = n - inst.a1
        t0 = time.perf_counter()
        cells, _ = ref.sdp_solve(inst.offsets, inst.init, n, "min")
        seq_ms = (time.perf_counter() - t0) * 1e3
        want = f"{ref.digest(cells):016x}"
        paper = PAPER[seed]
        rows.append(f"{label},sequential,{seq_ms:.3f},{want},{computed * k},cpu-1core,{paper['sequential']}")
        for solver, method, steps in (("naive", pd.SDP_NAIVE, computed * k),
                                      ("prefix", pd.SDP_PREFIX, computed * max((k - 1).bit_length(), 1)),
                                      ("pipeline", pd.SDP_PIPELINE, n + k - inst.a1 - 1)):
            if solver == "naive" and k > args.naive_max_k:
                rows.append(f"{label},{solver},,,{steps},skipped (O(nk) serialised atomics),{paper.get(solver, '')}")
                continue
            ms, dig, kern = gpu_time(inst, method, args.reps if solver == "pipeline" else 1)
            got = f"{dig:016x}"
            assert got == want, (label, solver, got, want)
            rows.append(f"{label},{solver},{ms:.3f},{got},{steps},{kern},{paper.get(solver, '')}")
        print("\n".join(rows[-4:]), flush=True)
    text = "\n".join(rows) + "\n"
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    print(text)


if __name__ == "__main__":
    main()
