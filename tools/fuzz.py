"""Randomised S-DP / MCM parity sweep against the C oracle (test tooling; run on
a GPU box: PYTHONPATH=. python tools/fuzz.py [seconds]).  Draws shapes that hit
every dispatch (jump, serial, chunked, v2 pipeline, strict-order CTA, batches,
tiled / square MCM) and reports any mismatch with its seed."""
import sys
import time

import numpy as np

import paper_2008_01938_b200 as pd
from oracle import pyoracle

orc = pyoracle.load_c()
OPS = ["min", "max", "saturating-add", "modular-add"]
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
t0 = time.time()
rng = np.random.default_rng(int(time.time()))
stats, bad = {}, 0
it = 0
while time.time() - t0 < budget:
    it += 1
    seed = int(rng.integers(1 << 31))
    r = np.random.default_rng(seed)
    kind = r.choice(["sdp_small", "sdp_mid", "sdp_big", "mcm", "sdp_batch", "sdp_cluster", "mcm_batch"],
                    p=[0.18, 0.22, 0.1, 0.15, 0.12, 0.13, 0.1])
    if kind == "sdp_cluster":
        # one instance over the thread-block cluster (chunked mode off for min/max)
        import os
        op = ["min", "max", "modular-add"][int(r.integers(3))]
        a1 = int(r.integers(300, 20000))
        k = int(r.integers(70, min(a1 - 1, 3000)))
        n = int(r.integers(a1 + 1, 400000))
        rest = r.choice(np.arange(1, a1), k - 1, replace=False)
        offs = np.concatenate([[a1], np.sort(rest)[::-1]]).astype(np.int64)
        init = r.integers(-(1 << 30), 1 << 30, a1) if op != "modular-add" else r.integers(0, 2**31 - 1, a1)
        os.environ["PIPEDP_SDP_CHUNKED"] = "0"
        try:
            t = pd.solve_sequential(pd.SdpInstance(n, offs, init, op))
            plan = pd.SdpPlan(1, n, k, a1, offs, init, op)
            name = plan.describe()[0].split("[")[0]
            plan.close()
        finally:
            del os.environ["PIPEDP_SDP_CHUNKED"]
        want, _ = orc.sdp_solve(offs, init, n, op)
        ok = np.array_equal(t.cells, want)
    elif kind == "sdp_batch":
        # warp-per-instance batches (a_1 <= 128): the three sdp_batch_warp paths
        op = ["min", "max", "saturating-add", "modular-add"][int(r.integers(4))]
        a1 = int(r.integers(2, 129))
        k = int(r.integers(2, min(a1, 64) + 1))
        n = int(r.integers(a1 + 1, 20000))
        count = int(r.integers(2, 40))
        insts = []
        for _ in range(count):
            lo = int(r.integers(1, 4))
            pool = np.arange(lo, a1)
            if len(pool) < k - 1:
                pool = np.arange(1, a1)
            rest = r.choice(pool, k - 1, replace=False)
            offs = np.concatenate([[a1], np.sort(rest)[::-1]]).astype(np.int64)
            init = r.integers(-(1 << 30), 1 << 30, a1) if op != "modular-add" else r.integers(0, 2**31 - 1, a1)
            insts.append(pd.SdpInstance(n, offs, init, op))
        ok = True
        for inst, t in zip(insts, pd.solve_sequential_batch(insts)):
            want, _ = orc.sdp_solve(inst.offsets, inst.init, inst.n, op)
            ok = ok and np.array_equal(t.cells, want)
        plan = pd.SdpPlan(count, n, k, a1, np.concatenate([i.offsets for i in insts]),
                          np.concatenate([i.init for i in insts]), op)
        name = plan.describe()[0].split("[")[0]
        plan.close()
    elif kind == "mcm_batch":
        # n <= 64 batches: mcm_batch_warp (packed keys; dims up to 255 can pass
        # 2^24 and rerun unpacked; 1290 is never packed), odd and even counts
        n = int(r.integers(1, 65))
        dmax = int(r.choice([100, 255, 1290]))
        cnt = int(r.integers(1, 41))
        insts = [pd.McmInstance(orc.generate_mcm(n, (seed + i) % 100000, 1, dmax)) for i in range(cnt)]
        ok = True
        for inst, (t, split) in zip(insts, pd.solve_mcm_batch(insts)):
            wc, _, ws = orc.mcm_solve(inst.dims)
            ok = ok and np.array_equal(t.cells, wc) and np.array_equal(split, ws)
        name = f"mcm_batch n={n} x{cnt} dmax={dmax}"
    elif kind == "mcm":
        n = int(r.integers(2, 700))
        dims = orc.generate_mcm(n, seed % 1000, 1, int(r.choice([100, 322, 1290])))
        t, split = pd.solve_mcm_with_split(pd.McmInstance(dims), pd.MCM_AUTO)
        wc, _, ws = orc.mcm_solve(dims)
        ok = np.array_equal(t.cells, wc) and np.array_equal(split, ws)
        name = f"mcm n={n}"
    else:
        op = OPS[int(r.integers(4))]
        if kind == "sdp_small":
            a1 = int(r.integers(2, 64))
            n = int(r.integers(a1 + 1, 200000))
        elif kind == "sdp_mid":
            a1 = int(r.integers(64, 8192))
            n = int(r.integers(a1 + 1, 600000))
        else:
            a1 = int(r.integers(64, 8192))
            n = int(r.integers(1_000_000, 4_000_000))
        k = int(r.integers(1, min(a1, 1024) + 1))
        rest = r.choice(np.arange(1, a1), k - 1, replace=False) if k > 1 else np.array([], dtype=np.int64)
        offs = np.concatenate([[a1], np.sort(rest)[::-1]]).astype(np.int64)
        cls = int(r.integers(3))
        init = (r.integers(0, 1 << 20, a1) if cls == 0 else
                r.integers(-(1 << 40), 1 << 40, a1) if cls == 1 else r.integers(-(1 << 62), 1 << 62, a1))
        if n * k > 4e9:
            continue
        t = pd.solve_sequential(pd.SdpInstance(n, offs, init, op))
        want, _ = orc.sdp_solve(offs, init, n, op)
        ok = np.array_equal(t.cells, want)
        plan = pd.SdpPlan(1, n, k, a1, offs, init, op)
        name = plan.describe()[0].split("[")[0]
        plan.close()
    stats[name.split(" ")[0]] = stats.get(name.split(" ")[0], 0) + 1
    if not ok:
        bad += 1
        print(f"MISMATCH seed={seed} kind={kind} {name}", flush=True)
print(f"fuzz: {it} cases in {time.time() - t0:.0f} s, {bad} mismatches; by kernel: {stats}")
