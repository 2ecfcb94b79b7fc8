"""Small instances of every kernel family, each checked against the C oracle --
the workload tests/test_gpu_sanitizer.py runs under compute-sanitizer
(memcheck / racecheck / synccheck).
usage: python tools/sanitize_cases.py [all|plain|mbarrier]
  plain:    kernels whose shared memory is ordered by __syncthreads / __syncwarp
            (and grid barriers): racecheck models those exactly;
  mbarrier: the warp-specialised pipelines ordered by mbarrier arrive
            (release) / try_wait (acquire), which racecheck does not model."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2008_01938_b200 as pd  # noqa: E402
from oracle import pyoracle  # noqa: E402

orc = pyoracle.load_c()


def sdp(inst, label):
    t = pd.solve_sequential(inst)
    want, _ = orc.sdp_solve(inst.offsets, inst.init, inst.n, inst.op)
    assert np.array_equal(t.cells, want), label
    print("ok", label, flush=True)


def main(which="all"):
    plain, mbar = which in ("all", "plain"), which in ("all", "mbarrier")
    if mbar:
        mbarrier_cases()
    if plain:
        plain_cases()
    print("ALL OK")


def mbarrier_cases():
    # S-DP single instances: chunked ranks (min/max), v2 pipeline, strict (mixed-sign
    # sat-add), jump segments, tiny serial, multi-CTA (wide a_1)
    sdp(pd.generate_sdp(n=70000, k=64, op="min", seed=3, a1_cap=128), "sdp chunked-rank min")
    sdp(pd.generate_sdp(n=70000, k=48, op="max", seed=4, a1_cap=100), "sdp chunked-rank max")
    sdp(pd.generate_sdp(n=6000, k=64, op="modular-add", seed=5, a1_cap=300), "sdp v2 mod-add")
    i = pd.generate_sdp(n=3000, k=24, op="saturating-add", seed=6, a1_cap=90)
    i.init[::2] *= -1
    sdp(i, "sdp strict mixed-sign sat-add")
    sdp(pd.generate_sdp(n=30000, k=256, op="modular-add", seed=7, a1_cap=9000), "sdp multi-CTA")
    dims = pd.generate_mcm(n=200, seed=200, dims_min=1, dims_max=100).dims
    t, split = pd.solve_mcm_with_split(pd.McmInstance(dims), pd.MCM_AUTO)
    wc, _, ws = orc.mcm_solve(dims)
    assert np.array_equal(t.cells, wc) and np.array_equal(split, ws), "tiled"
    print("ok mcm tiled", flush=True)


def plain_cases():
    sdp(pd.SdpInstance(9000, [3, 2, 1], [1, 2, 3], "saturating-add"), "sdp jump")
    sdp(pd.SdpInstance(500, [5, 3, 1], [4, 1, 7, 2, 9], "min"), "sdp serial")
    # S-DP batches: dominance kernel (+ fallback warp kernel), general warp kernel
    for op in ("min", "modular-add"):
        offs, init = pd.generate_sdp_batch(3000, 16, 11, 24)
        insts = [pd.SdpInstance(3000, o, v, op) for o, v in zip(offs, init)]
        for inst, t in zip(insts, pd.solve_sequential_batch(insts)):
            want, _ = orc.sdp_solve(inst.offsets, inst.init, inst.n, op)
            assert np.array_equal(t.cells, want), op
        print("ok sdp batch", op, flush=True)
    # MCM: tiled (n > 160), shared-memory CTA, wavefront, tournament, batch squares
    for n, kern, label in ((60, pd.MCM_SMEM, "smem"),
                           (90, pd.MCM_WAVEFRONT, "wavefront"), (70, pd.MCM_TOURNAMENT, "tournament")):
        dims = pd.generate_mcm(n=n, seed=n, dims_min=1, dims_max=100).dims
        t, split = pd.solve_mcm_with_split(pd.McmInstance(dims), kern)
        wc, _, ws = orc.mcm_solve(dims)
        assert np.array_equal(t.cells, wc) and np.array_equal(split, ws), label
        print("ok mcm", label, flush=True)
    for n in (32, 64):  # mcm_batch_warp: one- and two-pass diagonals, an odd batch
        insts = [pd.generate_mcm(n=n, seed=s, dims_min=1, dims_max=100) for s in range(5)]
        for inst, (t, split) in zip(insts, pd.solve_mcm_batch(insts)):
            wc, _, ws = orc.mcm_solve(inst.dims)
            assert np.array_equal(t.cells, wc) and np.array_equal(split, ws)
    print("ok mcm batch", flush=True)
    # the lock-step engine with its device analyses, both programs
    r = pd.solve_mcm_pipeline(pd.generate_mcm(n=20, seed=2, dims_min=1, dims_max=50), "paper_literal")
    assert len(r.hazards.hazards) > 0
    r = pd.solve_sdp_pipeline(pd.generate_sdp(n=600, k=8, op="min", seed=2))
    assert r.trace.collected
    print("ok engine", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
