"""Batch driver on the GPU: per-instance tables of a sharded batch equal the
checker's, and the digest list is identical for every shard count (the
cross-device-count parity of SURVEY.md 4: each world size is simulated here
by solving its shards one after the other on cuda:0)."""
import numpy as np
import pytest
import torch

from paper_2008_01938_b200 import batch as B

pytestmark = pytest.mark.gpu


def _digests(spec, world, split=False):
    out = []
    st = torch.cuda.current_stream()
    for r in range(world):
        s = B.BatchShard(spec, r, world, 0)
        s.upload(st)
        s.execute(st)
        out.append(s.digests(st, split).cpu().numpy().view(np.uint64).copy())
    torch.cuda.synchronize()
    return np.concatenate(out)


def test_sdp_batch_digests_match_oracle_and_world(gpu, oracle):
    spec = B.SdpBatchSpec(total=300, n=4096, k=64, op="min", seed0=40)
    d1 = _digests(spec, 1)
    offs, init = gpu.generate_sdp_batch(spec.n, spec.k, spec.seed0, spec.total)
    want = np.array([oracle.digest(oracle.sdp_solve(o, i, spec.n, "min")[0]) for o, i in zip(offs, init)],
                    dtype=np.uint64)
    assert np.array_equal(d1, want)
    for world in (2, 3, 8):
        assert np.array_equal(_digests(spec, world), d1)


@pytest.mark.parametrize("op", ["max", "saturating-add", "modular-add"])
def test_sdp_batch_ops(gpu, oracle, op):
    spec = B.SdpBatchSpec(total=40, n=3000, k=64, op=op, seed0=3)
    d = _digests(spec, 2)
    offs, init = gpu.generate_sdp_batch(spec.n, spec.k, spec.seed0, spec.total)
    want = [oracle.digest(oracle.sdp_solve(o, i, spec.n, op)[0]) for o, i in zip(offs, init)]
    assert d.tolist() == want


def test_mcm_batch_cells_and_split(gpu, oracle):
    spec = B.McmBatchSpec(total=257, n=64, seed0=9)
    dc, dsp = _digests(spec, 1), _digests(spec, 1, split=True)
    dims = gpu.generate_mcm_batch(spec.n, spec.seed0, spec.total)
    wc, ws = [], []
    for d in dims:
        c, _, s = oracle.mcm_solve(d)
        wc.append(oracle.digest(c))
        ws.append(oracle.digest(s))
    assert dc.tolist() == wc and dsp.tolist() == ws
    assert np.array_equal(_digests(spec, 4), dc)


def test_config5_sample_digests(gpu, oracle):
    # the first instances of BASELINE config 5 (a and b) against the checker
    sb = B.SdpBatchSpec(total=65536)
    s = B.BatchShard(sb, 0, 1024, 0)  # shard 0 of 1024 = instances 0..63
    st = torch.cuda.current_stream()
    s.upload(st)
    s.execute(st)
    got = s.digests(st).cpu().numpy().view(np.uint64)
    for i in (0, 7, 63):
        c, _ = oracle.sdp_solve(s.h_offsets[i], s.h_init[i], sb.n, "min")
        assert int(got[i]) == oracle.digest(c)


@pytest.mark.parametrize("op", ["min", "max"])
def test_sdp_batch_dominance_forms(gpu, oracle, op):
    # a_1 = 128 batches mixing the three paths of sdp_batch_warp: offset 1
    # (dominance form), no offset 1 but every d in [2, 127] a sum of offsets
    # (second form: {2, 3} and {2, 5}), and neither ({4, 6, ...} only)
    rng = np.random.default_rng(11 if op == "min" else 12)
    insts = []
    for i in range(48):
        kind = i % 4
        must = [1, 7] if kind == 0 else [2, 3] if kind == 1 else [2, 5] if kind == 2 else [4, 6]
        pool = np.arange(4, 128, 2) if kind == 3 else np.arange(2 if kind else 1, 128)
        pool = pool[~np.isin(pool, must + [128])]
        rest = rng.choice(pool, 40, replace=False)  # every instance: k = 43
        offs = np.sort(np.concatenate([[128], must, rest]))[::-1].astype(np.int64)
        init = rng.integers(-(2**30), 2**30, 128)
        insts.append(gpu.SdpInstance(6000, offs, init, op))
    for inst, t in zip(insts, gpu.solve_sequential_batch(insts)):
        want, _ = oracle.sdp_solve(inst.offsets, inst.init, inst.n, op)
        assert np.array_equal(t.cells, want)


# --- BASELINE config 5 at full size: every instance against the reference ----
# tests/golden/c5*_cells.npy / c5a_split.npy hold table_digest of all 65,536
# instances, produced by the reference library itself (make_c5_digests.py).

def _golden(name):
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", name))


def _full_batch_digests(spec, split=False):
    st = torch.cuda.current_stream()
    s = B.BatchShard(spec, 0, 1, 0)
    s.upload(st)
    s.execute(st)
    cells = s.digests(st).cpu().numpy().view(np.uint64).copy()
    sp = s.digests(st, split=True).cpu().numpy().view(np.uint64).copy() if split else None
    torch.cuda.synchronize()
    del s
    torch.cuda.empty_cache()
    return cells, sp


def test_config5a_full_batch_bit_exact(gpu):
    cells, split = _full_batch_digests(B.McmBatchSpec(), split=True)
    want_c, want_s = _golden("c5a_cells.npy"), _golden("c5a_split.npy")
    bad = np.nonzero(cells != want_c)[0]
    assert bad.size == 0, f"{bad.size} C5a cell tables differ, first instance {bad[:8]}"
    bad = np.nonzero(split != want_s)[0]
    assert bad.size == 0, f"{bad.size} C5a split tables differ, first instance {bad[:8]}"


def test_config5b_full_batch_bit_exact(gpu):
    cells, _ = _full_batch_digests(B.SdpBatchSpec())
    want = _golden("c5b_cells.npy")
    bad = np.nonzero(cells != want)[0]
    assert bad.size == 0, f"{bad.size} C5b tables differ, first instance {bad[:8]}"


def test_config5b_sharded_full_batch(gpu):
    # the strong-scaling shards of the bench (W = 8), solved one after another
    spec = B.SdpBatchSpec()
    want = _golden("c5b_cells.npy")
    st = torch.cuda.current_stream()
    for r in (0, 5, 7):
        s = B.BatchShard(spec, r, 8, 0)
        s.upload(st)
        s.execute(st)
        got = s.digests(st).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want[s.lo:s.hi]), f"shard {r} of 8 differs"
        del s
        torch.cuda.empty_cache()


def test_bench_two_ranks_share_one_gpu(gpu):
    # bench.py --gpus 2 starts its own ranks (gloo when they share the GPU);
    # the gathered digest list of the sharded C5b batch equals the reference's
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "c5b",
                          "--steps", "1", "--warmup", "1", "--no-cpu-baseline", "--e2e-steps", "0"],
                         capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "shard2"
    assert line["parity"]["match"] is True and line["parity"]["instances"] == 65536


def _mk(rng, a1, must, nrest, lo, n, op, step=1):
    pool = np.arange(lo, a1, step)
    pool = pool[~np.isin(pool, must)]
    rest = rng.choice(pool, min(nrest, len(pool)), replace=False)
    offs = np.unique(np.concatenate([[a1], must, rest]))[::-1].astype(np.int64)
    return offs, rng.integers(-(2**30), 2**30, a1)


@pytest.mark.parametrize("op", ["min", "max"])
@pytest.mark.parametrize("a1", [64, 97, 128])
def test_sdp_batch_dominance_kernel(gpu, oracle, op, a1):
    """sdp_batch_dom (window + closure form) on the shapes that stress it: F
    non-empty below g (in-step D terms), g near 32, odd a_1 (window start lane
    shuffles), and instances with g > 32 that must fall back to sdp_batch_warp
    in the same plan."""
    rng = np.random.default_rng(a1 * 7 + (op == "max"))
    kinds = [([1], 1), ([2, 3], 2), ([3, 5], 3), ([4, 6, 9], 4), ([7, 11], 6), ([5, 8], 3),
             ([13, 17, 19], 12), ([20, 25, 31], 20), ([33, 34], 33), ([40], 40)]
    n, k = 5000, None
    insts = []
    for i in range(60):
        must, lo = kinds[i % len(kinds)]
        offs, init = _mk(rng, a1, [m for m in must if m < a1], 24, max(lo, 1), n, op)
        insts.append((offs, init))
    k = min(len(o) for o, _ in insts)  # the batch API needs one k: trim each to its k largest + must
    batch = []
    for offs, init in insts:
        o = np.concatenate([offs[:k - 1], offs[-1:]]) if len(offs) > k else offs
        o = np.unique(o)[::-1].astype(np.int64)
        if len(o) < k:  # pad with fresh large offsets
            extra = [d for d in range(a1 - 1, 0, -1) if d not in o][: k - len(o)]
            o = np.unique(np.concatenate([o, extra]))[::-1].astype(np.int64)
        batch.append(gpu.SdpInstance(n, o, init, op))
    offs = np.stack([b.offsets for b in batch]).reshape(-1)
    init = np.stack([b.init for b in batch]).reshape(-1)
    plan = gpu.SdpPlan(len(batch), n, k, a1, offs, init, op, device=0)
    name = plan.describe()[0]
    assert name.startswith("sdp_batch_dom"), name
    for inst, t in zip(batch, gpu.solve_sequential_batch(batch)):
        want, _ = oracle.sdp_solve(inst.offsets, inst.init, inst.n, op)
        assert np.array_equal(t.cells, want), (list(inst.offsets[-6:]), op, a1)
