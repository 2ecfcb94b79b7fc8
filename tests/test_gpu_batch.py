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
