"""Pin the checker: the C restatement of the reference (oracle/pipedp_oracle.c)
against (1) the golden vectors produced by the reference itself
(tests/golden/golden.json, made by tests/golden/make_golden.py from
oracle/_ref), (2) the SPEC known-answer tests (SPEC.md lines cited per test)
and (3) the reference library directly, when oracle/_ref is built here.
CPU only."""
import json
import os

import numpy as np
import pytest

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
OPS = ["min", "max", "saturating-add", "modular-add"]


def hx(d):
    return f"{d:016x}"


# ------------------------------------------------------------ golden vectors --
def test_golden_apply(oracle):
    for op, a, b, want in GOLDEN["apply"]:
        assert oracle.apply(op, a, b) == want, (op, a, b)


def test_golden_sdp_full_tables(oracle):
    for case in GOLDEN["sdp_full"]:
        cells, filled = oracle.sdp_solve(case["offsets"], case["init"], case["n"], case["op"])
        assert cells.tolist() == case["cells"], case
        assert filled.all()


def test_golden_sdp_digests(oracle):
    for case in GOLDEN["sdp"]:
        n, k, seed, cons, cap = case["gen"]
        offs, init = oracle.generate_sdp(n, k, seed, cons, cap)
        cells, _ = oracle.sdp_solve(offs, init, n, case["op"])
        assert hx(oracle.digest(cells)) == case["digest"], case
        assert int(cells[-1]) == case["last"]


def test_golden_sdp_validate(oracle):
    for case in GOLDEN["sdp_validate"]:
        assert oracle.sdp_validate(case["offsets"], case["init_len"], case["n"]) == case["status"], case


def test_golden_generators(oracle):
    for case in GOLDEN["gen_sdp"]:
        n, k, seed, cons, cap = case["args"]
        offs, init = oracle.generate_sdp(n, k, seed, cons, cap)
        assert hx(oracle.digest(offs)) == case["offsets_digest"]
        assert hx(oracle.digest(init)) == case["init_digest"]
        assert offs[-12:].tolist() == case["offsets_tail"] and int(offs[0]) == case["a1"]
    for case in GOLDEN["gen_mcm"]:
        n, seed, lo, hi = case["args"]
        dims = oracle.generate_mcm(n, seed, lo, hi)
        assert hx(oracle.digest(dims)) == case["digest"] and dims[:8].tolist() == case["head"]


def test_golden_lin_coord(oracle):
    for r, c, n, want in GOLDEN["lin"]:
        assert oracle.lin(r, c, n) == want
    for a, n, r, c in GOLDEN["coord"]:
        assert oracle.coord(a, n) == (r, c)


def test_golden_mcm(oracle):
    for case in GOLDEN["mcm"]:
        if "dims" in case:
            cells, filled, split = oracle.mcm_solve(case["dims"])
            assert cells.tolist() == case["cells"] and split.tolist() == case["split"]
            assert filled.all()
            continue
        n, seed, lo, hi = case["gen"]
        if n > 600:
            continue  # test_config3_digest
        dims = oracle.generate_mcm(n, seed, lo, hi)
        cells, _, split = oracle.mcm_solve(dims)
        assert hx(oracle.digest(cells)) == case["digest"], case
        assert hx(oracle.digest(split)) == case["split_digest"], case
        assert int(cells[-1]) == case["apex"] and int(split[-1]) == case["apex_split"]


def test_golden_mcm_validate(oracle):
    for case in GOLDEN["mcm_validate"]:
        dims = case["dims"] if case["dims"] is not None else [case["fill"]] * case["dims_len"]
        assert oracle.mcm_validate(dims) == case["status"], case


def test_golden_mcm_pipeline(oracle):
    for case in GOLDEN["mcm_pipeline"]:
        n, seed, lo, hi = case["gen"]
        dims = oracle.generate_mcm(n, seed, lo, hi)
        cells, _, steps, stall = oracle.mcm_pipeline(dims, case["mode"])
        assert hx(oracle.digest(cells)) == case["digest"], case
        assert (steps, stall) == (case["steps"], case["stall"]), case


def test_golden_config1(oracle):
    for op in ("saturating-add", "modular-add"):
        cells, _ = oracle.sdp_solve([2, 1], [1, 1], 1 << 20, op)
        want = GOLDEN["configs"][f"c1_{op}"]
        assert hx(oracle.digest(cells)) == want["digest"] and int(cells[-1]) == want["last"]


def test_golden_config3_digest(oracle):
    # BASELINE config 3 (MCM n=1024, dims U[1,100], seed 1): SURVEY.md 8c digests
    dims = oracle.generate_mcm(1024, 1, 1, 100)
    cells, _, split = oracle.mcm_solve(dims)
    assert hx(oracle.digest(cells)) == "9e31907a82260f66"
    assert hx(oracle.digest(split)) == "42bfd8baf652c2f3"


def test_golden_config2_prefix(oracle):
    # the first 2^22 cells of config 2 depend only on the first 2^22 cells
    offs, init = oracle.generate_sdp(1 << 24, 1024, 1, False, 4096)
    cells, _ = oracle.sdp_solve(offs, init, 1 << 22, "min")
    assert hx(oracle.digest(cells)) == GOLDEN["configs"]["c2_prefix22"]["digest"]


# --------------------------------------------------------- SPEC known answers --
def test_spec_sdp_kats(oracle):
    assert oracle.sdp_solve([2, 1], [1, 1], 7, "saturating-add")[0].tolist() == [1, 1, 2, 3, 5, 8, 13]
    assert oracle.sdp_solve([5, 3, 1], [0] * 5, 10, "min")[0].tolist() == [0] * 10


def test_spec_mcm_kats(oracle):
    # SPEC.md:298-299, 318-319, 328-330
    assert oracle.lin(1, 4, 5) == 13 and oracle.lin(3, 5, 5) == 12
    for dims, apex, sp in [([10, 20, 30], 6000, 1), ([30, 35, 15, 5, 10, 20, 25], 15125, 3),
                           ([2, 3, 4, 5], 64, 2)]:
        cells, _, split = oracle.mcm_solve(dims)
        assert cells[-1] == apex and split[-1] == sp
    for d in (1, 3, 17):  # all dims d -> (n-1) d^3
        for n in (2, 5, 9):
            assert oracle.mcm_solve([d] * (n + 1))[0][-1] == (n - 1) * d**3


def test_spec_mcm_pipeline_steps(oracle):
    # paper-literal steps = n(n+1)/2 - 2; stall mode adds floor((n-2)^2/4)
    for n in range(2, 20):
        dims = oracle.generate_mcm(n, n, 1, 50)
        _, _, steps, stall = oracle.mcm_pipeline(dims, 0)
        assert steps == n * (n + 1) // 2 - 2 and stall == 0
        c1, _, steps1, stall1 = oracle.mcm_pipeline(dims, 1)
        assert stall1 == (n - 2) ** 2 // 4
        assert np.array_equal(c1, oracle.mcm_solve(dims)[0])  # stall mode == oracle


def test_mcm_bruteforce_agrees(oracle):
    for n in range(1, 9):
        for seed in range(3):
            dims = oracle.generate_mcm(n, seed, 1, 30)
            assert oracle.mcm_bruteforce(dims) == oracle.mcm_solve(dims)[0][-1]


def test_sdp_pointwise_recurrence(oracle):
    # SPEC invariant "Eq. (1) pointwise", re-evaluated independently in Python
    offs, init = oracle.generate_sdp(300, 7, 4, False, 0)
    for op in OPS:
        cells, _ = oracle.sdp_solve(offs, init, 300, op)
        for i in range(int(offs[0]), 300):
            acc = int(cells[i - offs[0]])
            for a in offs[1:]:
                acc = oracle.apply(op, acc, int(cells[i - a]))
            assert acc == cells[i]


# ---------------------------------------------------- the reference, directly --
def test_ref_sweep_sdp(oracle, ref):
    # SPEC acceptance #1: 200-instance sweep, all ops
    rng = np.random.default_rng(7)
    for case in range(200):
        op = OPS[case % 4]
        k = int(rng.integers(1, 65))
        offs, init = oracle.generate_sdp(int(rng.integers(2 * k + 1, 4097)), k, case, bool(case % 5 == 0), 0)
        n = int(offs[0]) + int(rng.integers(1, 3000))
        if case % 3 == 0:
            init = rng.integers(-(2**62), 2**62, len(init))
        a, _ = oracle.sdp_solve(offs, init, n, op)
        b, _ = ref.sdp_solve(offs, init, n, op)
        assert np.array_equal(a, b), case


def test_ref_sweep_mcm(oracle, ref):
    for n in list(range(1, 70)) + [128, 200]:
        dims = oracle.generate_mcm(n, n * 3, 1, 100)
        a = oracle.mcm_solve(dims)
        b = ref.mcm_solve(dims)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2]), n


def test_ref_generators(oracle, ref):
    for seed in range(40):
        for k, cap in [(4, 0), (64, 0), (300, 1000), (1024, 4096)]:
            a = oracle.generate_sdp(cap * 2 + 10 if cap else 4 * k + 10, k, seed, seed % 7 == 0, cap)
            b = ref.generate_sdp(cap * 2 + 10 if cap else 4 * k + 10, k, seed, seed % 7 == 0, cap)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(oracle.generate_mcm(50, seed, 1, 100), ref.generate_mcm(50, seed, 1, 100))


def test_ref_mcm_pipeline(oracle, ref):
    for n in (2, 3, 4, 6, 9, 16, 24):
        dims = oracle.generate_mcm(n, 7 * n, 1, 50)
        for mode in (0, 1):
            a = oracle.mcm_pipeline(dims, mode)
            b = ref.mcm_pipeline(dims, mode)
            assert np.array_equal(a[0], b[0]) and a[2:] == b[2:4], (n, mode)


def test_ref_apply_random(oracle, ref):
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.integers(-(2**63), 2**63 - 1, 300, dtype=np.int64),
                         rng.integers(-100, 100, 100)])
    for op in OPS:
        for a, b in zip(xs, np.roll(xs, 17)):
            assert oracle.apply(op, int(a), int(b)) == ref.apply(op, int(a), int(b))


def test_c5_golden_digest_lists(oracle):
    # tests/golden/c5*.npy (all 65,536 instances, written by the reference via
    # make_c5_digests.py) agree with the C restatement on a spread sample
    import os
    here = os.path.join(os.path.dirname(__file__), "golden")
    c5a_c = np.load(os.path.join(here, "c5a_cells.npy"))
    c5a_s = np.load(os.path.join(here, "c5a_split.npy"))
    c5b = np.load(os.path.join(here, "c5b_cells.npy"))
    assert c5a_c.shape == c5a_s.shape == c5b.shape == (65536,) and c5b.dtype == np.uint64
    for i in (0, 1, 2, 777, 40000, 65535):
        c, _, s = oracle.mcm_solve(oracle.generate_mcm(64, i, 1, 100))
        assert oracle.digest(c) == int(c5a_c[i]) and oracle.digest(s) == int(c5a_s[i])
    for i in (0, 9, 65535):
        offs, init = oracle.generate_sdp(1 << 16, 64, i, False, 0)
        assert oracle.digest(oracle.sdp_solve(offs, init, 1 << 16, "min")[0]) == int(c5b[i])
