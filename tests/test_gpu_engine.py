"""The GPU lock-step engine (csrc/engine_kernels.cuh, C ABI pipedp_*_engine)
against the reference's own engine: solve_mcm_pipeline / solve_sdp_pipeline
with their default collect_trace = true, compared by the digest vector of
tests/golden/engine_golden.json (generated from oracle/_ref by
tests/golden/make_engine_golden.py):  table, steps, stalls, stall heads, every
access record in canonical order (engine.hpp:61-76), the conflict report of
detect_conflicts (analysis.cpp:31-70, incl. per_step_cost) and the hazard
report of detect_hazards (analysis.cpp:72-103).  Beyond the reference's
reach: the paper-literal hazard frontier on the multi-CTA engine at n = 1024
checked against hazard_frontier (mcm_pipeline.cpp:79-94)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "engine_golden.json")))
MODES = ["paper_literal", "stall_on_hazard"]


def _digests(oracle, table, trace, conflicts, hazards):
    D = oracle.digest
    r = trace.records
    rec = np.stack([r["head"], r["substep"].astype(np.int64), r["lane"].astype(np.int64),
                    r["kind"].astype(np.int64), r["address"]], axis=1).ravel() if len(r) else np.zeros(0, np.int64)
    grp = []
    for g in conflicts.groups:
        grp += [g.head, g.substep, g.kind, g.address, len(g.lanes), *g.lanes]
    hz = hazards.hazards.view(np.int64).ravel() if hazards is not None and len(hazards.hazards) else np.zeros(0, np.int64)
    return [trace.steps_executed, trace.stall_iterations, trace.first_head, len(r), D(rec),
            conflicts.max_group_size, len(conflicts.groups), D(np.array(grp, np.int64)),
            D(conflicts.per_step_cost.astype(np.int64)), 0 if hazards is None else len(hazards.hazards), D(hz),
            len(trace.stall_heads), D(trace.stall_heads), D(table.cells)]


def _hex(v):
    return [f"{x & (2**64 - 1):016x}" for x in v]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["mcm"], ids=lambda c: f"n{c['gen'][0]}-m{c['mode']}")
def test_mcm_engine_matches_reference(gpu, oracle, case):
    n, seed, lo, hi = case["gen"]
    dims = oracle.generate_mcm(n, seed, lo, hi)
    r = gpu.solve_mcm_pipeline(gpu.McmInstance(dims), MODES[case["mode"]])
    assert r.trace.collected
    assert _hex(_digests(oracle, r.table, r.trace, r.conflicts, r.hazards)) == case["digests"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["sdp"], ids=lambda c: f"n{c['gen'][0]}-k{c['gen'][1]}-{c['op']}")
def test_sdp_engine_matches_reference(gpu, oracle, case):
    n, k, seed, cons, cap = case["gen"]
    inst = gpu.generate_sdp(n=n, k=k, op=case["op"], seed=seed, consecutive=cons, a1_cap=cap)
    r = gpu.solve_sdp_pipeline(inst)
    d = _digests(oracle, r.table, r.trace, r.conflicts, None)
    assert _hex(d) == case["digests"]
    # the paper's pipeline table equals the sequential oracle (hazard-free schedule)
    want, _ = oracle.sdp_solve(inst.offsets, inst.init, n, case["op"])
    assert np.array_equal(r.table.cells, want)


@pytest.mark.gpu
def test_sdp_engine_fibonacci(gpu, oracle):
    inst = gpu.SdpInstance(GOLD["fib"]["n"], [2, 1], [1, 1], "saturating-add")
    r = gpu.solve_sdp_pipeline(inst)
    assert _hex(_digests(oracle, r.table, r.trace, r.conflicts, None)) == GOLD["fib"]["digests"]


@pytest.mark.gpu
def test_collect_trace_off_keeps_counts(gpu, oracle):
    dims = oracle.generate_mcm(40, 8, 1, 100)
    for mode in MODES:
        a = gpu.solve_mcm_pipeline(gpu.McmInstance(dims), mode)
        b = gpu.solve_mcm_pipeline(gpu.McmInstance(dims), mode, collect_trace=False)
        assert not b.trace.collected and len(b.trace.records) == 0 and b.hazards.empty()
        assert np.array_equal(a.table.cells, b.table.cells)
        assert (a.trace.steps_executed, a.trace.stall_iterations) == (b.trace.steps_executed, b.trace.stall_iterations)
        assert np.array_equal(a.trace.stall_heads, b.trace.stall_heads)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [300, 1024])
def test_paper_literal_frontier_multi_cta(gpu, oracle, n):
    """n = 1024: 1023 lanes over two cooperative CTAs, 524,798 iterations; the
    trace (7e8 records) exceeds the trace limit, the device analyses do not."""
    dims = oracle.generate_mcm(n, 3, 1, 100)
    r = gpu.solve_mcm_pipeline(gpu.McmInstance(dims), "paper_literal")
    assert r.trace.steps_executed == n * (n + 1) // 2 - 2
    assert r.trace.collected == (n == 300)
    h = r.hazards.hazards
    cells = np.unique(h["head"] - h["lane"] + 1)  # hazard_cells (mcm_pipeline.cpp:96-103)
    assert np.array_equal(cells, np.asarray(gpu.hazard_frontier(n), np.int64))
    assert r.conflicts.max_group_size == 1 and not r.conflicts.groups  # Lemmas 1/2
    assert np.all(h["finalization_substep"] == 4)
    assert np.all((h["head"] < h["finalization_head"]) | ((h["head"] == h["finalization_head"]) & (h["substep"] <= 4)))


@pytest.mark.gpu
def test_stall_mode_multi_cta_equals_oracle(gpu, oracle):
    n = 1100
    dims = oracle.generate_mcm(n, 4, 1, 100)
    r = gpu.solve_mcm_pipeline(gpu.McmInstance(dims), "stall_on_hazard")
    wc, _, _ = oracle.mcm_solve(dims, with_split=False)
    assert np.array_equal(r.table.cells, wc)
    assert r.hazards.empty() and r.conflicts.max_group_size == 1
    heads = n * (n + 1) // 2 - 2
    assert r.trace.steps_executed == heads + r.trace.stall_iterations
    assert r.trace.stall_iterations == (n - 2) ** 2 // 4  # SURVEY 8a probe: floor((n-2)^2/4)
    assert len(r.trace.stall_heads) > 0
