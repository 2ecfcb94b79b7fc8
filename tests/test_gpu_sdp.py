"""S-DP parity on the GPU: every table bit-exact against the C restatement of
the reference (oracle/pipedp_oracle.c, pinned to the reference by
test_oracle.py), through the C ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OPS = ["min", "max", "saturating-add", "modular-add"]


def _check(gpu, oracle, offs, init, n, op):
    inst = gpu.SdpInstance(n, offs, init, op)
    t = gpu.solve_sequential(inst)
    want, wfilled = oracle.sdp_solve(offs, init, n, op)
    bad = np.nonzero(t.cells != want)[0]
    assert bad.size == 0, f"first mismatch at {bad[:5]}: got {t.cells[bad[:5]]} want {want[bad[:5]]}"
    assert np.array_equal(t.filled, wfilled)


def test_fibonacci_kat(gpu):
    # k=2, a=(2,1), add, init [1,1], n=7
    t = gpu.solve_sequential(gpu.SdpInstance(7, [2, 1], [1, 1], "saturating-add"))
    assert t.cells.tolist() == [1, 1, 2, 3, 5, 8, 13]
    assert t.all_filled()


def test_min_zeros_kat(gpu):
    # (5,3,1), min, zeros, n=10
    t = gpu.solve_sequential(gpu.SdpInstance(10, [5, 3, 1], [0] * 5, "min"))
    assert t.cells.tolist() == [0] * 10


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("seed", range(12))
def test_random_small(gpu, oracle, op, seed):
    rng = np.random.default_rng(seed * 7 + OPS.index(op))
    k = int(rng.integers(1, 40))
    cap = int(rng.integers(k, 200))
    offs = np.sort(rng.choice(np.arange(1, cap + 1), k, replace=False))[::-1].copy()
    n = int(offs[0] + rng.integers(1, 3000))
    if seed % 3 == 0:
        init = rng.integers(-(2**62), 2**62, offs[0])
    elif seed % 3 == 1:
        init = rng.integers(-1000, 1000, offs[0])
    else:
        init = rng.integers(0, 2**20, offs[0])
    _check(gpu, oracle, offs, init, n, op)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("shape", [(4096, 64, 0), (20000, 1024, 4096), (9000, 300, 700),
                                   (5000, 32, 0), (3000, 7, 0), (70000, 2000, 20000)])
def test_generated(gpu, oracle, op, shape):
    n, k, cap = shape
    offs, init = oracle.generate_sdp(n, k, 11, False, cap)
    _check(gpu, oracle, offs, init, n, op)


@pytest.mark.parametrize("op", OPS)
def test_consecutive_offsets(gpu, oracle, op):
    offs, init = oracle.generate_sdp(6000, 200, 3, True, 0)
    _check(gpu, oracle, offs, init, 6000, op)


def test_sat_add_mixed_signs_strict_order(gpu, oracle):
    # saturating-add is not associative with mixed signs: the kernels must keep
    # the reference's j-ascending fold (sdp.cpp:53-56)
    rng = np.random.default_rng(5)
    offs = np.array(sorted(rng.choice(np.arange(1, 600), 120, replace=False))[::-1])
    init = rng.choice([2**62, -(2**62), 2**61, -(2**61), 3, -3], offs[0])
    _check(gpu, oracle, offs, init, 8000, "saturating-add")


def test_modadd_raw_copy_k1(gpu, oracle):
    # k=1 copies raw (unnormalised) values (SURVEY hard part 5)
    _check(gpu, oracle, [3], [-5, 3000000000, 7], 50, "modular-add")


def test_large_a1_hbm_far_stage(gpu, oracle):
    # a_1 too large for a shared-memory ring -> far stage reads HBM
    offs, init = oracle.generate_sdp(120000, 700, 2, False, 60000)
    _check(gpu, oracle, offs, init, 120000, "min")
    _check(gpu, oracle, offs, init, 120000, "saturating-add")


def test_fibonacci_config1(gpu, oracle):
    # BASELINE config 1 (and its modular-add companion)
    n = 1 << 20
    for op in ("saturating-add", "modular-add"):
        _check(gpu, oracle, [2, 1], [1, 1], n, op)


@pytest.mark.parametrize("op", OPS)
def test_batch_matches_single(gpu, oracle, op):
    insts = []
    for i in range(37):
        offs, init = oracle.generate_sdp(3000, 64, i, False, 0)
        insts.append(gpu.SdpInstance(3000, offs, init, op))
    tabs = gpu.solve_sequential_batch(insts)
    for inst, t in zip(insts, tabs):
        want, _ = oracle.sdp_solve(inst.offsets, inst.init, inst.n, op)
        assert np.array_equal(t.cells, want)


def test_batch_large_a1_uses_cta_kernel(gpu, oracle):
    insts = []
    for i in range(5):
        offs, init = oracle.generate_sdp(30000, 256, 100 + i, False, 4096)
        insts.append(gpu.SdpInstance(30000, offs, init, "min"))
    for inst, t in zip(insts, gpu.solve_sequential_batch(insts)):
        want, _ = oracle.sdp_solve(inst.offsets, inst.init, inst.n, "min")
        assert np.array_equal(t.cells, want)


def test_pipeline_trace_fields(gpu):
    inst = gpu.generate_sdp(n=4096, k=64, seed=1)
    r = gpu.solve_sdp_pipeline(inst)
    assert r.trace.first_head == inst.a1
    assert r.trace.steps_executed == inst.n + inst.k - inst.a1 - 1
    assert r.trace.stall_iterations == 0


def test_large_a1_mixed_signs_hbm_far(gpu, oracle):
    # non-associative (mixed-sign saturating-add) + a_1 too large for the ring:
    # single CTA, strict order, far stage reading the HBM table
    rng = np.random.default_rng(9)
    offs, _ = oracle.generate_sdp(90000, 300, 4, False, 50000)
    init = rng.choice([2**62, -(2**62), 5, -7], offs[0])
    _check(gpu, oracle, offs, init, 90000, "saturating-add")


@pytest.mark.parametrize("op", ["min", "modular-add"])
def test_single_cta_path_when_multi_disabled(gpu, oracle, op, monkeypatch):
    monkeypatch.setenv("PIPEDP_SDP_MULTI", "0")
    offs, init = oracle.generate_sdp(40000, 1024, 21, False, 4096)
    _check(gpu, oracle, offs, init, 40000, op)


@pytest.mark.parametrize("ctas,warps", [(1, 1), (3, 4), (64, 8)])
def test_multi_cta_shapes(gpu, oracle, ctas, warps, monkeypatch):
    monkeypatch.setenv("PIPEDP_SDP_REMOTE_CTAS", str(ctas))
    monkeypatch.setenv("PIPEDP_SDP_REMOTE_WARPS", str(warps))
    offs, init = oracle.generate_sdp(60000, 1500, 8, False, 6000)
    _check(gpu, oracle, offs, init, 60000, "max")


@pytest.mark.parametrize("op", OPS)
def test_k1_large_a1_raw_copy(gpu, oracle, op):
    # k = 1 with a_1 >= 64: the table is a raw periodic copy of init for every op
    rng = np.random.default_rng(3)
    init = rng.integers(-(2**62), 2**62, 100)
    _check(gpu, oracle, [100], init, 1000, op)


@pytest.mark.parametrize("op", OPS)
def test_all_offsets_below_64_with_large_one(gpu, oracle, op):
    # a_1 >= 64 but every other offset < 64: empty mid range, chain does the rest
    offs = [200, 63, 40, 33, 32, 31, 17, 2, 1]
    rng = np.random.default_rng(4)
    init = rng.integers(0, 2**20, 200) if op != "saturating-add" else rng.integers(0, 5, 200)
    _check(gpu, oracle, offs, init, 7000, op)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("shape", [(300, 5, 0), (3000, 64, 0), (9000, 300, 700), (5000, 1500, 4096)])
def test_paper_methods_prefix_and_naive(gpu, oracle, op, shape):
    # solve_prefix_parallel / solve_naive_parallel run the paper's tournament and
    # naive methods on the device (sdp.cpp:91-111: same table as the oracle)
    n, k, cap = shape
    offs, init = oracle.generate_sdp(n, k, 17, False, cap)
    want, _ = oracle.sdp_solve(offs, init, n, op)
    inst = gpu.SdpInstance(n, offs, init, op)
    p = gpu.solve_prefix_parallel(inst)
    assert np.array_equal(p.table.cells, want) and p.depth_per_cell == (k - 1).bit_length()
    q = gpu.solve_naive_parallel(inst)
    assert np.array_equal(q.table.cells, want) and q.serialized_accesses_per_cell == k - 1


def test_paper_methods_mixed_sign_sat_add(gpu, oracle):
    # non-associative: the strict pipeline is kept (reference table)
    rng = np.random.default_rng(2)
    offs, _ = oracle.generate_sdp(4000, 40, 3, False, 0)
    init = rng.choice([2**62, -(2**62), 3, -5], offs[0])
    want, _ = oracle.sdp_solve(offs, init, 4000, "saturating-add")
    inst = gpu.SdpInstance(4000, offs, init, "saturating-add")
    assert np.array_equal(gpu.solve_prefix_parallel(inst).table.cells, want)
    assert np.array_equal(gpu.solve_naive_parallel(inst).table.cells, want)


@pytest.mark.parametrize("op,writers", [("min", "1"), ("modular-add", "2")])
def test_streamed_copy_out_while_kernel_runs(gpu, oracle, op, writers, monkeypatch):
    # >= 64 MiB single-instance multi-CTA solve: the host-buffer entry point
    # copies finished 16 MiB chunks out while the kernel is still producing the
    # tail (progress from the writers' published counters, min over writers)
    monkeypatch.setenv("PIPEDP_SDP2_WRITERS", writers)
    n = 9_000_000 + 777
    offs, init = oracle.generate_sdp(n, 256, 5, False, 4096)
    _check(gpu, oracle, offs, init, n, op)


def test_cached_plan_reuse_with_new_init_and_op(gpu, oracle):
    # the host-buffer entry point keeps its last plan: same offsets with new
    # init values (same value class), then another value class, then another op
    n = 50000
    offs, init = oracle.generate_sdp(n, 500, 3, False, 3000)
    rng = np.random.default_rng(5)
    for op, lo, hi in [("min", -1000, 1000), ("min", -1000, 1000), ("min", -(2**60), 2**60),
                       ("max", 0, 100), ("modular-add", 0, 2**31 - 1)]:
        _check(gpu, oracle, offs, rng.integers(lo, hi, len(init)), n, op)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("seed", range(6))
def test_jump_segments_small_a1(gpu, oracle, op, seed):
    # a_1 <= 8, k >= 2: jump-ahead segments (sdp_jump); sat-add takes the jump
    # path only with non-negative presets (otherwise the serial kernel)
    rng = np.random.default_rng(100 + seed * 4 + OPS.index(op))
    a1 = int(rng.integers(2, 9))
    k = int(rng.integers(2, a1 + 1))
    offs = np.sort(rng.choice(np.arange(1, a1), k - 1, replace=False))[::-1] if k > 1 else []
    offs = np.concatenate([[a1], offs]).astype(np.int64)
    n = int(rng.integers(4200, 60000))
    if op == "saturating-add":
        init = rng.integers(0, 2**40, a1) if seed % 2 == 0 else rng.integers(0, 3, a1)
    elif op == "modular-add":
        init = rng.integers(-(2**40), 2**40, a1)
    else:
        init = rng.integers(-(2**62), 2**62, a1)
    inst = gpu.SdpInstance(n, offs, init, op)
    plan = gpu.SdpPlan(1, n, len(offs), a1, offs, init, op)
    assert plan.describe()[0] == "sdp_jump"
    plan.close()
    _check(gpu, oracle, offs, init, n, op)


def test_jump_fibonacci_saturates_like_reference(gpu, oracle):
    # the C1 shape: clamped counts in the jump matrices, INT64_MAX tail
    _check(gpu, oracle, [2, 1], [1, 1], 300000, "saturating-add")
    _check(gpu, oracle, [3, 2], [0, 5, 7], 100000, "saturating-add")


@pytest.mark.parametrize("op", ["min", "max"])
@pytest.mark.parametrize("shape", [(70000, 20, 64), (66000, 150, 300), (140000, 400, 1000), (560000, 1024, 4096)])
def test_chunked_min_max(gpu, oracle, op, shape):
    # one large min/max instance as a batch of chunks with entry states from
    # boolean matrix powers (sdp_chunked.cuh); ragged last chunk
    n, k, cap = shape
    offs, init = oracle.generate_sdp(n + 777, k, 31, False, cap)
    n = n + 777
    plan = gpu.SdpPlan(1, n, len(offs), len(init), offs, init, op)
    assert plan.describe()[0].startswith("sdp_chunked")
    plan.close()
    _check(gpu, oracle, offs, init, n, op)


@pytest.mark.parametrize("op", ["min", "max"])
def test_chunked_periodic_reachability(gpu, oracle, op):
    # even offsets only (gcd 2): the matrix powers stay periodic, half the
    # preset cells are unreachable from each cell
    rng = np.random.default_rng(9)
    a1 = 512
    offs = np.array([512] + sorted(rng.choice(np.arange(2, 511, 2), 40, replace=False).tolist(), reverse=True))
    init = rng.integers(-(2**40), 2**40, a1)
    n = 16 * 4096 + a1 + 1234
    plan = gpu.SdpPlan(1, n, len(offs), a1, offs, init, op)
    assert plan.describe()[0].startswith("sdp_chunked")
    plan.close()
    _check(gpu, oracle, offs, init, n, op)


@pytest.mark.parametrize("a1,k,op", [(7000, 300, "min"), (8192, 1500, "max")])
def test_chunked_wide_state(gpu, oracle, a1, k, op):
    # a_1 > 4096: 128-word matrix rows (the padded 8192-bit state)
    n = 16 * 65536 + a1 + 4321
    offs, init = oracle.generate_sdp(n, k, 5, False, a1)
    assert offs[0] == a1
    plan = gpu.SdpPlan(1, n, len(offs), len(init), offs, init, op)
    assert plan.describe()[0].startswith("sdp_chunked")
    plan.close()
    _check(gpu, oracle, offs, init, n, op)


def test_chunked_equals_pipeline(gpu, monkeypatch):
    # the same instance through the chunked mode and the pipeline-only path
    inst = gpu.generate_sdp(n=1_200_000, k=512, op="min", seed=4, a1_cap=4096)
    a = gpu.solve_sequential(inst).cells
    monkeypatch.setenv("PIPEDP_SDP_CHUNKED", "0")
    b = gpu.solve_sequential(inst).cells
    assert np.array_equal(a, b)


def test_chunked_large_table_host_copy(gpu, oracle):
    # >= 64 MiB output through the host-buffer entry point of a chunked plan
    # (whose copy-out must not take the pipeline's progress-polling path)
    n = 9_000_000 + 17
    offs, init = oracle.generate_sdp(n, 20, 8, False, 64)
    _check(gpu, oracle, offs, init, n, "max")


@pytest.mark.parametrize("op", ["min", "max"])
def test_chunked_overlapped_copy_out(gpu, oracle, op, monkeypatch):
    # G = 200 > SM count: chunks run in two launches and the first range is
    # copied out (narrowed to int32, widened on the host) while the second runs
    monkeypatch.setenv("PIPEDP_CHUNK_OVERLAP", "1")
    n = 200 * 16384 + 512 + 99
    offs, init = oracle.generate_sdp(n, 50, 12, False, 512)
    _check(gpu, oracle, offs, init, n, op)


@pytest.mark.parametrize("op", ["min", "max"])
@pytest.mark.parametrize("progressive", ["1", "0"])
def test_rank_progressive_copy_out(gpu, oracle, op, progressive, monkeypatch):
    # rank-compressed chunks through the host-buffer call: with progressive
    # copy-out the chunks publish their progress into mapped host memory and
    # the finished column band of all chunks is copied and converted while they
    # run (ragged last chunk); without it, one copy after the launch
    monkeypatch.setenv("PIPEDP_D2H_PROGRESSIVE", progressive)
    n = 3_000_000 + 12_345
    offs, init = oracle.generate_sdp(n, 300, 21, False, 2048)
    plan = gpu.SdpPlan(1, n, len(offs), len(init), offs, init, op)
    name = plan.describe()[0]
    plan.close()
    assert "chunk_rank_kernel" in name
    for _ in range(2):  # a second call: the progress words carry the previous epoch
        _check(gpu, oracle, offs, init, n, op)


@pytest.mark.parametrize("op", ["min", "max"])
def test_chunked_int64_values(gpu, oracle, op):
    # presets beyond int32: 64-bit chunk kernels, entry states and a full-width copy-out
    rng = np.random.default_rng(77)
    n = 2_500_000
    offs, _ = oracle.generate_sdp(n, 40, 9, False, 300)
    init = rng.integers(-(2**62), 2**62, len(_))
    plan = gpu.SdpPlan(1, n, len(offs), len(init), offs, init, op)
    name, bits, _l = plan.describe()
    plan.close()
    assert name.startswith("sdp_chunked") and bits == 64
    _check(gpu, oracle, offs, init, n, op)


def test_config2_full_table_digest(gpu):
    # BASELINE config 2 at full size (n = 2^24, k = 1024, a_1 = 4096, min,
    # seed 1): the whole 128 MiB table against the reference's table_digest,
    # through the drop-in call (host buffers) and the device-resident plan
    import json
    import os
    import torch
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["configs"]["c2"]
    inst = gpu.generate_sdp(n=1 << 24, k=1024, op="min", seed=1, a1_cap=4096)
    t = gpu.solve_sequential(inst)
    assert f"{gpu.table_digest(t.cells):016x}" == g["digest"] and int(t.cells[-1]) == g["last"]
    plan = gpu.SdpPlan(1, inst.n, inst.k, inst.a1, inst.offsets, inst.init, inst.op, 0)
    d_init = torch.tensor(inst.init, dtype=torch.int64, device="cuda")
    d_cells = torch.empty(inst.n, dtype=torch.int64, device="cuda")
    for _ in range(2):  # plan reuse
        d_cells.fill_(-1)
        plan.execute(d_init.data_ptr(), d_cells.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert f"{gpu.table_digest(d_cells.cpu().numpy()):016x}" == g["digest"]


@pytest.mark.parametrize("op,n,k,cap", [("min", 100003, 1024, 4096), ("max", 70001, 700, 12000),
                                        ("modular-add", 50017, 2000, 8000), ("min", 29103, 7168, 14336)])
def test_cluster_pipeline(gpu, oracle, op, n, k, cap):
    """sdp_cluster_kernel: one instance over a 16-CTA cluster, the far offsets
    folded by producer CTAs from rings fed through DSMEM (st.async with
    mbarrier transaction bytes).  Forced by disabling the chunked mode."""
    import os
    inst = gpu.generate_sdp(n=n, k=k, op=op, seed=n % 97, a1_cap=cap)
    old = os.environ.get("PIPEDP_SDP_CHUNKED")
    os.environ["PIPEDP_SDP_CHUNKED"] = "0"
    try:
        plan = gpu.SdpPlan(1, n, inst.k, inst.a1, inst.offsets, inst.init, op, device=0)
        assert plan.describe()[0] == "sdp_cluster_kernel"
        plan.close()
        t = gpu.solve_sequential(inst)
    finally:
        if old is None:
            del os.environ["PIPEDP_SDP_CHUNKED"]
        else:
            os.environ["PIPEDP_SDP_CHUNKED"] = old
    want, _ = oracle.sdp_solve(inst.offsets, inst.init, n, op)
    assert np.array_equal(t.cells, want)


@pytest.mark.parametrize("shape", [
    ("chunked rank", 3_000_000 + 77, 300, 21, 2048, "min", {}),
    ("cluster", 300_000 + 5, 400, 22, 4096, "max", {"PIPEDP_SDP_CHUNKED": "0"}),
    ("jump", 200_000, 3, 23, 6, "saturating-add", {}),
    ("v2 mod-add", 150_000, 200, 24, 1500, "modular-add", {"PIPEDP_SDP_CLUSTER": "0"}),
])
def test_plan_execute_is_graph_capturable(gpu, oracle, shape, monkeypatch):
    # the device plans are asynchronous: a whole execute (matrix powers, the
    # cooperative entry-state chain, the chunk batch / the cluster pipeline /
    # jump segments) replays from a CUDA graph with the same table
    import torch
    _, n, k, seed, cap, op, env = shape
    for key, v in env.items():
        monkeypatch.setenv(key, v)
    offs, init = oracle.generate_sdp(n, k, seed, False, cap)
    if op == "saturating-add":
        init = np.abs(init) % 1000
    want, _ = oracle.sdp_solve(offs, init, n, op)
    plan = gpu.SdpPlan(1, n, len(offs), len(init), offs, init, op)
    d_init = torch.from_numpy(np.asarray(init, np.int64)).cuda()
    out = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.execute(d_init.data_ptr(), out.data_ptr(), st.cuda_stream)  # warm-up
    torch.cuda.synchronize()
    out.fill_(-1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        plan.execute(d_init.data_ptr(), out.data_ptr(), st.cuda_stream)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)
        out.fill_(-1)
    plan.close()
