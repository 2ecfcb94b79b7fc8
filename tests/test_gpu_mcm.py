"""MCM parity on the GPU: cells AND split tables bit-exact against the C
restatement of solve_mcm_sequential, lock-step pipeline tables / step counts
against the restated engine."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(gpu, oracle, dims, kernel):
    t, split = gpu.solve_mcm_with_split(gpu.McmInstance(dims), kernel)
    wc, wf, ws = oracle.mcm_solve(dims)
    assert np.array_equal(t.cells, wc), np.nonzero(t.cells != wc)[0][:5]
    assert np.array_equal(split, ws), np.nonzero(split != ws)[0][:5]
    assert np.array_equal(t.filled, wf)


def test_spec_apex_kats(gpu):
    # SPEC.md:328-330
    for dims, apex, sp in [([10, 20, 30], 6000, 1), ([30, 35, 15, 5, 10, 20, 25], 15125, 3),
                           ([2, 3, 4, 5], 64, 2)]:
        t, split = gpu.solve_mcm_with_split(gpu.McmInstance(dims))
        assert t.cells[-1] == apex and split[-1] == sp


@pytest.mark.parametrize("kernel", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 16, 33, 64, 100])
def test_small(gpu, oracle, kernel, n):
    _check(gpu, oracle, oracle.generate_mcm(n, n, 1, 100), kernel)


@pytest.mark.parametrize("kernel", [0, 1, 3, 4])
@pytest.mark.parametrize("n", [129, 200, 257, 511])
def test_medium(gpu, oracle, kernel, n):
    _check(gpu, oracle, oracle.generate_mcm(n, 3, 1, 100), kernel)


def test_ties_first_min(gpu, oracle):
    # all-equal dims produce massive ties: split must be the FIRST minimal j
    for n in (5, 40, 300):
        _check(gpu, oracle, [7] * (n + 1), 0)
        _check(gpu, oracle, [7] * (n + 1), 1)
    for n in (65, 200, 300):
        _check(gpu, oracle, [7] * (n + 1), 4)
        _check(gpu, oracle, [1] * (n + 1), 4)


@pytest.mark.parametrize("t32_maxn", ["0", "100000"])  # tile edge 64 / 32
@pytest.mark.parametrize("n", [2, 3, 31, 32, 33, 63, 64, 65, 127, 128, 130, 191, 192, 320, 700])
def test_tiled_shapes(gpu, oracle, n, t32_maxn, monkeypatch):
    # exact multiples of the tile edge, one-past and ragged last tiles, 1..22 tiles per side
    monkeypatch.setenv("PIPEDP_MCM_T32_MAXN", t32_maxn)
    _check(gpu, oracle, oracle.generate_mcm(n, 17 + n, 1, 100), 4)


def test_tiled_wide_dims_and_overflow(gpu, oracle):
    _check(gpu, oracle, oracle.generate_mcm(260, 5, 1, 1290), 4)    # 32-bit, large values
    _check(gpu, oracle, oracle.generate_mcm(300, 9, 1000, 1290), 4)  # reaches 2^30 -> exact int64 rerun
    _check(gpu, oracle, oracle.generate_mcm(200, 2, 1, 100000), 4)   # max_dim^3 >= 2^31 -> int64 path


def test_int32_overflow_falls_back_to_int64(gpu, oracle):
    # dims near 1290 drive values past 2^30: the 32-bit kernel must flag and
    # the 64-bit kernel rerun (still on the GPU)
    dims = oracle.generate_mcm(300, 9, 1000, 1290)
    _check(gpu, oracle, dims, 1)
    _check(gpu, oracle, dims[:60], 2)


def test_wide_dims_int64(gpu, oracle):
    dims = oracle.generate_mcm(150, 4, 1, 100000)
    _check(gpu, oracle, dims, 1)
    _check(gpu, oracle, dims[:80], 2)


@pytest.mark.parametrize("kernel", [0, 1, 4])
@pytest.mark.parametrize("t32_maxn", ["0", "100000"])
def test_config3_n1024(gpu, oracle, kernel, t32_maxn, monkeypatch):
    monkeypatch.setenv("PIPEDP_MCM_T32_MAXN", t32_maxn)
    dims = oracle.generate_mcm(1024, 1, 1, 100)
    t, split = gpu.solve_mcm_with_split(gpu.McmInstance(dims), kernel)
    assert gpu.digest_hex(gpu.table_digest(t.cells)) == "9e31907a82260f66"
    assert gpu.digest_hex(gpu.table_digest(split)) == "42bfd8baf652c2f3"


def test_config4_n8192_digest(gpu):
    # BASELINE config 4: digests from SURVEY 8c (the reference took 48 min on one core)
    dims = gpu.generate_mcm(n=8192, seed=1, dims_min=1, dims_max=100).dims
    t, split = gpu.solve_mcm_with_split(gpu.McmInstance(dims))
    assert gpu.digest_hex(gpu.table_digest(t.cells)) == "cc41fd2d4975b51b"
    assert gpu.digest_hex(gpu.table_digest(split)) == "f9e2c86f904b28e1"
    assert t.cells[-1] == 21215156


@pytest.mark.parametrize("mode", ["paper_literal", "stall_on_hazard"])
@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 17, 32, 64])
def test_lockstep_pipeline(gpu, oracle, mode, n):
    dims = oracle.generate_mcm(n, n + 100, 1, 50)
    r = gpu.solve_mcm_pipeline(gpu.McmInstance(dims), mode)
    wc, wf, steps, stall = oracle.mcm_pipeline(dims, 0 if mode == "paper_literal" else 1)
    assert np.array_equal(r.table.cells, wc)
    assert r.trace.steps_executed == steps and r.trace.stall_iterations == stall


def test_batch(gpu, oracle):
    insts = [gpu.McmInstance(oracle.generate_mcm(64, i, 1, 100)) for i in range(50)]
    for inst, (t, split) in zip(insts, gpu.solve_mcm_batch(insts)):
        wc, _, ws = oracle.mcm_solve(inst.dims)
        assert np.array_equal(t.cells, wc) and np.array_equal(split, ws)


@pytest.mark.parametrize("t32_maxn", ["0", "100000"])
@pytest.mark.parametrize("n", [33, 64, 130, 300])
def test_tiled_blocked_variant(gpu, oracle, n, t32_maxn, monkeypatch):
    # the 8x8 sub-blocked in-tile pipeline (PIPEDP_MCM_BLOCKED=1) gives the same tables
    monkeypatch.setenv("PIPEDP_MCM_T32_MAXN", t32_maxn)
    monkeypatch.setenv("PIPEDP_MCM_BLOCKED", "1")
    _check(gpu, oracle, oracle.generate_mcm(n, 5 + n, 1, 100), 4)
    _check(gpu, oracle, [7] * (n + 1), 4)


@pytest.mark.parametrize("t32_maxn", ["0", "100000"])
def test_tiled_packed_far_keys_fallback(gpu, oracle, t32_maxn, monkeypatch):
    # dims <= 322 enable packed far keys (64-wide tiles); cells past 2^25 (but
    # below 2^30) must trigger the unpacked 32-bit rerun, not a wrong table
    monkeypatch.setenv("PIPEDP_MCM_T32_MAXN", t32_maxn)
    dims = oracle.generate_mcm(300, 7, 100, 200)
    _check(gpu, oracle, dims, 4)
    _check(gpu, oracle, oracle.generate_mcm(700, 8, 1, 322), 4)  # packed, values small


def test_batch_packed_square_and_fallback(gpu, oracle, monkeypatch):
    # n <= 64 batches fold packed keys (opt-in); large dims (cells past 2^24) rerun unpacked
    monkeypatch.setenv("PIPEDP_MCM_PACKED_SQUARE", "1")
    for lo, hi in [(1, 100), (200, 255)]:
        insts = [gpu.McmInstance(oracle.generate_mcm(64, 300 + i, lo, hi)) for i in range(24)]
        for inst, (t, split) in zip(insts, gpu.solve_mcm_batch(insts)):
            wc, _, ws = oracle.mcm_solve(inst.dims)
            assert np.array_equal(t.cells, wc) and np.array_equal(split, ws)


@pytest.mark.parametrize("n,lo,hi", [(330, 1, 100),     # 32-bit table too big for shared memory
                                     (250, 1300, 2000),  # 64-bit values from the start
                                     (300, 1000, 1290)])  # 32-bit square, overflows -> exact int64 rerun
def test_batch_beyond_shared_memory(gpu, oracle, n, lo, hi):
    # batches whose tables do not fit one CTA's shared memory run the dataflow
    # wavefront instance by instance; every instance is checked
    insts = [gpu.generate_mcm(n=n, seed=s, dims_min=lo, dims_max=hi) for s in (1, 2, 3)]
    for inst, (t, split) in zip(insts, gpu.solve_mcm_batch(insts)):
        wc, _, ws = oracle.mcm_solve(inst.dims)
        assert np.array_equal(t.cells, wc) and np.array_equal(split, ws)
    # the same plan executed twice keeps its dispatch (the overflow rerun must
    # not rewrite the plan)
    import torch
    dims = np.concatenate([i.dims for i in insts])
    plan = gpu.McmPlan(3, n, dims, device=0)
    size = gpu.cell_count(n) + 1
    for _ in range(2):
        c = torch.full((3 * size,), -1, dtype=torch.int64, device="cuda")
        s = torch.full((3 * size,), -1, dtype=torch.int64, device="cuda")
        plan.execute(c.data_ptr(), s.data_ptr(), torch.cuda.current_stream().cuda_stream)
        c, s = c.cpu().numpy(), s.cpu().numpy()
        for b, inst in enumerate(insts):
            wc, _, ws = oracle.mcm_solve(inst.dims)
            assert np.array_equal(c[b * size:(b + 1) * size], wc)
            assert np.array_equal(s[b * size:(b + 1) * size], ws)


@pytest.mark.parametrize("warp", ["1", "0"])
def test_batch_warp_kernel_and_square(gpu, oracle, monkeypatch, warp):
    # n <= 64 batches: mcm_batch_warp (one warp per instance, packed keys with
    # the split column in the low field; the default) and, with
    # PIPEDP_MCM_BATCH_WARP=0, the square-table CTAs' packed fold
    monkeypatch.setenv("PIPEDP_MCM_BATCH_WARP", warp)
    for n in (1, 2, 17, 31, 32, 33, 63, 64):
        insts = [gpu.McmInstance(oracle.generate_mcm(n, 900 + i, 1, 100)) for i in range(20)]
        for inst, (t, split) in zip(insts, gpu.solve_mcm_batch(insts)):
            wc, _, ws = oracle.mcm_solve(inst.dims)
            assert np.array_equal(t.cells, wc) and np.array_equal(split, ws)
    # all-equal dimensions (every cell a tie: the first split must win), and
    # weights just under 2^24 whose cells pass 2^24 (overflow bit 2: the
    # launch reruns unpacked)
    for dims in ([7] * 65, [3] * 40, oracle.generate_mcm(64, 5, 200, 255), oracle.generate_mcm(50, 6, 240, 255)):
        insts = [gpu.McmInstance(dims)] * 3
        for inst, (t, split) in zip(insts, gpu.solve_mcm_batch(insts)):
            wc, _, ws = oracle.mcm_solve(inst.dims)
            assert np.array_equal(t.cells, wc) and np.array_equal(split, ws)


@pytest.mark.parametrize("shape", [(1, 300, 1, 100), (1, 300, 5000, 20000), (40, 64, 1, 100), (9, 64, 240, 255)])
def test_plan_execute_is_graph_capturable(gpu, oracle, shape):
    # the device plan's overflow reruns are launched behind the first attempt,
    # gated on its flag on the device (no host round trip), so a whole
    # execute -- including a rerun it turns out to need (wide dims: 64-bit;
    # dims near 255: cells past 2^24 -> unpacked) -- replays from a CUDA graph
    import torch
    batch, n, lo, hi = shape
    insts = [oracle.generate_mcm(n, 40 + i, lo, hi) for i in range(batch)]
    dims = np.concatenate([np.asarray(d, np.int64) for d in insts])
    plan = gpu.McmPlan(batch, n, dims)
    size = gpu.cell_count(n) + 1
    c = torch.full((batch * size,), -1, dtype=torch.int64, device="cuda")
    s = torch.full_like(c, -1)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.execute(c.data_ptr(), s.data_ptr(), st.cuda_stream)  # warm-up: kernel attributes, scratch
    torch.cuda.synchronize()
    c.fill_(-1)
    s.fill_(-1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        plan.execute(c.data_ptr(), s.data_ptr(), st.cuda_stream)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        cc, ss = c.cpu().numpy(), s.cpu().numpy()
        for b, d in enumerate(insts):
            wc, _, ws = oracle.mcm_solve(d)
            assert np.array_equal(cc[b * size:(b + 1) * size], wc)
            assert np.array_equal(ss[b * size:(b + 1) * size], ws)
        c.fill_(-1)
        s.fill_(-1)
    plan.close()
