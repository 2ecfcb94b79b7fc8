"""pipedp-b200: B200-native pipelined DP solvers (S-DP and matrix-chain
multiplication) behind the reference ``pipedp`` solver interface.

This module is the Python mirror of the reference's C++ API
(/root/reference/proj/include/pipedp): same names, same argument meaning,
same error codes -- ``Error`` carries the reference ``errc`` name.  Every
solver calls the C ABI in ``_lib/libpipedp_cuda.so`` (include/pipedp_cuda.h);
there is no CPU solver anywhere in the package, and a missing library or GPU
raises instead of falling back.

Reference map:
  solve_sequential / solve_prefix_parallel / solve_naive_parallel   sdp.cpp:84-111
  solve_sdp_pipeline                                                sdp_pipeline.cpp:34-44
  solve_mcm_sequential (with split table)                           mcm.cpp:85-110
  solve_mcm_pipeline (paper_literal / stall_on_hazard)              mcm_pipeline.cpp:32-47
  generate_sdp / generate_mcm                                       generate.cpp:21-60
  table_digest                                                      table.cpp:12-25
New (no reference counterpart): solve_sequential_batch, solve_mcm_batch,
solve_mcm_tournament, SdpPlan / McmPlan (device-resident execution).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIPEDP_LIB") or os.path.join(_HERE, "_lib", "libpipedp_cuda.so")
DROPIN_PATH = os.path.join(_HERE, "_lib", "libpipedp_b200.so")

ERRC = [
    "NonDecreasingOffsets", "NonPositiveOffset", "InitLengthMismatch", "TableTooSmall",
    "CoordOutOfRange", "AddressOutOfRange", "BaseCellHasNoDeps", "TooLargeForBruteForce",
    "StallLivelock", "WeightOverflow", "InvalidParams",
]
OPS = ("min", "max", "saturating-add", "modular-add")  # OpKind order, semigroup.hpp:13

MCM_AUTO, MCM_WAVEFRONT, MCM_SMEM, MCM_TOURNAMENT, MCM_TILED = 0, 1, 2, 3, 4
SDP_PIPELINE, SDP_PREFIX, SDP_NAIVE = 0, 1, 2  # pipedp_sdp_plan_set_method
PAPER_LITERAL, STALL_ON_HAZARD = "paper_literal", "stall_on_hazard"

# C ABI exports declared in include/pipedp_cuda.h (checked by tests/test_host.py)
EXPORTS = (
    "pipedp_last_error", "pipedp_version", "pipedp_device_count", "pipedp_sdp_validate",
    "pipedp_mcm_validate", "pipedp_table_digest", "pipedp_generate_sdp", "pipedp_generate_mcm",
    "pipedp_sdp_solve", "pipedp_sdp_solve_batch", "pipedp_sdp_plan_create",
    "pipedp_sdp_plan_execute", "pipedp_sdp_plan_describe", "pipedp_sdp_plan_destroy",
    "pipedp_mcm_solve", "pipedp_mcm_pipeline", "pipedp_mcm_solve_batch",
    "pipedp_mcm_plan_create", "pipedp_mcm_plan_execute", "pipedp_mcm_plan_describe",
    "pipedp_mcm_plan_destroy", "pipedp_digest_device", "pipedp_chain_step_ns",
    "pipedp_profile_read", "pipedp_generate_sdp_batch", "pipedp_generate_mcm_batch",
    "pipedp_op_latency_ns", "pipedp_mcm_bruteforce", "pipedp_sdp_solve_method",
    "pipedp_sdp_plan_set_method", "pipedp_mcm_engine", "pipedp_sdp_engine", "pipedp_engine_records",
    "pipedp_engine_hazards", "pipedp_engine_conflicts", "pipedp_engine_stall_heads", "pipedp_engine_free",
    "pipedp_sdp_plan_set_timing", "pipedp_sdp_plan_phase_ms",
)
ENGINE_TRACE, ENGINE_ANALYSIS = 1, 2
TRACE_LIMIT = 1 << 28  # engine.cu kMaxRecords


class EngineSummary(C.Structure):
    """pipedp_engine_summary (include/pipedp_cuda.h)."""
    _fields_ = [(f, C.c_int64) for f in ("first_head", "steps_executed", "stall_iterations", "records",
                                         "hazards", "conflict_groups", "conflict_lanes", "max_group_size",
                                         "stall_heads")]


class Error(RuntimeError):
    """pipedp::Error -- a reference errc (error.hpp:25-36)."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.name = ERRC[code - 1]
        super().__init__(message)


class DeviceError(RuntimeError):
    """No usable sm_100 GPU, CUDA failure or out of memory (no CPU fallback)."""

    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(message)


# ------------------------------------------------------------------ library --
_lib = None
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)


def lib():
    """The loaded C ABI library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH} -- run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    L.pipedp_last_error.restype = C.c_char_p
    L.pipedp_version.restype = C.c_char_p
    L.pipedp_device_count.restype = C.c_int32
    L.pipedp_sdp_validate.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int64]
    L.pipedp_mcm_validate.argtypes = [_i64p, C.c_int64]
    L.pipedp_table_digest.restype = C.c_uint64
    L.pipedp_table_digest.argtypes = [_i64p, C.c_int64]
    L.pipedp_generate_sdp.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_uint64, C.c_int32,
                                      C.c_int64, _i64p, _i64p, C.c_int64, _i64p]
    L.pipedp_generate_mcm.argtypes = [C.c_int64, C.c_uint64, C.c_int64, C.c_int64, _i64p]
    L.pipedp_generate_sdp_batch.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int64, C.c_int32,
                                            C.c_int64, _i64p, _i64p, _i64p]
    L.pipedp_generate_mcm_batch.argtypes = [C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                            _i64p]
    L.pipedp_sdp_solve.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int32,
                                   _i64p, _u8p]
    L.pipedp_sdp_solve_batch.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p,
                                         C.c_int32, _i64p, C.c_int32]
    L.pipedp_sdp_plan_create.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p,
                                         C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    L.pipedp_sdp_plan_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.pipedp_sdp_plan_describe.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t,
                                           C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.pipedp_sdp_plan_destroy.argtypes = [C.c_void_p]
    L.pipedp_mcm_solve.argtypes = [_i64p, C.c_int64, C.c_int32, _i64p, _u8p, _i64p]
    L.pipedp_mcm_pipeline.argtypes = [_i64p, C.c_int64, C.c_int32, _i64p, _u8p, _i64p, _i64p]
    L.pipedp_mcm_solve_batch.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _i64p, C.c_int32]
    L.pipedp_mcm_plan_create.argtypes = [C.c_int64, C.c_int64, _i64p, C.c_int32, C.c_int32,
                                         C.POINTER(C.c_void_p)]
    L.pipedp_mcm_plan_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.pipedp_mcm_plan_describe.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t,
                                           C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.pipedp_mcm_plan_destroy.argtypes = [C.c_void_p]
    L.pipedp_digest_device.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    L.pipedp_chain_step_ns.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
    L.pipedp_op_latency_ns.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
    L.pipedp_mcm_bruteforce.argtypes = [_i64p, C.c_int64, _i64p]
    L.pipedp_sdp_solve_method.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int32,
                                          C.c_int32, _i64p, _u8p]
    L.pipedp_sdp_plan_set_method.argtypes = [C.c_void_p, C.c_int32]
    L.pipedp_sdp_plan_set_timing.argtypes = [C.c_void_p, C.c_int32]
    L.pipedp_sdp_plan_phase_ms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    _i32p = C.POINTER(C.c_int32)
    L.pipedp_mcm_engine.argtypes = [_i64p, C.c_int64, C.c_int32, C.c_int32, _i64p, C.POINTER(EngineSummary),
                                    C.POINTER(C.c_void_p)]
    L.pipedp_sdp_engine.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _i64p,
                                    C.POINTER(EngineSummary), C.POINTER(C.c_void_p)]
    L.pipedp_engine_records.argtypes = [C.c_void_p, _i64p, _i32p, _i32p, _i32p, _i64p]
    L.pipedp_engine_hazards.argtypes = [C.c_void_p, _i64p]
    L.pipedp_engine_conflicts.argtypes = [C.c_void_p, _i64p, _i32p, _i32p, _i32p]
    L.pipedp_engine_stall_heads.argtypes = [C.c_void_p, _i64p]
    L.pipedp_engine_free.argtypes = [C.c_void_p]
    L.pipedp_engine_free.restype = None
    _lib = L
    return L


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().pipedp_last_error().decode()
    if 1 <= status <= len(ERRC):
        raise Error(status, msg)
    raise DeviceError(status, msg)


def _a64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int64)


def _p(a: Optional[np.ndarray], t=_i64p):
    return None if a is None else a.ctypes.data_as(t)


def device_count() -> int:
    return int(lib().pipedp_device_count())


# -------------------------------------------------------------------- types --
def _op_index(op) -> int:
    if isinstance(op, str):
        if op not in OPS:
            raise Error(11, f"InvalidParams: unknown operator name: {op}")
        return OPS.index(op)
    return int(op)


@dataclass
class SdpInstance:
    """SdpInstance (sdp.hpp:24-31): n cells, strictly decreasing offsets, a_1 init values."""

    n: int
    offsets: Sequence[int]
    init: Sequence[int]
    op: str = "min"

    @property
    def k(self) -> int:
        return len(self.offsets)

    @property
    def a1(self) -> int:
        return int(self.offsets[0])


@dataclass
class McmInstance:
    """McmInstance (mcm.hpp:11-17): dims p_0..p_n."""

    dims: Sequence[int]

    @property
    def n(self) -> int:
        return len(self.dims) - 1


@dataclass
class SolutionTable:
    """SolutionTable (table.hpp:11-23): int64 cells + uint8 filled flags."""

    cells: np.ndarray
    filled: np.ndarray

    def all_filled(self) -> bool:
        return bool(np.all(self.filled != 0))

    def __eq__(self, other) -> bool:  # defaulted == compares both vectors
        return (np.array_equal(self.cells, other.cells)
                and np.array_equal(self.filled, other.filled))


RECORD_DTYPE = np.dtype([("head", np.int64), ("substep", np.int32), ("lane", np.int32), ("kind", np.int32),
                         ("address", np.int64)])
HAZARD_DTYPE = np.dtype([("head", np.int64), ("substep", np.int64), ("lane", np.int64), ("address", np.int64),
                         ("finalization_head", np.int64), ("finalization_substep", np.int64)])


@dataclass
class PipelineTrace:
    """PipelineTrace (engine.hpp:68-77).  records: RECORD_DTYPE array in
    record_less order (kind 0 read, 1 write), emitted by the GPU lock-step
    engine when collected."""

    first_head: int = 0
    steps_executed: int = 0
    stall_iterations: int = 0
    records: np.ndarray = field(default_factory=lambda: np.zeros(0, RECORD_DTYPE))
    collected: bool = False
    stall_heads: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


@dataclass
class ConflictGroup:
    head: int
    substep: int
    kind: int
    address: int
    lanes: list


@dataclass
class ConflictReport:
    """ConflictReport (analysis.hpp:23-34), computed on the device."""

    groups: list = field(default_factory=list)
    max_group_size: int = 1
    first_head: int = 0
    per_step_cost: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))


@dataclass
class HazardReport:
    """HazardReport (analysis.hpp:54-58): HAZARD_DTYPE records, detect_hazards order."""

    hazards: np.ndarray = field(default_factory=lambda: np.zeros(0, HAZARD_DTYPE))

    def empty(self) -> bool:
        return len(self.hazards) == 0


@dataclass
class SdpPipelineResult:
    table: SolutionTable
    trace: PipelineTrace
    conflicts: ConflictReport = field(default_factory=ConflictReport)


@dataclass
class McmPipelineResult:
    table: SolutionTable
    trace: PipelineTrace
    conflicts: ConflictReport = field(default_factory=ConflictReport)
    hazards: HazardReport = field(default_factory=HazardReport)


def _engine_results(run, summ: "EngineSummary", collected: bool, analysis: bool):
    """Copy one pipedp_*_engine run's results into the reference's result types."""
    L = lib()
    try:
        tr = PipelineTrace(summ.first_head, summ.steps_executed, summ.stall_iterations, collected=collected)
        tr.stall_heads = np.zeros(summ.stall_heads, np.int64)
        _check(L.pipedp_engine_stall_heads(run, _p(tr.stall_heads)))
        nr = summ.records
        if nr:
            rec = np.zeros(nr, RECORD_DTYPE)
            cols = {f: np.zeros(nr, RECORD_DTYPE[f]) for f in RECORD_DTYPE.names}
            i32 = C.POINTER(C.c_int32)
            _check(L.pipedp_engine_records(run, _p(cols["head"]), _p(cols["substep"], i32), _p(cols["lane"], i32),
                                           _p(cols["kind"], i32), _p(cols["address"])))
            for f in RECORD_DTYPE.names:
                rec[f] = cols[f]
            tr.records = rec
        conf, haz = ConflictReport(first_head=summ.first_head), HazardReport()
        if analysis:
            g = summ.conflict_groups
            groups = np.zeros(4 * g, np.int64)
            sizes = np.zeros(g, np.int32)
            lanes = np.zeros(summ.conflict_lanes, np.int32)
            conf.per_step_cost = np.zeros(max(summ.steps_executed, 0), np.int32)
            i32 = C.POINTER(C.c_int32)
            _check(L.pipedp_engine_conflicts(run, _p(groups), _p(sizes, i32), _p(lanes, i32),
                                             _p(conf.per_step_cost, i32)))
            at = 0
            for i in range(g):
                h, sub, kind, addr = (int(x) for x in groups[4 * i:4 * i + 4])
                conf.groups.append(ConflictGroup(h, sub, kind, addr, [int(x) for x in lanes[at:at + sizes[i]]]))
                at += int(sizes[i])
            conf.max_group_size = int(summ.max_group_size)
            hz = np.zeros(summ.hazards * 6, np.int64)
            _check(L.pipedp_engine_hazards(run, _p(hz)))
            haz.hazards = hz.view(HAZARD_DTYPE).copy() if summ.hazards else np.zeros(0, HAZARD_DTYPE)
        return tr, conf, haz
    finally:
        L.pipedp_engine_free(run)


@dataclass
class PrefixParallelResult:
    table: SolutionTable
    depth_per_cell: int
    modeled_steps: int


@dataclass
class NaiveParallelResult:
    table: SolutionTable
    serialized_accesses_per_cell: int
    modeled_steps: int


def table_digest(cells) -> int:
    a = _a64(cells)
    return int(lib().pipedp_table_digest(_p(a), len(a)))


def digest_hex(d: int) -> str:
    return f"{d:016x}"


# ------------------------------------------------------------------- S-DP ----
def validate(instance):
    """validate(SdpInstance) sdp.cpp:10-32 / validate(McmInstance) mcm.cpp:11-28."""
    if isinstance(instance, SdpInstance):
        offs = _a64(instance.offsets)
        _check(lib().pipedp_sdp_validate(_p(offs), len(offs), len(instance.init), instance.n))
    else:
        d = _a64(instance.dims)
        _check(lib().pipedp_mcm_validate(_p(d), len(d)))
    return instance


def solve_sequential(inst: SdpInstance) -> SolutionTable:
    offs, init = _a64(inst.offsets), _a64(inst.init)
    op = _op_index(inst.op)
    validate(inst)
    cells = np.empty(inst.n, dtype=np.int64)
    filled = np.empty(inst.n, dtype=np.uint8)
    _check(lib().pipedp_sdp_solve(_p(offs), len(offs), _p(init), len(init), inst.n, op,
                                  _p(cells), _p(filled, _u8p)))
    return SolutionTable(cells, filled)


def _ceil_log2(k: int) -> int:
    return (k - 1).bit_length()


def _solve_method(inst: SdpInstance, method: int) -> SolutionTable:
    offs, init = _a64(inst.offsets), _a64(inst.init)
    op = _op_index(inst.op)
    validate(inst)
    cells = np.empty(inst.n, dtype=np.int64)
    filled = np.empty(inst.n, dtype=np.uint8)
    _check(lib().pipedp_sdp_solve_method(_p(offs), len(offs), _p(init), len(init), inst.n, op, method,
                                         _p(cells), _p(filled, _u8p)))
    return SolutionTable(cells, filled)


def solve_prefix_parallel(inst: SdpInstance) -> PrefixParallelResult:
    """solve_prefix_parallel (sdp.cpp:91-100): the paper's tournament per cell on
    the device (kernel sdp_tournament), plus the reference's step model."""
    t = _solve_method(inst, SDP_PREFIX)
    depth = _ceil_log2(inst.k)
    return PrefixParallelResult(t, depth, (inst.n - inst.a1) * max(depth, 1))


def solve_naive_parallel(inst: SdpInstance) -> NaiveParallelResult:
    """solve_naive_parallel (sdp.cpp:102-111): the paper's naive k-1-thread
    method on the device (kernel sdp_naive), plus the reference's step model."""
    t = _solve_method(inst, SDP_NAIVE)
    return NaiveParallelResult(t, inst.k - 1, (inst.n - inst.a1) * inst.k)


def solve_sdp_pipeline(inst: SdpInstance, collect_trace: bool = True) -> SdpPipelineResult:
    """solve_sdp_pipeline (sdp_pipeline.cpp:34-44; SdpRunConfig default
    collect_trace = true).  With collect_trace the GPU lock-step engine runs
    SdpProgram and returns the trace records (when within TRACE_LIMIT) and the
    conflict report computed on the device; otherwise the fast solvers."""
    validate(inst)
    if not collect_trace:
        t = solve_sequential(inst)
        return SdpPipelineResult(t, PipelineTrace(inst.a1, inst.n + inst.k - inst.a1 - 1, 0))
    fits = (inst.n - inst.a1) * (3 * inst.k - 1) <= TRACE_LIMIT
    offs, init = _a64(inst.offsets), _a64(inst.init)
    cells = np.empty(inst.n, np.int64)
    summ, run = EngineSummary(), C.c_void_p()
    _check(lib().pipedp_sdp_engine(_p(offs), len(offs), _p(init), len(init), inst.n, _op_index(inst.op),
                                   ENGINE_ANALYSIS | (ENGINE_TRACE if fits else 0), _p(cells), C.byref(summ),
                                   C.byref(run)))
    tr, conf, _ = _engine_results(run, summ, fits, True)
    return SdpPipelineResult(SolutionTable(cells, np.ones(inst.n, np.uint8)), tr, conf)


def solve_sequential_batch(insts: List[SdpInstance], device: int = -1) -> List[SolutionTable]:
    if not insts:
        return []
    f = insts[0]
    for s in insts:
        validate(s)
        if (s.n, s.k, s.a1, s.op) != (f.n, f.k, f.a1, f.op):
            raise Error(11, "InvalidParams: batched instances must share n, k, a_1 and the operator")
    offs = _a64(np.concatenate([_a64(s.offsets) for s in insts]))
    init = _a64(np.concatenate([_a64(s.init) for s in insts]))
    cells = np.empty(len(insts) * f.n, dtype=np.int64)
    _check(lib().pipedp_sdp_solve_batch(len(insts), f.n, f.k, f.a1, _p(offs), _p(init),
                                        _op_index(f.op), _p(cells), device))
    return [SolutionTable(cells[i * f.n:(i + 1) * f.n].copy(), np.ones(f.n, np.uint8))
            for i in range(len(insts))]


def generate_sdp(n=64, k=4, op="min", seed=0, consecutive=False, a1_cap=0) -> SdpInstance:
    """generate_sdp (generate.cpp:21-47): same mt19937_64 draws as the reference."""
    cap = k if consecutive else (a1_cap if a1_cap > 0 else 2 * k)
    offs = np.zeros(max(k, 1), dtype=np.int64)
    init = np.zeros(max(cap, k, 1), dtype=np.int64)
    a1 = C.c_int64()
    _check(lib().pipedp_generate_sdp(n, k, _op_index(op), seed, int(consecutive), a1_cap,
                                     _p(offs), _p(init), len(init), C.byref(a1)))
    return SdpInstance(n, offs, init[: a1.value].copy(), op)


def generate_sdp_batch(n, k, seed0, count, consecutive=False, a1_cap=0):
    """Instances generate_sdp(seed = seed0 + i), i < count, as SoA arrays
    (offsets [count, k], init [count, a_1])."""
    a1 = k if consecutive else (a1_cap if a1_cap > 0 else 2 * k)
    offs = np.empty((count, k), dtype=np.int64)
    init = np.empty((count, a1), dtype=np.int64)
    got = C.c_int64()
    _check(lib().pipedp_generate_sdp_batch(n, k, seed0, count, int(consecutive), a1_cap, _p(offs),
                                           _p(init), C.byref(got)))
    return offs, init


# -------------------------------------------------------------------- MCM ----
def cell_count(n: int) -> int:
    return n * (n + 1) // 2


def lin(row: int, col: int, n: int) -> int:
    """lin (mcm.cpp:30-37)."""
    if row < 1 or row > col or col > n:
        raise Error(5, f"CoordOutOfRange: ({row},{col}) outside the order-{n} triangle")
    d = col - row
    return d * n - d * (d - 1) // 2 + row


def coord(address: int, n: int):
    """coord (mcm.cpp:39-53)."""
    if address < 1 or address > cell_count(n):
        raise Error(6, f"AddressOutOfRange: address {address} outside table of {cell_count(n)} cells")
    d, base = 0, 0
    while address > base + (n - d):
        base += n - d
        d += 1
    row = address - base
    return row, row + d


def _mcm(inst: McmInstance, kernel: int, want_split: bool):
    d = _a64(inst.dims)
    validate(inst)
    size = cell_count(inst.n) + 1
    cells = np.empty(size, dtype=np.int64)
    filled = np.empty(size, dtype=np.uint8)
    split = np.empty(size, dtype=np.int64) if want_split else None
    _check(lib().pipedp_mcm_solve(_p(d), len(d), kernel, _p(cells), _p(filled, _u8p), _p(split)))
    return SolutionTable(cells, filled), split


def solve_mcm_sequential(inst: McmInstance, split_points: Optional[list] = None,
                         kernel: int = MCM_AUTO):
    """solve_mcm_sequential (mcm.cpp:85-110).  As in the reference, the split
    table is produced only when a container is passed: it is filled in place."""
    t, split = _mcm(inst, kernel, split_points is not None)
    if split_points is not None:
        split_points[:] = split.tolist() if isinstance(split_points, list) else split
    return t


def solve_mcm_with_split(inst: McmInstance, kernel: int = MCM_AUTO):
    """(table, split ndarray) in one call -- the convenient form for tests/bench."""
    return _mcm(inst, kernel, True)


def solve_mcm_tournament(inst: McmInstance):
    return _mcm(inst, MCM_TOURNAMENT, True)


def solve_mcm_bruteforce(inst: McmInstance) -> int:
    """solve_mcm_bruteforce (mcm.cpp:130-138): enumeration over every
    parenthesisation (n <= 12), on the device."""
    d = _a64(inst.dims)
    out = C.c_int64()
    _check(lib().pipedp_mcm_bruteforce(_p(d), len(d), C.byref(out)))
    return out.value


def solve_mcm_pipeline(inst: McmInstance, mode: str = PAPER_LITERAL, collect_trace: bool = True) -> McmPipelineResult:
    """solve_mcm_pipeline (mcm_pipeline.cpp:32-47; McmScheduleConfig default
    collect_trace = true): the GPU lock-step engine running McmProgram -- table,
    steps, stalls, stall heads; with collect_trace the access records (within
    TRACE_LIMIT) and the conflict and hazard reports computed on the device."""
    d = _a64(inst.dims)
    validate(inst)
    if inst.n < 2:
        raise Error(11, "InvalidParams: pipeline needs at least two matrices")
    m = {PAPER_LITERAL: 0, STALL_ON_HAZARD: 1}[mode]
    n = inst.n
    size = cell_count(n) + 1
    fits = 4 * ((n ** 3 - n) // 6) - (size - 1 - n) <= TRACE_LIMIT
    flags = (ENGINE_ANALYSIS | (ENGINE_TRACE if fits else 0)) if collect_trace else 0
    cells = np.empty(size, dtype=np.int64)
    summ, run = EngineSummary(), C.c_void_p()
    _check(lib().pipedp_mcm_engine(_p(d), len(d), m, flags, _p(cells), C.byref(summ), C.byref(run)))
    tr, conf, haz = _engine_results(run, summ, collect_trace and fits, collect_trace)
    return McmPipelineResult(SolutionTable(cells, np.ones(size, np.uint8)), tr, conf, haz)


def solve_mcm_batch(insts: List[McmInstance], device: int = -1):
    """Independent instances of equal n: [(table, split)]."""
    if not insts:
        return []
    n = insts[0].n
    for m in insts:
        validate(m)
        if m.n != n:
            raise Error(11, "InvalidParams: batched MCM instances must share n")
    dims = _a64(np.concatenate([_a64(m.dims) for m in insts]))
    size = cell_count(n) + 1
    cells = np.empty(len(insts) * size, dtype=np.int64)
    split = np.empty(len(insts) * size, dtype=np.int64)
    _check(lib().pipedp_mcm_solve_batch(len(insts), n, _p(dims), _p(cells), _p(split), device))
    return [(SolutionTable(cells[i * size:(i + 1) * size].copy(), np.ones(size, np.uint8)),
             split[i * size:(i + 1) * size].copy()) for i in range(len(insts))]


def generate_mcm(n=8, seed=0, dims_min=1, dims_max=50) -> McmInstance:
    """generate_mcm (generate.cpp:49-60)."""
    dims = np.zeros(max(n + 1, 1), dtype=np.int64)
    _check(lib().pipedp_generate_mcm(n, seed, dims_min, dims_max, _p(dims)))
    return McmInstance(dims)


def generate_mcm_batch(n, seed0, count, dims_min=1, dims_max=100):
    """Instances generate_mcm(seed = seed0 + i) as dims [count, n+1]."""
    dims = np.empty((count, n + 1), dtype=np.int64)
    _check(lib().pipedp_generate_mcm_batch(n, seed0, count, dims_min, dims_max, _p(dims)))
    return dims


# ----------------------------------------------------- device-resident plans --
class SdpPlan:
    """Device-resident S-DP execution (C ABI pipedp_sdp_plan_*).  Host copies of
    offsets/init are used for validation and value-width planning; execute()
    takes device pointers (e.g. torch tensor .data_ptr()) and a stream handle."""

    def __init__(self, batch, n, k, a1, offsets, init, op="min", device=-1):
        self.batch, self.n, self.k, self.a1 = batch, n, k, a1
        self._offs, self._init = _a64(offsets), _a64(init)
        h = C.c_void_p()
        _check(lib().pipedp_sdp_plan_create(batch, n, k, a1, _p(self._offs), _p(self._init),
                                            _op_index(op), device, C.byref(h)))
        self.handle = h

    def execute(self, d_init: int, d_cells: int, stream: int = 0) -> None:
        _check(lib().pipedp_sdp_plan_execute(self.handle, C.c_void_p(d_init), C.c_void_p(d_cells),
                                             C.c_void_p(stream)))

    def set_method(self, method: int) -> None:
        """SDP_PIPELINE (default), SDP_PREFIX or SDP_NAIVE (the paper's methods)."""
        _check(lib().pipedp_sdp_plan_set_method(self.handle, method))

    def set_timing(self, on: bool = True) -> None:
        """chunked mode: record per-phase CUDA events on the execute stream"""
        _check(lib().pipedp_sdp_plan_set_timing(self.handle, int(on)))

    def phase_ms(self):
        """accumulated (powers, chain, chunk batch) ms and the number of executes"""
        out = (C.c_double * 3)()
        runs = C.c_int64()
        _check(lib().pipedp_sdp_plan_phase_ms(self.handle, out, C.byref(runs)))
        return tuple(out), runs.value

    def describe(self):
        buf = C.create_string_buffer(64)
        bits, launches = C.c_int32(), C.c_int32()
        _check(lib().pipedp_sdp_plan_describe(self.handle, buf, 64, C.byref(bits), C.byref(launches)))
        return buf.value.decode(), bits.value, launches.value

    def close(self):
        if self.handle:
            lib().pipedp_sdp_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class McmPlan:
    """Device-resident MCM execution (C ABI pipedp_mcm_plan_*)."""

    def __init__(self, batch, n, dims, kernel=MCM_AUTO, device=-1):
        self.batch, self.n = batch, n
        self._dims = _a64(dims)
        h = C.c_void_p()
        _check(lib().pipedp_mcm_plan_create(batch, n, _p(self._dims), kernel, device, C.byref(h)))
        self.handle = h

    def execute(self, d_cells: int, d_split: int, stream: int = 0) -> None:
        _check(lib().pipedp_mcm_plan_execute(self.handle, C.c_void_p(d_cells), C.c_void_p(d_split),
                                             C.c_void_p(stream)))

    def describe(self):
        buf = C.create_string_buffer(64)
        bits, launches = C.c_int32(), C.c_int32()
        _check(lib().pipedp_mcm_plan_describe(self.handle, buf, 64, C.byref(bits), C.byref(launches)))
        return buf.value.decode(), bits.value, launches.value

    def close(self):
        if self.handle:
            lib().pipedp_mcm_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def digest_device(d_tables: int, count: int, ntables: int, d_out: int, stream: int = 0) -> None:
    _check(lib().pipedp_digest_device(C.c_void_p(d_tables), count, ntables, C.c_void_p(d_out),
                                      C.c_void_p(stream)))


def profile_read(reset=True):
    """Role cycle counters (profiling build only, PIPEDP_LIB=..._prof.so)."""
    out = (C.c_uint64 * 128)()
    lib().pipedp_profile_read.argtypes = [C.POINTER(C.c_uint64), C.c_int32, C.c_int32]
    _check(lib().pipedp_profile_read(out, 128, int(reset)))
    return list(out)


def chain_step_ns(op="min", value_bits=32, device=-1):
    ns, mhz = C.c_double(), C.c_double()
    _check(lib().pipedp_chain_step_ns(_op_index(op), value_bits, device, C.byref(ns), C.byref(mhz)))
    return ns.value, mhz.value


def op_latency_ns(op="min", value_bits=32, device=-1):
    """(ns, SM cycles) of one dependent (x) -- the dependency-chain floor per cell."""
    ns, cyc = C.c_double(), C.c_double()
    _check(lib().pipedp_op_latency_ns(_op_index(op), value_bits, device, C.byref(ns), C.byref(cyc)))
    return ns.value, cyc.value


def hazard_frontier(n: int):
    """hazard_frontier (mcm_pipeline.hpp:128-131): addresses of the cells the
    paper-literal MCM schedule reads before they are final.  Host logic; the
    condition depends on the diagonal only (see include/pipedp/mcm_pipeline.hpp)."""
    if n < 2:
        raise Error(11, "InvalidParams: frontier needs n >= 2")
    out = []
    for D in range(1, n):
        if any(j * n - j * (2 * D - j - 1) // 2 - j <= D - 2 * j for j in range(1, D + 1)):
            base = D * n - D * (D - 1) // 2
            out.extend(base + r for r in range(1, n - D + 1))
    return out
