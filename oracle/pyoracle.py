"""ctypes bindings for the CHECKERS -- test infrastructure only.

* ``C``   -- oracle/_build/libpipedp_oracle.so, the plain-C restatement of the
             reference hot path (pipedp_oracle.c, every function cites the
             reference file:line it restates).
* ``REF`` -- oracle/_ref/libpipedp_ref.so, the unmodified reference library
             compiled from /root/reference/proj/src by oracle/Makefile (None when
             it was not built, e.g. a checkout without the reference mounted).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpipedp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpipedp_ref.so")

OPS = {"min": 0, "max": 1, "saturating-add": 2, "modular-add": 3}
ERRC = [
    "NonDecreasingOffsets", "NonPositiveOffset", "InitLengthMismatch", "TableTooSmall",
    "CoordOutOfRange", "AddressOutOfRange", "BaseCellHasNoDeps", "TooLargeForBruteForce",
    "StallLivelock", "WeightOverflow", "InvalidParams",
]

_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _p64(a):
    return a.ctypes.data_as(_i64p) if a is not None else None


def _pu8(a):
    return a.ctypes.data_as(_u8p) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code: int):
        self.code = code
        super().__init__(ERRC[code - 1] if 1 <= code <= len(ERRC) else f"status {code}")


def _check(rc):
    if rc:
        raise OracleError(rc)


class _Lib:
    """Common surface of the C restatement (prefix or_) and the reference shim (ref_)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.lib = C.CDLL(path)
        self.prefix = prefix
        L = self.lib
        f = lambda name: getattr(L, prefix + name)  # noqa: E731
        self._apply = f("apply")
        self._apply.restype = C.c_int64
        self._apply.argtypes = [C.c_int, C.c_int64, C.c_int64]
        self._sdp = f("sdp_solve")
        self._sdp.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int, _i64p, _u8p]
        self._mcm = f("mcm_solve")
        self._mcm.argtypes = [_i64p, C.c_int64, _i64p, _u8p, _i64p]
        self._brute = f("mcm_bruteforce")
        self._brute.restype = C.c_int64
        self._brute.argtypes = [_i64p, C.c_int64]
        self._lin = f("mcm_lin")
        self._lin.restype = C.c_int64
        self._lin.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        self._coord = f("mcm_coord")
        self._coord.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        self._digest = f("table_digest")
        self._digest.restype = C.c_uint64
        self._digest.argtypes = [_i64p, C.c_int64]
        self._gen_mcm = f("generate_mcm")
        self._gen_mcm.argtypes = [C.c_int64, C.c_uint64, C.c_int64, C.c_int64, _i64p]

    # -- semigroup ---------------------------------------------------------
    def apply(self, op, a: int, b: int) -> int:
        return int(self._apply(OPS.get(op, op), a, b))

    # -- S-DP --------------------------------------------------------------
    def sdp_solve(self, offsets, init, n: int, op):
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        ini = np.ascontiguousarray(init, dtype=np.int64)
        cells = np.zeros(max(n, 1), dtype=np.int64)
        filled = np.zeros(max(n, 1), dtype=np.uint8)
        _check(self._sdp(_p64(offs), len(offs), _p64(ini), len(ini), n, OPS.get(op, op),
                         _p64(cells), _pu8(filled)))
        return cells, filled

    # -- MCM ---------------------------------------------------------------
    def mcm_solve(self, dims, with_split: bool = True):
        d = np.ascontiguousarray(dims, dtype=np.int64)
        n = len(d) - 1
        size = max(n * (n + 1) // 2 + 1, 1)
        cells = np.zeros(size, dtype=np.int64)
        filled = np.zeros(size, dtype=np.uint8)
        split = np.zeros(size, dtype=np.int64) if with_split else None
        _check(self._mcm(_p64(d), len(d), _p64(cells), _pu8(filled), _p64(split)))
        return cells, filled, split

    def mcm_bruteforce(self, dims) -> int:
        d = np.ascontiguousarray(dims, dtype=np.int64)
        v = int(self._brute(_p64(d), len(d)))
        if v < 0:
            raise OracleError(-v)
        return v

    def lin(self, row, col, n):
        return int(self._lin(row, col, n))

    def coord(self, address, n):
        r, c = C.c_int64(), C.c_int64()
        _check(self._coord(address, n, C.byref(r), C.byref(c)))
        return r.value, c.value

    def digest(self, cells) -> int:
        a = np.ascontiguousarray(cells, dtype=np.int64)
        return int(self._digest(_p64(a), len(a)))

    def generate_mcm(self, n, seed, lo=1, hi=50):
        dims = np.zeros(n + 1, dtype=np.int64)
        _check(self._gen_mcm(n, seed, lo, hi, _p64(dims)))
        return dims


class OracleC(_Lib):
    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path, "or_")
        L = self.lib
        L.or_mcm_pipeline.argtypes = [_i64p, C.c_int64, C.c_int, _i64p, _u8p, _i64p, _i64p]
        L.or_generate_sdp.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_int64,
                                      _i64p, _i64p, C.c_int64]
        L.or_sdp_validate.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int64]
        L.or_mcm_validate.argtypes = [_i64p, C.c_int64]

    def mcm_pipeline(self, dims, mode: int):
        d = np.ascontiguousarray(dims, dtype=np.int64)
        n = len(d) - 1
        size = n * (n + 1) // 2 + 1
        cells = np.zeros(size, dtype=np.int64)
        filled = np.zeros(size, dtype=np.uint8)
        steps, stall = C.c_int64(), C.c_int64()
        _check(self.lib.or_mcm_pipeline(_p64(d), len(d), mode, _p64(cells), _pu8(filled),
                                        C.byref(steps), C.byref(stall)))
        return cells, filled, steps.value, stall.value

    def generate_sdp(self, n, k, seed, consecutive=False, a1_cap=0):
        cap = k if consecutive else (a1_cap if a1_cap > 0 else 2 * k)
        offs = np.zeros(k, dtype=np.int64)
        init = np.zeros(max(cap, k), dtype=np.int64)
        _check(self.lib.or_generate_sdp(n, k, seed, int(consecutive), a1_cap, _p64(offs),
                                        _p64(init), len(init)))
        return offs, init[: offs[0]].copy()

    def sdp_validate(self, offsets, init_len, n):
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        return int(self.lib.or_sdp_validate(_p64(offs), len(offs), init_len, n))

    def mcm_validate(self, dims):
        d = np.ascontiguousarray(dims, dtype=np.int64)
        return int(self.lib.or_mcm_validate(_p64(d), len(d)))


class OracleRef(_Lib):
    def __init__(self, path: str = REF_SO):
        super().__init__(path, "ref_")
        L = self.lib
        L.ref_mcm_pipeline.argtypes = [_i64p, C.c_int64, C.c_int, C.c_int, _i64p, _u8p, _i64p,
                                       _i64p, _i64p]
        L.ref_sdp_pipeline.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int,
                                       _i64p, _u8p, _i64p, _i64p]
        L.ref_sdp_solve_model.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int,
                                          C.c_int, _i64p, _u8p, _i64p, _i64p]
        L.ref_generate_sdp.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_int64,
                                       _i64p, _i64p, C.c_int64, _i64p]
        L.ref_hazard_frontier.restype = C.c_int64
        L.ref_hazard_frontier.argtypes = [C.c_int64, _i64p, C.c_int64]
        L.ref_validate_sdp.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int64]
        L.ref_validate_mcm.argtypes = [_i64p, C.c_int64]

    def mcm_pipeline(self, dims, mode: int, collect_trace: bool = False):
        d = np.ascontiguousarray(dims, dtype=np.int64)
        n = len(d) - 1
        size = n * (n + 1) // 2 + 1
        cells = np.zeros(size, dtype=np.int64)
        filled = np.zeros(size, dtype=np.uint8)
        steps, stall, hz = C.c_int64(), C.c_int64(), C.c_int64()
        _check(self.lib.ref_mcm_pipeline(_p64(d), len(d), mode, int(collect_trace), _p64(cells),
                                         _pu8(filled), C.byref(steps), C.byref(stall),
                                         C.byref(hz)))
        return cells, filled, steps.value, stall.value, hz.value

    def sdp_pipeline(self, offsets, init, n, op):
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        ini = np.ascontiguousarray(init, dtype=np.int64)
        cells = np.zeros(n, dtype=np.int64)
        filled = np.zeros(n, dtype=np.uint8)
        steps, first = C.c_int64(), C.c_int64()
        _check(self.lib.ref_sdp_pipeline(_p64(offs), len(offs), _p64(ini), len(ini), n,
                                         OPS.get(op, op), _p64(cells), _pu8(filled),
                                         C.byref(steps), C.byref(first)))
        return cells, filled, steps.value, first.value

    def sdp_model(self, offsets, init, n, op, which: int):
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        ini = np.ascontiguousarray(init, dtype=np.int64)
        cells = np.zeros(n, dtype=np.int64)
        filled = np.zeros(n, dtype=np.uint8)
        model, aux = C.c_int64(), C.c_int64()
        _check(self.lib.ref_sdp_solve_model(_p64(offs), len(offs), _p64(ini), len(ini), n,
                                            OPS.get(op, op), which, _p64(cells), _pu8(filled),
                                            C.byref(model), C.byref(aux)))
        return cells, filled, model.value, aux.value

    def generate_sdp(self, n, k, seed, consecutive=False, a1_cap=0):
        cap = k if consecutive else (a1_cap if a1_cap > 0 else 2 * k)
        offs = np.zeros(k, dtype=np.int64)
        init = np.zeros(max(cap, k), dtype=np.int64)
        a1 = C.c_int64()
        _check(self.lib.ref_generate_sdp(n, k, seed, int(consecutive), a1_cap, _p64(offs),
                                         _p64(init), len(init), C.byref(a1)))
        return offs, init[: a1.value].copy()

    def mcm_engine_digests(self, dims, mode: int):
        """ref_mcm_engine_digests: trace/report digest vector of solve_mcm_pipeline."""
        d = np.ascontiguousarray(dims, dtype=np.int64)
        out = np.zeros(14, dtype=np.uint64)
        _check(self.lib.ref_mcm_engine_digests(_p64(d), len(d), mode, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return [int(x) for x in out]

    def sdp_engine_digests(self, offsets, init, n, op):
        """ref_sdp_engine_digests: trace/report digest vector of solve_sdp_pipeline."""
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        ini = np.ascontiguousarray(init, dtype=np.int64)
        out = np.zeros(14, dtype=np.uint64)
        _check(self.lib.ref_sdp_engine_digests(_p64(offs), len(offs), _p64(ini), len(ini), n, OPS.get(op, op),
                                               out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return [int(x) for x in out]

    def hazard_frontier(self, n):
        out = np.zeros(n * n, dtype=np.int64)
        cnt = int(self.lib.ref_hazard_frontier(n, _p64(out), len(out)))
        return out[:cnt].copy()

    def sdp_validate(self, offsets, init_len, n):
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        return int(self.lib.ref_validate_sdp(_p64(offs), len(offs), init_len, n))

    def mcm_validate(self, dims):
        d = np.ascontiguousarray(dims, dtype=np.int64)
        return int(self.lib.ref_validate_mcm(_p64(d), len(d)))


def load_c() -> OracleC:
    if not os.path.exists(ORACLE_SO):
        build()
    return OracleC()


def load_ref():
    """The reference build, or None when oracle/_ref was never built."""
    return OracleRef() if os.path.exists(REF_SO) else None
