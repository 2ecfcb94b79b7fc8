"""Host side of the boundary, CPU only: the C-ABI library loads and exports
every symbol include/pipedp_cuda.h declares; validation, error codes, the
generators and the digest agree with the reference (golden vectors); the
Python mirror raises the reference's errc names; and with no GPU every solver
fails loudly (there is no CPU path in the product)."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pipedp_cuda.h")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int32_t|uint64_t|void)\s+(pipedp_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported(pd):
    lib = C.CDLL(pd.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/pipedp_cuda.h but not exported"
    assert sorted(pd.EXPORTS) == syms  # the Python mirror binds exactly the header


def test_library_is_sm100a_only(pd):
    # the fatbin carries sm_100a SASS and nothing else (no PTX fallback)
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pd.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches
    ptx = subprocess.run(["cuobjdump", "--list-ptx", pd.LIB_PATH], capture_output=True, text=True).stdout
    assert "ptx" not in ptx.lower() or not re.search(r"\.ptx", ptx)


def test_version_and_device_count(pd):
    assert b"sm_100a" in pd.lib().pipedp_version()
    assert pd.device_count() >= 0


def test_validation_matches_reference(pd):
    for case in GOLDEN["sdp_validate"]:
        offs = np.asarray(case["offsets"], dtype=np.int64)
        st = pd.lib().pipedp_sdp_validate(offs.ctypes.data_as(C.POINTER(C.c_int64)), len(offs),
                                          case["init_len"], case["n"])
        assert st == case["status"], case
    for case in GOLDEN["mcm_validate"]:
        dims = case["dims"] if case["dims"] is not None else [case["fill"]] * case["dims_len"]
        d = np.asarray(dims, dtype=np.int64)
        st = pd.lib().pipedp_mcm_validate(d.ctypes.data_as(C.POINTER(C.c_int64)) if len(d) else None, len(d))
        assert st == case["status"], case


def test_error_names_match_reference(pd):
    with pytest.raises(pd.Error) as e:
        pd.validate(pd.SdpInstance(16, [3, 3, 1], [0, 0, 0]))
    assert e.value.name == "NonDecreasingOffsets" and str(e.value).startswith("NonDecreasingOffsets: ")
    with pytest.raises(pd.Error) as e:
        pd.validate(pd.SdpInstance(16, [5, 3, 1], [0] * 4))
    assert e.value.name == "InitLengthMismatch"
    with pytest.raises(pd.Error) as e:
        pd.validate(pd.McmInstance([1000001, 2]))
    assert e.value.name == "WeightOverflow"
    with pytest.raises(pd.Error) as e:
        pd.lin(3, 2, 5)
    assert e.value.name == "CoordOutOfRange"
    with pytest.raises(pd.Error) as e:
        pd.coord(16, 5)
    assert e.value.name == "AddressOutOfRange"
    # validation precedes any device work: the reference error, not a device error
    with pytest.raises(pd.Error):
        pd.solve_sequential(pd.SdpInstance(5, [5, 3, 1], [0] * 5))
    with pytest.raises(pd.Error):
        pd.solve_mcm_pipeline(pd.McmInstance([4, 3]))


def test_generators_match_reference(pd):
    for case in GOLDEN["gen_sdp"]:
        n, k, seed, cons, cap = case["args"]
        inst = pd.generate_sdp(n=n, k=k, seed=seed, consecutive=cons, a1_cap=cap)
        assert f"{pd.table_digest(inst.offsets):016x}" == case["offsets_digest"]
        assert f"{pd.table_digest(inst.init):016x}" == case["init_digest"]
    for case in GOLDEN["gen_mcm"]:
        n, seed, lo, hi = case["args"]
        inst = pd.generate_mcm(n=n, seed=seed, dims_min=lo, dims_max=hi)
        assert f"{pd.table_digest(inst.dims):016x}" == case["digest"]


def test_lin_coord_match_reference(pd):
    for r, c, n, want in GOLDEN["lin"]:
        assert pd.lin(r, c, n) == want
    for a, n, r, c in GOLDEN["coord"]:
        assert pd.coord(a, n) == (r, c)


def test_digest_matches_reference(pd, oracle):
    rng = np.random.default_rng(1)
    for size in (0, 1, 7, 1000):
        x = rng.integers(-(2**63), 2**63 - 1, size, dtype=np.int64)
        assert pd.table_digest(x) == oracle.digest(x)


def test_no_cpu_fallback_without_gpu(pd):
    if pd.device_count() > 0:
        pytest.skip("GPU visible")
    with pytest.raises(pd.DeviceError) as e:
        pd.solve_sequential(pd.SdpInstance(7, [2, 1], [1, 1], "saturating-add"))
    assert "NoDevice" in str(e.value)
    for f in (lambda: pd.solve_mcm_with_split(pd.McmInstance([10, 20, 30])),
              lambda: pd.solve_mcm_pipeline(pd.McmInstance([10, 20, 30, 40])),
              lambda: pd.SdpPlan(1, 100, 2, 2, [2, 1], [1, 1]),
              lambda: pd.McmPlan(1, 8, pd.generate_mcm(8).dims)):
        with pytest.raises(pd.DeviceError):
            f()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import importlib
    import paper_2008_01938_b200 as pkg
    monkeypatch.setattr(pkg, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(pkg, "_lib", None)
    with pytest.raises(RuntimeError, match="native library missing"):
        pkg.solve_sequential(pkg.SdpInstance(7, [2, 1], [1, 1]))
    importlib.reload(pkg)


def test_product_never_imports_oracle():
    # the checker is test infrastructure: nothing under the package references it
    pkg = os.path.join(ROOT, "paper_2008_01938_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "pyoracle", "pipedp_oracle", "libpipedp_ref",
                            "oracle/_ref", "oracle/_build"):
                    assert pat not in text, (os.path.join(dirpath, f), pat)


def test_instance_text_io_round_trip_and_batch(pd):
    from paper_2008_01938_b200 import io
    s = pd.SdpInstance(40, [7, 3, 1], [5, -4, 3, 2, 1, 0, 9], "modular-add")
    m = pd.McmInstance([30, 35, 15, 5, 10, 20, 25])
    assert io.to_text(s) == "sdp 40 3 modular-add\n7 3 1\n5 -4 3 2 1 0 9\n"
    assert io.to_text(m) == "mcm 6\n30 35 15 5 10 20 25\n"
    back = io.read_instances(io.to_text(m) + io.to_text(s) + io.to_text(m))
    assert [type(x).__name__ for x in back] == ["McmInstance", "SdpInstance", "McmInstance"]
    assert list(back[1].offsets) == [7, 3, 1] and list(back[1].init) == [5, -4, 3, 2, 1, 0, 9]
    assert back[1].op == "modular-add" and list(back[0].dims) == list(m.dims)
    for bad, code in [("dp 3\n", 11), ("mcm 3\n1 2 3\n", 11), ("sdp 10 2 min\n2 2\n0 0\n", 1), ("", 11)]:
        with pytest.raises(pd.Error) as e:
            io.read_instances(bad)
        assert e.value.code == code


def test_parenthesization_from_oracle_split(pd, oracle):
    from paper_2008_01938_b200 import io
    dims = [30, 35, 15, 5, 10, 20, 25]  # CLRS 15.2: cost 15125
    cells, _, split = oracle.mcm_solve(dims)
    assert io.mcm_parenthesization(dims, split) == "((A1(A2A3))((A4A5)A6))"
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(1, 60))
        d = rng.integers(1, 100, n + 1).tolist()
        cells, _, split = oracle.mcm_solve(d)
        s = io.mcm_parenthesization(d, split)
        # evaluate the product order's cost; it must equal the apex cell
        stack = []
        i = 0
        while i < len(s):
            if s[i] == "A":
                j = i + 1
                while j < len(s) and s[j].isdigit():
                    j += 1
                a = int(s[i + 1:j])
                stack.append((d[a - 1], d[a], 0))
                i = j
            elif s[i] == ")":
                r2, c2, x2 = stack.pop()
                r1, c1, x1 = stack.pop()
                stack.append((r1, c2, x1 + x2 + r1 * c1 * c2))
                i += 1
            else:
                i += 1
        assert stack[0][2] == (int(cells[-1]) if n > 1 else 0)


def test_hazard_frontier_matches_reference(pd, ref):
    # the reference's per-cell scan (mcm_pipeline.cpp:79-93) vs the per-diagonal form
    for n in [2, 3, 4, 5, 8, 17, 64, 130]:
        got = pd.hazard_frontier(n)
        want = []
        for D in range(1, n):  # restated per cell, as the reference loops
            for r in range(1, n - D + 1):
                addr = D * n - D * (D - 1) // 2 + r
                for j in range(1, D + 1):
                    right = (D - j) * n - (D - j) * (D - j - 1) // 2 + (r + j)
                    if addr - right <= D - 2 * j:
                        want.append(addr)
                        break
        assert got == sorted(want)
        if ref is not None:  # the reference library itself (oracle/_ref)
            assert got == ref.hazard_frontier(n).tolist()
    with pytest.raises(pd.Error):
        pd.hazard_frontier(1)
