"""The C++ drop-in (include/pipedp/*.hpp -> _lib/libpipedp_b200.so): compile a
caller the way the reference's callers are written (tests/cpp/dropin_test.cpp)
and check it.  CPU: validation/errc/generators and the loud no-GPU failure.
GPU: the solvers' tables against the reference's golden digests."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")
LIB = os.path.join(ROOT, "paper_2008_01938_b200", "_lib")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


@pytest.fixture(scope="module")
def binary(pd):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    dropin = os.path.join(LIB, "libpipedp_b200.so")
    assert os.path.exists(dropin), "drop-in library not built"
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(SRC), os.path.getmtime(dropin)):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                        "-L", LIB, "-lpipedp_b200", "-lpipedp_cuda", f"-Wl,-rpath,{LIB}",
                        "-o", OUT], check=True)
    return OUT


def _run(binary, mode):
    r = subprocess.run([binary, mode], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout


def test_dropin_validation_and_generators(binary):
    rc, out = _run(binary, "validate")
    assert rc == 0 and out.strip().endswith("OK"), out
    lines = dict(l.split(" ", 1) for l in out.splitlines() if l.startswith("gen_"))
    g = next(c for c in GOLDEN["gen_sdp"] if c["args"][:3] == [1 << 24, 1024, 1])
    assert lines["gen_sdp"].split() == [g["offsets_digest"], g["init_digest"]]
    m = next(c for c in GOLDEN["gen_mcm"] if c["args"] == [1024, 1, 1, 100])
    assert lines["gen_mcm"].strip() == m["digest"]


def test_dropin_no_cpu_fallback(binary, pd):
    if pd.device_count() > 0:
        pytest.skip("a GPU is visible; the no-GPU contract is checked on the CPU box")
    rc, out = _run(binary, "nogpu")
    assert rc == 0 and out.strip().endswith("OK"), out


@pytest.mark.gpu
def test_dropin_solvers_on_gpu(binary, gpu):
    rc, out = _run(binary, "solve")
    assert rc == 0 and out.strip().endswith("OK"), out
    for line in out.splitlines():
        f = line.split()
        if f[0] == "sdp":
            want = next(c for c in GOLDEN["sdp"] if c["gen"] == [20000, 1024, 11, False, 4096] and c["op"] == f[5])
            assert f[6] == want["digest"], line
        elif f[0] == "mcm":
            n = int(f[1])
            if n == 64:
                want = GOLDEN["configs"]["mcm64"]
            else:
                want = next(c for c in GOLDEN["mcm"] if c.get("gen", [0])[0] == n)
            assert f[2] == want["digest"] and f[3] == want["split_digest"], line


def test_dropin_instance_io_and_parenthesization(binary):
    # reference io.cpp formats, the batched loader, split-table parenthesisation
    rc, out = _run(binary, "io")
    assert rc == 0 and out.strip().endswith("OK"), out


# ---- INTEGRATION.md §2 for real: the reference's own callers on the drop-in ----
CALLERS = os.path.join(ROOT, "tests", "cpp", "_build", "ref_callers")
GOLD_DIR = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def ref_callers(pd):
    """tests/cpp/Makefile: proj/src/commands.cpp, analysis.cpp, io.cpp compiled
    against include/ (+ the reference's include/ for commands.hpp) and linked
    with -lpipedp_b200 -lpipedp_cuda -- built here from /root/reference, or
    prebuilt (build()) where the reference is absent."""
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), CALLERS], check=True)
    if not os.path.exists(CALLERS):
        pytest.skip("reference callers not built (reference sources absent and no prebuilt binary)")
    return CALLERS


def _strip_msec(text):
    return "".join(l + "\n" for l in text.splitlines() if not l.startswith("msec:"))


def test_reference_callers_link_and_fail_loudly_without_gpu(ref_callers, pd):
    if pd.device_count() > 0:
        pytest.skip("a GPU is visible; the no-GPU contract is checked on the CPU box")
    r = subprocess.run([ref_callers, "run"], capture_output=True, text=True, timeout=120)
    rcs = [l for l in r.stdout.splitlines() if " rc=" in l]
    assert len(rcs) == 6 and all(l.endswith("rc=2") for l in rcs), r.stdout
    assert r.stderr.count("error: NoDevice") == 6, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["run", "verify"])
def test_reference_callers_on_gpu(ref_callers, gpu, mode):
    """cmd_run / cmd_verify of the reference, unchanged, over the B200 drop-in:
    same digests, steps, conflict counts, hazard frontier and verdicts as the
    same program linked with the reference's own solvers."""
    r = subprocess.run([ref_callers, mode], capture_output=True, text=True, timeout=600)
    want = open(os.path.join(GOLD_DIR, f"ref_callers_{mode}.txt")).read()
    assert _strip_msec(r.stdout) == want, r.stderr[-2000:]
