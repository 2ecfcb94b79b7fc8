"""Build recipe for the native libraries (sm_100a only, in-tree outputs).

    python -m paper_2008_01938_b200.build

produces

* ``_lib/libpipedp_cuda.so`` -- the C ABI of include/pipedp_cuda.h (kernels +
  host planning), CUDA runtime linked statically;
* ``_lib/libpipedp_b200.so`` -- the C++ drop-in for the reference's solver
  entry points (namespace ``pipedp``, include/pipedp/*.hpp), layered on the C
  ABI.

Both are built with ``nvcc -gencode arch=compute_100a,code=sm_100a`` (no
other architecture, no PTX fallback) and land next to the package so gpurun
ships them to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
LIB = os.path.join(PKG, "_lib")
INCLUDE = os.path.join(ROOT, "include")

CUDA_SO = os.path.join(LIB, "libpipedp_cuda.so")
DROPIN_SO = os.path.join(LIB, "libpipedp_b200.so")
PROF_SO = os.path.join(LIB, "libpipedp_cuda_prof.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target: str, sources) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _deps(path, seen=None):
    """path plus every file it #includes with quotes, recursively."""
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    import re
    for inc in re.findall(r'^\s*#\s*include\s+"([^"]+)"', open(path).read(), re.M):
        _deps(os.path.normpath(os.path.join(os.path.dirname(path), inc)), seen)
    return seen


def _sources(d, exts):
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith(exts))


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> None:
    """profile=True builds _lib/libpipedp_cuda_prof.so with the role profiler."""
    os.makedirs(LIB, exist_ok=True)
    nvcc = _nvcc()
    cuda_srcs = _sources(CSRC, (".cu", ".cuh", ".inc", ".hpp")) + [os.path.join(INCLUDE, "pipedp_cuda.h")]
    target = PROF_SO if profile else CUDA_SO
    if force or _newer(target, cuda_srcs):
        # one object per top-level translation unit, compiled in parallel, then
        # one shared library (CUDA runtime linked statically)
        tus = [os.path.join(CSRC, f) for f in ("capi.cu", "engine.cu", "sdp_rank.cu", "sdp_batch_dom.cu", "mcm_tournament.cu", "sdp_cluster.cu", "mcm_batch.cu")]
        flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                 "-Xptxas", "-v" if verbose else "-O3", "-Xcompiler", "-fPIC,-O3",
                 *(["-DPIPEDP_PROFILE"] if profile else []), "-I", INCLUDE]
        objdir = os.path.join(LIB, "obj_prof" if profile else "obj")
        os.makedirs(objdir, exist_ok=True)
        objs = [os.path.join(objdir, os.path.basename(t) + ".o") for t in tus]
        todo = [(t, o) for t, o in zip(tus, objs) if force or _newer(o, sorted(_deps(t)))]
        procs = [(subprocess.Popen([nvcc, *flags, "-c", t, "-o", o], stdout=subprocess.PIPE,
                                   stderr=subprocess.STDOUT, text=True), t) for t, o in todo]
        for p, t in procs:
            out = p.communicate()[0]
            if verbose or p.returncode:
                sys.stdout.write(out)
            if p.returncode:
                raise RuntimeError(f"build failed: nvcc -c {os.path.basename(t)}")
        _run([nvcc, *ARCH, "-shared", "-cudart", "static", *objs, "-o", target + ".tmp"], verbose)
        os.replace(target + ".tmp", target)
    if profile:
        return
    host_srcs = _sources(HOST, (".cpp", ".hpp")) + _sources(os.path.join(INCLUDE, "pipedp"), (".hpp",))
    if force or _newer(DROPIN_SO, host_srcs + [CUDA_SO]):
        cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-shared", "-I", INCLUDE,
               *[s for s in host_srcs if s.endswith(".cpp")],
               "-L", LIB, "-lpipedp_cuda", "-Wl,-rpath,$ORIGIN", "-o", DROPIN_SO + ".tmp"]
        _run(cmd, verbose)
        os.replace(DROPIN_SO + ".tmp", DROPIN_SO)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode:
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv)
