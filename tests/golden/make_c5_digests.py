"""Full-config golden digests for BASELINE config 5 (and config 2), produced by
the REFERENCE ITSELF (oracle/_ref, compiled from /root/reference/proj/src by
oracle/Makefile).  Test infrastructure only; run in the build container:

    make -C oracle && python tests/golden/make_c5_digests.py [--threads 8]

Writes, as little-endian uint64 arrays (np.save):

  c5a_cells.npy  table_digest(solve_mcm_sequential(generate_mcm({64, i, 1, 100})))
  c5a_split.npy  table_digest(SolutionTable{cells = split}) of the same solve
  c5b_cells.npy  table_digest(solve_sequential(generate_sdp({2^16, 64, min, i})))

for i in [0, 65536) -- one entry per instance of the batch, in instance order,
every one from the reference's own generator (generate.cpp:21-60), solver
(sdp.cpp:84-89, mcm.cpp:85-110) and digest (table.cpp:12-25).  The C5 batch
tests (tests/test_gpu_batch.py) and bench.py's c5a/c5b parity field compare
the device-computed digests of every instance with these lists.

The reference is single-threaded; instances are spread over a thread pool of
ctypes calls into the reference library (ctypes drops the GIL), the same
harness as bench.py's reference arm for the batch configs.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
TOTAL = 65536
C5A = dict(n=64, lo=1, hi=100)
C5B = dict(n=1 << 16, k=64)


def _c5a(ref, lo, hi):
    cells = np.empty(hi - lo, dtype=np.uint64)
    split = np.empty(hi - lo, dtype=np.uint64)
    for i in range(lo, hi):
        dims = ref.generate_mcm(C5A["n"], i, C5A["lo"], C5A["hi"])
        c, _, s = ref.mcm_solve(dims)
        cells[i - lo] = ref.digest(c)
        split[i - lo] = ref.digest(s)
    return lo, cells, split


def _c5b(ref, lo, hi):
    out = np.empty(hi - lo, dtype=np.uint64)
    for i in range(lo, hi):
        offs, init = ref.generate_sdp(C5B["n"], C5B["k"], i)
        c, _ = ref.sdp_solve(offs, init, C5B["n"], "min")
        out[i - lo] = ref.digest(c)
    return lo, out, None


def run(fn, ref, threads, total=TOTAL, chunk=256):
    a = np.empty(total, dtype=np.uint64)
    b = np.empty(total, dtype=np.uint64)
    with ThreadPoolExecutor(threads) as ex:
        for lo, x, y in ex.map(lambda lo: fn(ref, lo, min(lo + chunk, total)), range(0, total, chunk)):
            a[lo: lo + len(x)] = x
            if y is not None:
                b[lo: lo + len(y)] = y
    return a, b


def list_digest(d: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(d, dtype="<u8").tobytes()).hexdigest()[:16]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--only", choices=["c5a", "c5b"], default=None)
    a = ap.parse_args()
    ref = pyoracle.load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref not built (needs /root/reference): make -C oracle")
    if a.only in (None, "c5a"):
        t = time.time()
        cells, split = run(_c5a, ref, a.threads)
        np.save(os.path.join(HERE, "c5a_cells.npy"), cells)
        np.save(os.path.join(HERE, "c5a_split.npy"), split)
        print(f"c5a: {TOTAL} instances in {time.time() - t:.1f} s, cells {list_digest(cells)} "
              f"split {list_digest(split)}")
    if a.only in (None, "c5b"):
        t = time.time()
        cells, _ = run(_c5b, ref, a.threads)
        np.save(os.path.join(HERE, "c5b_cells.npy"), cells)
        print(f"c5b: {TOTAL} instances in {time.time() - t:.1f} s, cells {list_digest(cells)}")


if __name__ == "__main__":
    main()
