"""Generate tests/golden/golden.json from the REFERENCE ITSELF (oracle/_ref,
the unmodified reference library compiled from /root/reference/proj/src by
oracle/Makefile).  Run in the build container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixture pins the C restatement (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py) on boxes where the reference is absent.  Every vector is
produced by a reference entry point named next to it:
  apply            SemigroupOp::apply               semigroup.cpp:28-40
  sdp / sdp_full   solve_sequential                 sdp.cpp:84-89
  sdp_validate     validate(SdpInstance)            sdp.cpp:10-32
  sdp_pipeline     solve_sdp_pipeline               sdp_pipeline.cpp:34-44
  gen_sdp/gen_mcm  generate_sdp / generate_mcm      generate.cpp:21-60
  mcm              solve_mcm_sequential (+split)    mcm.cpp:85-110
  mcm_validate     validate(McmInstance)            mcm.cpp:11-28
  mcm_pipeline     solve_mcm_pipeline               mcm_pipeline.cpp:32-47
  lin / coord      lin / coord                      mcm.cpp:30-53
  configs          BASELINE.json configs 1-4 digests (table_digest, table.cpp:12-25)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
OPS = ["min", "max", "saturating-add", "modular-add"]
I64_MAX, I64_MIN = 2**63 - 1, -(2**63)


def hx(d: int) -> str:
    return f"{d:016x}"


def main(skip_big: bool = False) -> None:
    ref = pyoracle.load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref not built (needs /root/reference): make -C oracle")
    g: dict = {"generated_by": "oracle/_ref (reference sources) via tests/golden/make_golden.py"}

    # --- semigroup -------------------------------------------------------
    vals = [0, 1, -1, 2, -2, 5, -7, 2**31 - 2, 2**31 - 1, 2**31, -(2**31), 3 * 2**31 + 5,
            2**62, -(2**62), I64_MAX, I64_MAX - 1, I64_MIN, I64_MIN + 1, 123456789012345]
    g["apply"] = [[op, a, b, ref.apply(op, a, b)] for op in OPS for a in vals for b in vals]

    # --- S-DP --------------------------------------------------------------
    rng = np.random.default_rng(2008_01938)
    sdp_full, sdp = [], []
    kats = [([2, 1], [1, 1], 7, "saturating-add"), ([5, 3, 1], [0] * 5, 10, "min"),
            ([3], [-5, 3000000000, 7], 20, "modular-add"), ([4, 3, 2, 1], [3, 1, 4, 1], 40, "max")]
    for offs, init, n, op in kats:
        cells, _ = ref.sdp_solve(offs, init, n, op)
        sdp_full.append({"offsets": offs, "init": init, "n": n, "op": op, "cells": cells.tolist()})
    for case in range(48):
        op = OPS[case % 4]
        k = int(rng.integers(1, 24))
        cap = int(rng.integers(k, 90))
        offs = sorted(rng.choice(np.arange(1, cap + 1), k, replace=False).tolist(), reverse=True)
        n = int(offs[0] + rng.integers(1, 200))
        kind = case % 3
        if kind == 0:
            init = rng.integers(-(2**62), 2**62, offs[0]).tolist()
        elif kind == 1:
            init = rng.integers(-50, 50, offs[0]).tolist()
        else:
            init = rng.integers(0, 2**20, offs[0]).tolist()
        cells, _ = ref.sdp_solve(offs, init, n, op)
        sdp_full.append({"offsets": offs, "init": init, "n": n, "op": op, "cells": cells.tolist()})
    for (n, k, seed, cons, cap) in [(4096, 64, 1, False, 0), (20000, 1024, 11, False, 4096),
                                    (9000, 300, 5, False, 700), (6000, 200, 3, True, 0),
                                    (1 << 16, 64, 0, False, 0), (1 << 16, 64, 7, False, 0),
                                    (120000, 700, 2, False, 60000)]:
        offs, init = ref.generate_sdp(n, k, seed, cons, cap)
        for op in OPS:
            cells, _ = ref.sdp_solve(offs, init, n, op)
            sdp.append({"gen": [n, k, seed, cons, cap], "op": op, "digest": hx(ref.digest(cells)),
                        "last": int(cells[-1])})
    g["sdp_full"], g["sdp"] = sdp_full, sdp

    g["sdp_validate"] = []
    for offs, il, n in [([5, 3, 1], 5, 16), ([3, 3, 1], 3, 16), ([5, 3, 1], 4, 16), ([5, 3, 0], 5, 16),
                        ([5, -3], 5, 16), ([5, 3, 1], 5, 5), ([5, 3, 1], 5, 6), ([1], 1, 2),
                        ([2, 1, 4], 2, 10), ([], 0, 10), ([7, 6, 4, 3, 2], 7, 7)]:
        g["sdp_validate"].append({"offsets": offs, "init_len": il, "n": n,
                                  "status": ref.sdp_validate(offs, il, n)})

    g["sdp_pipeline"] = []
    for n, k, seed in [(64, 4, 0), (300, 16, 1), (4096, 64, 1)]:
        offs, init = ref.generate_sdp(n, k, seed, False, 0)
        cells, _, steps, first = ref.sdp_pipeline(offs, init, n, "min")
        g["sdp_pipeline"].append({"gen": [n, k, seed], "steps": steps, "first_head": first,
                                  "digest": hx(ref.digest(cells))})

    g["gen_sdp"] = []
    for n, k, seed, cons, cap in [(64, 4, 0, False, 0), (100, 8, 1, False, 0), (5000, 64, 42, False, 0),
                                  (1 << 24, 1024, 1, False, 4096), (1 << 16, 64, 65535, False, 0),
                                  (50, 10, 3, True, 0)]:
        offs, init = ref.generate_sdp(n, k, seed, cons, cap)
        g["gen_sdp"].append({"args": [n, k, seed, cons, cap], "offsets_digest": hx(ref.digest(offs)),
                             "init_digest": hx(ref.digest(init)), "offsets_tail": offs[-12:].tolist(),
                             "a1": int(offs[0])})
    g["gen_mcm"] = []
    for n, seed, lo, hi in [(8, 0, 1, 50), (64, 1, 1, 100), (1024, 1, 1, 100), (8192, 1, 1, 100),
                            (64, 65535, 1, 100)]:
        dims = ref.generate_mcm(n, seed, lo, hi)
        g["gen_mcm"].append({"args": [n, seed, lo, hi], "digest": hx(ref.digest(dims)),
                             "head": dims[:8].tolist()})

    # --- MCM ---------------------------------------------------------------
    g["lin"] = [[r, c, n, ref.lin(r, c, n)] for n in (1, 2, 5, 9) for r in range(1, n + 1)
                for c in range(r, n + 1)]
    g["coord"] = [[a, n, *ref.coord(a, n)] for n in (1, 5, 9) for a in range(1, n * (n + 1) // 2 + 1)]
    mcm = []
    for dims in ([10, 20, 30], [30, 35, 15, 5, 10, 20, 25], [2, 3, 4, 5], [7] * 9, [5, 5]):
        cells, _, split = ref.mcm_solve(dims)
        mcm.append({"dims": dims, "cells": cells.tolist(), "split": split.tolist()})
    for n, seed, lo, hi in [(16, 1, 1, 100), (33, 2, 1, 50), (64, 1, 1, 100), (100, 5, 1, 100),
                            (257, 3, 1, 100), (300, 9, 1000, 1290), (150, 4, 1, 100000),
                            (512, 7, 1, 100), (1024, 1, 1, 100)]:
        dims = ref.generate_mcm(n, seed, lo, hi)
        cells, _, split = ref.mcm_solve(dims)
        mcm.append({"gen": [n, seed, lo, hi], "digest": hx(ref.digest(cells)),
                    "split_digest": hx(ref.digest(split)), "apex": int(cells[-1]),
                    "apex_split": int(split[-1])})
    g["mcm"] = mcm
    g["mcm_validate"] = []
    for dims in ([10, 20], [10], [], [0, 5], [5, -1, 3], [1000000] * 3, [1000001, 2],
                 [1000000] * 4, [1000000] * 10, [1290] * 500, [100000] * 2000):
        g["mcm_validate"].append({"dims": dims if len(dims) <= 10 else None, "dims_len": len(dims),
                                  "fill": dims[0] if dims else None,
                                  "status": ref.mcm_validate(dims)})
    g["mcm_pipeline"] = []
    for n in (2, 3, 4, 5, 8, 17, 32):
        dims = ref.generate_mcm(n, n + 100, 1, 50)
        for mode in (0, 1):
            cells, _, steps, stall, hz = ref.mcm_pipeline(dims, mode, collect_trace=n <= 17)
            g["mcm_pipeline"].append({"gen": [n, n + 100, 1, 50], "mode": mode, "steps": steps,
                                      "stall": stall, "hazard_cells": hz if n <= 17 else None,
                                      "digest": hx(ref.digest(cells))})
    g["hazard_frontier"] = {str(n): ref.hazard_frontier(n).tolist() for n in (3, 4, 5, 8)}

    # --- BASELINE configs ------------------------------------------------------
    cfg = {}
    for op in ("saturating-add", "modular-add"):
        cells, _ = ref.sdp_solve([2, 1], [1, 1], 1 << 20, op)
        cfg[f"c1_{op}"] = {"digest": hx(ref.digest(cells)), "last": int(cells[-1])}
    dims = ref.generate_mcm(64, 1, 1, 100)
    cells, _, split = ref.mcm_solve(dims)
    cfg["mcm64"] = {"digest": hx(ref.digest(cells)), "split_digest": hx(ref.digest(split)),
                    "apex": int(cells[-1])}
    if not skip_big:
        t0 = time.time()
        offs, init = ref.generate_sdp(1 << 24, 1024, 1, False, 4096)
        cells, _ = ref.sdp_solve(offs, init, 1 << 24, "min")
        cfg["c2"] = {"digest": hx(ref.digest(cells)), "last": int(cells[-1]),
                     "ref_seconds": round(time.time() - t0, 2)}
        # prefix property used by the bench: the first 2^22 cells of C2
        cfg["c2_prefix22"] = {"digest": hx(ref.digest(cells[: 1 << 22]))}
    # SURVEY.md 8c (n=8192 took 48 min on one core; recorded, not recomputed)
    cfg["c4_survey"] = {"digest": "cc41fd2d4975b51b", "split_digest": "f9e2c86f904b28e1",
                        "apex": 21215156}
    g["configs"] = cfg
    with open(OUT, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main(skip_big="--skip-big" in sys.argv)
