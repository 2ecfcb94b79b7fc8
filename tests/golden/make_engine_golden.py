"""Generate tests/golden/engine_golden.json from the REFERENCE ITSELF
(oracle/_ref): the lock-step engine's trace and analysis reports for
solve_mcm_pipeline (both McmMode values) and solve_sdp_pipeline, each with
its default collect_trace = true, reduced to the digest vector of
ref_mcm_engine_digests / ref_sdp_engine_digests (oracle/ref_shim.cpp):

  [0] steps_executed  [1] stall_iterations  [2] first_head  [3] records
  [4] D(records)  [5] max_group_size  [6] conflict groups  [7] D(groups)
  [8] D(per_step_cost)  [9] hazards  [10] D(hazards)  [11] stall heads
  [12] D(stall heads)  [13] D(table cells)

D = table_digest (table.cpp:12-25) of the flattened int64 sequence.  Run in the
build container:  make -C oracle && python tests/golden/make_engine_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "engine_golden.json")

# (n, seed, dims_lo, dims_hi); all-equal dims included (every term ties)
MCM = [(2, 1, 1, 50), (3, 2, 1, 50), (4, 3, 1, 50), (5, 4, 1, 50), (8, 5, 1, 50), (13, 6, 1, 100),
       (24, 7, 1, 100), (40, 8, 1, 100), (64, 9, 1, 100), (16, 10, 7, 7)]
# (n, k, seed, op, consecutive, a1_cap)
SDP = [(300, 8, 3, "min", False, 0), (500, 16, 4, "max", False, 0), (400, 12, 5, "min", True, 0),
       (700, 24, 6, "modular-add", False, 40), (350, 6, 7, "saturating-add", True, 0),
       (2000, 64, 8, "min", False, 128)]


def main() -> None:
    ref = pyoracle.load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref not built (needs /root/reference): make -C oracle")
    g = {"generated_by": "oracle/_ref (reference sources) via tests/golden/make_engine_golden.py",
         "mcm": [], "sdp": [], "fib": None}
    for n, seed, lo, hi in MCM:
        dims = ref.generate_mcm(n, seed, lo, hi)
        for mode in (0, 1):
            t = time.time()
            d = ref.mcm_engine_digests(dims, mode)
            g["mcm"].append({"gen": [n, seed, lo, hi], "mode": mode, "digests": [f"{x:016x}" for x in d]})
            print(f"mcm n={n} mode={mode} records={d[3]} hazards={d[9]} groups={d[6]} {time.time() - t:.2f}s")
    for n, k, seed, op, cons, cap in SDP:
        offs, init = ref.generate_sdp(n, k, seed, cons, cap)
        d = ref.sdp_engine_digests(offs, init, n, op)
        g["sdp"].append({"gen": [n, k, seed, cons, cap], "op": op, "digests": [f"{x:016x}" for x in d]})
        print(f"sdp n={n} k={k} {op} records={d[3]} groups={d[6]} max={d[5]}")
    d = ref.sdp_engine_digests([2, 1], [1, 1], 90, "saturating-add")  # SPEC.md:71 Fibonacci
    g["fib"] = {"n": 90, "digests": [f"{x:016x}" for x in d]}
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)
    # the reference's own callers (commands.cpp) linked with the reference's
    # solvers: expected stdout of tests/cpp/ref_callers_main.cpp (msec dropped)
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "ref_callers_ref")
    for mode in ("run", "verify"):
        out = subprocess.run([exe, mode], capture_output=True, text=True, check=True).stdout
        keep = "".join(l + "\n" for l in out.splitlines() if not l.startswith("msec:"))
        path = os.path.join(os.path.dirname(OUT), f"ref_callers_{mode}.txt")
        with open(path, "w") as f:
            f.write(keep)
        print("wrote", path)


if __name__ == "__main__":
    main()
