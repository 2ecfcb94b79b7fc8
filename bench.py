#!/usr/bin/env python
"""bench.py -- pipedp-b200 benchmark (BASELINE.json metric: DP relaxations/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

One process per GPU.  Under torchrun (WORLD_SIZE set) every process is one
rank; `--gpus N` without torchrun starts the N ranks itself (127.0.0.1
rendezvous).  NCCL carries only the barrier, the max-over-ranks timing
reduction and the post-timing digest gather (gloo when ranks share a GPU);
the data path has no collective.

Default workload: c2 at N = 1 (BASELINE's headline single instance), the
sharded c5b batch at N > 1 (the only configuration that shards, SURVEY.md
8e), with a c5a companion measurement in the same line.

Workloads (BASELINE.json configs; inputs from the reference's own seeded
generators, generate.cpp:21-60, restated bit-exactly in the C ABI):
  c1   S-DP Fibonacci n=2^20, offsets {2,1}, saturating-add, init {1,1}
  c2   S-DP n=2^24, k=1024, a_1=4096, min, seed 1           (default at N = 1, the headline)
  c3   MCM n=1024, dims U[1,100], seed 1 (pipeline kernel; --mcm-kernel tournament for the paper's method)
  c4   MCM n=8192, dims U[1,100], seed 1 (table in HBM)
  c5a  65,536 x MCM n=64 (batch, sharded over ranks)
  c5b  65,536 x S-DP n=2^16, k=64, min (batch, sharded over ranks; default at N > 1)
Single-instance workloads (c1-c4) cannot be split (every cell depends on its
predecessors): at N > 1 every rank solves its own instance
(seed 1 + rank), i.e. a batch of N independent instances, one per GPU -- weak
scaling.  c5a/c5b shard a fixed batch of 65,536 instances -- strong scaling.

A "step" is one solve of the workload on inputs already resident in HBM
(`value`); `e2e` repeats it through the reference-facing C-ABI call with HOST
buffers (H2D of offsets/init or dims and D2H of every table inside the timed
region).  L2 (126 MB) is flushed by writing a 256 MiB buffer before every
timed step.  The CPU baseline is the reference library itself
(oracle/_ref, compiled from the reference sources) on the box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DP relaxations/sec (S-DP, MCM n=1024/8192) and % of roofline vs CPU ref"
UNIT = "relaxations/s"

WORKLOADS = {
    "c1": "S-DP Fibonacci n=2^20 k=2 offsets{2,1} saturating-add init{1,1}",
    "c2": "S-DP n=2^24 k=1024 a1=4096 min seed1",
    "c3": "MCM n=1024 dims U[1,100] seed1 (+split table)",
    "c4": "MCM n=8192 dims U[1,100] seed1 (+split table, table in HBM)",
    "c5a": "batch 65536 x MCM n=64 dims U[1,100] (+split)",
    "c5b": "batch 65536 x S-DP n=2^16 k=64 a1=128 min",
}
BATCH = {"c5a", "c5b"}


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v else default


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi samples of SM clock and throttle reasons while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a moment to start: have the first sample in hand
            # before the timed region (sub-millisecond steps end before it)
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) == 6:
                self.rows.append(f)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# -------------------------------------------------------------- workloads ---
class Single:
    """One instance per rank (c1-c4), device-resident plan + buffers."""

    def __init__(self, pd, torch, name, rank, dev, mcm_kernel):
        self.pd, self.torch, self.name = pd, torch, name
        seed = 1 + rank
        self.seed = seed
        self.dev = torch.device("cuda", dev)
        if name in ("c1", "c2"):
            if name == "c1":
                self.inst = pd.SdpInstance(1 << 20, [2, 1], [1, 1], "saturating-add")
            else:
                self.inst = pd.generate_sdp(n=1 << 24, k=1024, op="min", seed=seed, a1_cap=4096)
            i = self.inst
            self.relax = (i.n - i.a1) * i.k
            self.plan = pd.SdpPlan(1, i.n, i.k, i.a1, i.offsets, i.init, i.op, dev)
            self.d_init = torch.tensor(list(map(int, i.init)), dtype=torch.int64, device=self.dev)
            self.d_cells = torch.empty(i.n, dtype=torch.int64, device=self.dev)
            self.out_bytes = i.n * 8
            self.in_bytes = (i.k + i.a1) * 8
            self.table_cells = i.n
        else:
            n = 1024 if name == "c3" else 8192
            self.inst = pd.generate_mcm(n=n, seed=seed, dims_min=1, dims_max=100)
            self.kernel = {"pipeline": pd.MCM_AUTO, "wavefront": pd.MCM_WAVEFRONT,
                           "tournament": pd.MCM_TOURNAMENT, "tiled": pd.MCM_TILED}[mcm_kernel]
            self.relax = (n ** 3 - n) // 6
            self.plan = pd.McmPlan(1, n, self.inst.dims, self.kernel, dev)
            size = pd.cell_count(n) + 1
            self.d_cells = torch.empty(size, dtype=torch.int64, device=self.dev)
            self.d_split = torch.empty(size, dtype=torch.int64, device=self.dev)
            self.out_bytes = 2 * size * 8
            self.in_bytes = (n + 1) * 8
            self.table_cells = size

    def execute(self, stream):
        if self.name in ("c1", "c2"):
            self.plan.execute(self.d_init.data_ptr(), self.d_cells.data_ptr(), stream.cuda_stream)
        else:
            self.plan.execute(self.d_cells.data_ptr(), self.d_split.data_ptr(), stream.cuda_stream)

    def launches(self):
        return max(1, self.plan.describe()[2])

    def kernel_name(self):
        return self.plan.describe()[0]

    def value_bits(self):
        return self.plan.describe()[1]

    def e2e_step(self):
        """The reference-facing call with host buffers (C ABI pipedp_*_solve)."""
        pd = self.pd
        if self.name in ("c1", "c2"):
            t = pd.solve_sequential(self.inst)
            return t.cells
        t, split = pd.solve_mcm_with_split(self.inst, self.kernel)
        return t.cells

    def e2e_bytes(self):
        return self.in_bytes, self.out_bytes

    def digest(self):
        return self.pd.table_digest(self.d_cells.cpu().numpy())


class Batch:
    def __init__(self, pd, torch, name, rank, world, dev):
        from paper_2008_01938_b200 import batch as B
        self.pd, self.torch, self.name = pd, torch, name
        spec = B.McmBatchSpec() if name == "c5a" else B.SdpBatchSpec()
        self.spec = spec
        self.shard = B.BatchShard(spec, rank, world, dev)
        self.shard.upload(torch.cuda.current_stream())  # the shard's init cells into HBM (once)
        torch.cuda.synchronize()
        self.relax = self.shard.relaxations()
        n = spec.n
        if name == "c5a":
            self.out_bytes = 2 * self.shard.count * (pd.cell_count(n) + 1) * 8
            self.in_bytes = self.shard.count * (n + 1) * 8
        else:
            self.out_bytes = self.shard.count * n * 8
            self.in_bytes = self.shard.count * (spec.k + self.shard.a1) * 8

    def execute(self, stream):
        self.shard.execute(stream)

    def launches(self):
        return self.shard.launches_per_execute()

    def kernel_name(self):
        return self.shard.plan.describe()[0]

    def value_bits(self):
        return self.shard.plan.describe()[1]

    def e2e_step(self):
        import numpy as np
        pd, s = self.pd, self.shard
        L = pd.lib()
        if self.name == "c5b":
            cells = np.empty(s.count * self.spec.n, dtype=np.int64)
            pd._check(L.pipedp_sdp_solve_batch(s.count, self.spec.n, self.spec.k, s.a1,
                                               pd._p(s.h_offsets.reshape(-1)), pd._p(s.h_init.reshape(-1)),
                                               0, pd._p(cells), s.device))
            return cells
        size = s.count * (pd.cell_count(self.spec.n) + 1)
        cells = np.empty(size, dtype=np.int64)
        split = np.empty(size, dtype=np.int64)
        pd._check(L.pipedp_mcm_solve_batch(s.count, self.spec.n, pd._p(s.h_dims.reshape(-1)),
                                           pd._p(cells), pd._p(split), s.device))
        return cells

    def e2e_bytes(self):
        return self.in_bytes, self.out_bytes


# ----------------------------------------------------------- CPU baselines ---
def cpu_reference_sample(name, threads, steps=1):
    """The reference library (oracle/_ref) on a bounded sample of the workload.
    Returns (relax/s, cores, kind, sample description, seconds)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import pyoracle
    ref = pyoracle.load_ref()
    kind = "reference"
    if ref is None:  # reference sources absent at build time: the C restatement
        ref, kind = pyoracle.load_c(), "port"
    jobs = []  # (callable, relaxations)
    if name == "c1":
        reps = 100
        jobs = [(lambda: ref.sdp_solve([2, 1], [1, 1], 1 << 20, "saturating-add"), (2**20 - 2) * 2)] * reps
        sample = f"{reps} x full c1 instance, solve_sequential (sdp.cpp:84)"
        threads = 1
    elif name == "c2":
        offs, init = ref.generate_sdp(1 << 24, 1024, 1, False, 4096)
        n = 1 << 23
        jobs = [(lambda: ref.sdp_solve(offs, init, n, "min"), (n - 4096) * 1024)]
        sample = "first 2^23 cells of the c2 instance (same offsets/init), solve_sequential (sdp.cpp:84), 1 thread"
        threads = 1
    elif name in ("c3", "c4"):
        n = 1024 if name == "c3" else 1536
        dims = ref.generate_mcm(n, 1, 1, 100)
        jobs = [(lambda: ref.mcm_solve(dims), (n**3 - n) // 6)]
        sample = (f"MCM n={n} seed 1 dims U[1,100], solve_mcm_sequential with split (mcm.cpp:85), 1 thread"
                  + ("; n=8192 takes ~48 min, so n=1536 stands in" if name == "c4" else ""))
        threads = 1
    elif name == "c5a":
        cnt = 4096
        dims = [ref.generate_mcm(64, i, 1, 100) for i in range(cnt)]
        jobs = [((lambda d=d: ref.mcm_solve(d)), (64**3 - 64) // 6) for d in dims]
        sample = f"{cnt} of the 65,536 c5a instances, solve_mcm_sequential, {threads}-thread pool"
    else:
        cnt = 512
        insts = [ref.generate_sdp(1 << 16, 64, i, False, 0) for i in range(cnt)]
        jobs = [((lambda o=o, i=i: ref.sdp_solve(o, i, 1 << 16, "min")), ((1 << 16) - 128) * 64) for o, i in insts]
        sample = f"{cnt} of the 65,536 c5b instances, solve_sequential, {threads}-thread pool"
    relax = sum(r for _, r in jobs)
    t0 = time.perf_counter()
    for _ in range(steps):
        if threads == 1:
            for f, _ in jobs:
                f()
        else:
            with ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
                list(ex.map(lambda j: j[0](), jobs))
    dt = time.perf_counter() - t0
    return relax * steps / dt, threads, kind, sample, dt


def traffic_for(name):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/ncu_summary.json), or None."""
    s = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {}
    e = s.get(name)
    return e.get("dram_bytes_per_launch") if isinstance(e, dict) else None


# ------------------------------------------------------------ launching ---
def spawn_ranks(n):
    """`--gpus N` without torchrun: start N ranks of this script (one per GPU,
    or sharing the visible GPUs round-robin) with a 127.0.0.1 rendezvous; only
    rank 0's stdout is the bench line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


# --------------------------------------------------------------------- main ---
class Ranks:
    """Process-group plumbing: barrier and scalar reductions.  NCCL when every
    rank has its own GPU, gloo when ranks share one (a 1-GPU box running
    `--gpus 2`)."""

    def __init__(self, torch, world, rank, device):
        import torch.distributed as dist
        self.torch, self.dist, self.world, self.rank = torch, dist, world, rank
        self.backend = None
        if world > 1:
            shared = torch.cuda.device_count() < world
            self.backend = "gloo" if shared else "nccl"
            kw = {} if shared else {"device_id": torch.device("cuda", device)}
            dist.init_process_group(self.backend, **kw)
        self.dev = "cpu" if self.backend == "gloo" else "cuda"

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, x, op):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x):
        return self.reduce(x, self.dist.ReduceOp.MAX) if self.world > 1 else x

    def sum(self, x):
        return self.reduce(x, self.dist.ReduceOp.SUM) if self.world > 1 else x

    def gather_digests(self, local, total):
        """Per-instance digests of every rank in global instance order (rank 0)."""
        import numpy as np
        from paper_2008_01938_b200 import batch as B
        if self.world == 1:
            return local.cpu().numpy().view(np.uint64).copy()
        src = local.cpu() if self.dev == "cpu" else local
        out = B.gather_digests(src, total)
        return None if out is None else np.asarray(out).view(np.uint64)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def golden_batch_digests(name):
    import numpy as np
    here = os.path.join(ROOT, "tests", "golden")
    try:
        if name == "c5a":
            return np.load(os.path.join(here, "c5a_cells.npy")), np.load(os.path.join(here, "c5a_split.npy"))
        return np.load(os.path.join(here, "c5b_cells.npy")), None
    except OSError:
        return None, None


def measure(pd, torch, R, name, args, rank, world, local, flush, with_e2e=True):
    """Warm up, time K steps (device events, max over ranks), check parity,
    then the end-to-end C-ABI leg.  Returns the per-workload record."""
    single = name not in BATCH
    W = Batch(pd, torch, name, rank, world, local) if not single else Single(pd, torch, name, rank, local,
                                                                               args.mcm_kernel)
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 0)):
        flush.zero_()
        W.execute(stream)
    torch.cuda.synchronize()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    phased = single and W.name == "c2" and W.kernel_name().startswith("sdp_chunked")
    if phased:  # per-phase CUDA events on the execute stream (pipedp_sdp_plan_set_timing)
        W.plan.set_timing(True)
    R.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            W.execute(stream)
            e1.record(stream)
        torch.cuda.synchronize()
    R.barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    kernel_ms = sum(step_ms)
    phases = None
    if phased:
        (p_pow, p_chain, p_chunks), runs = W.plan.phase_ms()
        W.plan.set_timing(False)
        if runs:
            phases = {"matrix_powers_ms": p_pow / runs, "entry_chain_ms": p_chain / runs,
                      "chunk_batch_ms": p_chunks / runs, "runs": runs,
                      "source": "CUDA events on the execute stream inside the timed steps"}
    kernel_ms_max = R.max(kernel_ms)
    relax_total = R.sum(float(W.relax))
    value = relax_total * K / (kernel_ms_max / 1e3)

    # parity of the benchmarked output (after timing): single instances by the
    # reference's table digest of the seed-1 instance, batches by every
    # instance's device digest against the reference-generated lists
    parity = None
    if single:
        if rank == 0:
            golden = load_json(os.path.join(ROOT, "tests", "golden", "golden.json")) or {}
            want = {"c1": golden.get("configs", {}).get("c1_saturating-add", {}).get("digest"),
                    "c2": golden.get("configs", {}).get("c2", {}).get("digest"),
                    "c3": "9e31907a82260f66", "c4": "cc41fd2d4975b51b"}.get(name)
            got = f"{W.digest():016x}"
            parity = {"cells_digest": got, "golden": want, "match": (got == want) if want else None}
    else:
        import numpy as np
        cells = R.gather_digests(W.shard.digests(stream), W.spec.total)
        split = R.gather_digests(W.shard.digests(stream, split=True), W.spec.total) if name == "c5a" else None
        if rank == 0:
            want_c, want_s = golden_batch_digests(name)
            if want_c is None:
                parity = {"match": None, "note": "golden digest lists absent"}
            else:
                bad = int(np.count_nonzero(cells != want_c))
                if split is not None:
                    bad += int(np.count_nonzero(split != want_s))
                parity = {"instances": int(cells.size), "tables_checked": int(cells.size) * (2 if split is not None else 1),
                          "mismatches": bad, "match": bad == 0,
                          "golden": "tests/golden/%s (reference, make_c5_digests.py)" %
                                    ("c5a_cells.npy+c5a_split.npy" if name == "c5a" else "c5b_cells.npy")}

    e2e = None
    if with_e2e:
        ek = args.e2e_steps if args.e2e_steps is not None else max(K, 5)  # host-side timings are noisy: >= 5 steps
        if ek:
            W.e2e_step()  # warm-up: staging buffers, copy pool, cached plan / device buffers
        R.barrier()
        t0 = time.perf_counter()
        for _ in range(ek):
            W.e2e_step()
        e2e_s = R.max(time.perf_counter() - t0)
        h2d, d2h = W.e2e_bytes()
        e2e = {"value": relax_total * ek / e2e_s if ek else None, "unit": UNIT,
               "h2d_bytes_per_step": int(R.sum(h2d)), "d2h_bytes_per_step": int(R.sum(d2h)),
               "steps": ek, "ms_per_step": e2e_s * 1e3 / max(ek, 1),
               "call": "pipedp_sdp_solve / pipedp_mcm_solve (C ABI, host buffers)" if single
               else "pipedp_sdp_solve_batch / pipedp_mcm_solve_batch (C ABI, host buffers)"}
    rec = {"W": W, "value": value, "kernel_ms": kernel_ms, "kernel_ms_max": kernel_ms_max, "K": K,
           "step_ms": step_ms, "parity": parity, "e2e": e2e, "clocks": clk.summary(),
           "launches": W.launches() * K, "kernel": W.kernel_name(), "bits": W.value_bits(), "phases": phases}
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: c2 at N = 1, c5b (+ c5a companion) at N > 1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mcm-kernel", default="pipeline", choices=["pipeline", "tiled", "wavefront", "tournament"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-companion", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    name = args.workload or ("c2" if world == 1 else "c5b")
    single = name not in BATCH
    config = {"workload": f"{name}: {WORKLOADS[name]}", "n_instances": world if single else 65536,
              "parallelism": (f"replicas{world}" if single else f"shard{world}"),
              "l2": "flushed (256 MiB write) before every timed step"}
    if name in ("c3", "c4"):
        config["mcm_kernel"] = args.mcm_kernel

    if args.impl == "reference":
        if rank != 0:
            return
        cores = os.cpu_count() or 1
        thr = 1 if single else cores
        cpu_reference_sample(name, thr, 1)  # warm-up sample
        v, thr, kind, sample, dt = cpu_reference_sample(name, thr, max(1, args.steps))
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3 / max(1, args.steps),
                "higher_is_better": True, "scaling": "weak" if single else "strong",
                "vs_baseline": None, "dtype": "int64", "data": "synthetic (reference generators)",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": kind, "sample": sample},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2008_01938_b200 as pd

    ndev = max(torch.cuda.device_count(), 1)
    local = local % ndev
    torch.cuda.set_device(local)
    R = Ranks(torch, world, rank, local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    rec = measure(pd, torch, R, name, args, rank, world, local, flush)
    companion = None
    if world > 1 and args.workload is None and not args.no_companion:
        del rec["W"].shard  # free the c5b tables before the companion batch
        torch.cuda.empty_cache()
        c = measure(pd, torch, R, "c5a", args, rank, world, local, flush, with_e2e=False)
        companion = {"workload": f"c5a: {WORKLOADS['c5a']}", "value": c["value"], "unit": UNIT,
                     "ms_per_step": c["kernel_ms_max"] / c["K"], "kernel": c["kernel"],
                     "parity": c["parity"], "gpu_launches": c["launches"]}
    W, K = rec["W"], rec["K"]
    kernel_ms, kernel_ms_max = rec["kernel_ms"], rec["kernel_ms_max"]

    if rank != 0:
        R.close()
        return

    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (burst copy)" if hbm_peak else "fallback 6650 GB/s (B200_PROFILING.md)"
    hbm_peak = hbm_peak or 6650.0
    avg_ms = kernel_ms / K
    alg_bytes = W.in_bytes + W.out_bytes
    # the dominant kernel's own launch time where the step has several phases
    # (C2: the chunk batch writes the whole table; events on its stream)
    dom_ms = (rec["phases"] or {}).get("chunk_batch_ms") or avg_ms
    achieved = alg_bytes / (dom_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic_for(name), "peak_source": peak_src,
                "kernel": rec["kernel"], "algorithmic_bytes_per_launch": alg_bytes,
                "avg_launch_ms": dom_ms, "step_ms": avg_ms}
    extra = {}
    if name in ("c1", "c2"):
        i = W.inst
        bits = W.value_bits()
        op_ns, op_cyc = pd.op_latency_ns(i.op, bits, local)
        hand_ns, _ = pd.chain_step_ns(i.op, bits, local) if (i.op, bits) != ("saturating-add", 32) else (None, None)
        kname = rec["kernel"]
        # north_star's dependency-chain bound: one output per step (a_k = 1),
        # n - a_1 steps, each the measured latency of one dependent (x).  The
        # chunked / jump paths regroup the recurrence algebraically, so they
        # are not bound by it (frac > 1 = faster than any one-cell-per-step
        # pipeline); their own critical path is reported next to it.
        steps = i.n - i.a1
        floor_ms = steps * op_ns / 1e6
        extra["chain_roofline"] = {
            "definition": "(n - a_1) dependent steps x latency of one dependent (x) (north_star)",
            "steps": steps, "t_op_ns": op_ns, "t_op_cycles": op_cyc, "floor_ms": floor_ms,
            "achieved_ms": avg_ms, "frac": floor_ms / avg_ms, "t_warp_handoff_ns": hand_ns,
            "value_bits": bits}
        if kname.startswith("sdp_chunked"):
            import re
            m = re.search(r"L=(\d+),G=(\d+)", kname)
            L, G = (int(m.group(1)), int(m.group(2))) if m else (i.n - i.a1, 1)
            extra["chain_roofline"]["critical_path"] = {
                "definition": "sdp_chunked: one chunk (L cells) + G entry-state steps", "steps": L + G,
                "floor_ms": (L + G) * op_ns / 1e6}
            # the binding resource of the chunk batch (the step's dominant
            # kernel, timed by its own events): shared-memory bandwidth,
            # 128 B/cycle/SM.  The rank kernel (chunk_rank_kernel) reads one
            # 4-byte u16x2 word per TWO relaxations (2 B each); the generic
            # chunk pipeline one 4-byte operand per relaxation.
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            sm_clk = (rec["clocks"] or {}).get("sm_mhz") or 1965.0
            smem_gbs = sms * 128 * sm_clk * 1e6 / 1e9
            bpr = 2 if "chunk_rank" in kname else 4
            relax_bytes = (i.n - i.a1) * i.k * bpr
            chunk_ms = (rec["phases"] or {}).get("chunk_batch_ms") or avg_ms
            extra["relaxation_roofline"] = {
                "bound": "shared-memory bandwidth (LSU), %d B of operand per relaxation" % bpr,
                "kernel": "chunk_rank_kernel" if bpr == 2 else "sdp_pipeline_cta",
                "bytes": relax_bytes, "peak_gbs": smem_gbs, "floor_ms": relax_bytes / smem_gbs / 1e6,
                "achieved_ms": chunk_ms, "frac": relax_bytes / smem_gbs / 1e6 / chunk_ms,
                "step_ms": avg_ms, "chunks": G, "chunk_cells": L}
            if rec["phases"]:
                extra["phases"] = rec["phases"]
        elif kname == "sdp_jump":
            nseg = -(-(i.n - i.a1) // 64)
            cp = 64 + max(1, (nseg - 1).bit_length())
            extra["chain_roofline"]["critical_path"] = {
                "definition": "sdp_jump: 64-cell segment chain + log2(segments) entry-state levels",
                "steps": cp, "floor_ms": cp * op_ns / 1e6}
    if name in ("c3", "c4"):
        n = W.inst.n
        extra["mcm_steps"] = {"cells": n * (n - 1) // 2, "ns_per_cell": avg_ms * 1e6 / (n * (n - 1) // 2),
                              "diagonals": n - 1, "us_per_diagonal": avg_ms * 1e3 / (n - 1)}
    if companion:
        extra["companion"] = companion

    R.close()  # the CPU baseline below runs on rank 0 alone, after every collective
    cpu = None
    if not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        v, thr, kind, sample, _ = cpu_reference_sample(name, 1 if single else cores, 1)
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": kind, "sample": sample}

    line = {"metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": kernel_ms_max / K, "higher_is_better": True,
            "scaling": "weak" if single else "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (the reference's seeded generators, generate.cpp:21-60)",
            "config": config, "e2e": rec["e2e"], "gpu_launches": rec["launches"],
            "roofline": roofline, "cpu_baseline": cpu, "clocks": rec["clocks"],
            "kernel_value_bits": rec["bits"], "parity": rec["parity"], "step_ms": rec["step_ms"],
            "process_group": R.backend, **extra}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
