"""Batch driver host logic (paper_2008_01938_b200/batch.py), CPU only:
contiguous sharding, per-shard generation equal to the global generation, and
the rank-ordered digest gather over a world_size-2 gloo group.  The per-shard
tables here come from the CPU checker (the GPU path is covered by
test_gpu_batch.py); what is under test is the partition/gather plumbing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_01938_b200 import batch


def test_shard_range_partitions():
    for total in (0, 1, 7, 64, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            spans = [batch.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        batch.shard_range(10, 2, 2)


def test_shard_generation_matches_global(pd):
    total = 37
    g_offs, g_init = pd.generate_sdp_batch(500, 8, 5, total)
    g_dims = pd.generate_mcm_batch(20, 5, total)
    for world in (2, 4):
        for r in range(world):
            lo, hi = batch.shard_range(total, r, world)
            o, i = pd.generate_sdp_batch(500, 8, 5 + lo, hi - lo)
            assert np.array_equal(o, g_offs[lo:hi]) and np.array_equal(i, g_init[lo:hi])
            assert np.array_equal(pd.generate_mcm_batch(20, 5 + lo, hi - lo), g_dims[lo:hi])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import paper_2008_01938_b200 as pd
    from oracle import pyoracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        orc = pyoracle.load_c()
        lo, hi = batch.shard_range(total, rank, world)
        offs, init = pd.generate_sdp_batch(400, 6, 100 + lo, hi - lo)
        dig = []
        for o, i in zip(offs, init):
            cells, _ = orc.sdp_solve(o, i, 400, "min")
            dig.append(orc.digest(cells))
        local = torch.tensor(np.array(dig, dtype=np.uint64).view(np.int64))
        out = batch.gather_digests(local, total)
        if rank == 0:
            q.put(out.tolist())
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def test_gather_digests_world2_gloo(pd):
    from oracle import pyoracle
    total = 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    orc = pyoracle.load_c()
    offs, init = pd.generate_sdp_batch(400, 6, 100, total)
    want = [orc.digest(orc.sdp_solve(o, i, 400, "min")[0]) for o, i in zip(offs, init)]
    assert got == want
