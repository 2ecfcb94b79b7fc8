"""Multi-instance batch driver (no reference
counterpart -- the reference only loops serially over instances in
cmd_bench, commands.cpp:480-507).

One process per GPU (launched by torchrun).  Instance i of a batch of
`total` independent instances is generate_sdp / generate_mcm with seed
`seed0 + i` (generate.cpp:21-60); rank r of W owns the contiguous range
shard_range(total, r, W) and solves it with ONE kernel launch on its own GPU
(sdp_batch_warp / mcm_smem_cta).  There is no collective on the data path: the
per-instance FNV-1a digests (table.cpp:12-25) are computed on the device and
gathered to rank 0 only after timing, for reporting and cross-device-count
parity (the digest list is identical for every W).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import McmPlan, SdpPlan, cell_count, digest_device, generate_mcm_batch, generate_sdp_batch


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced partition [lo, hi) of `total` instances; the first
    total % world ranks get one extra instance."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class SdpBatchSpec:
    """S-DP batch (BASELINE config 5b): n, k, operator, a_1 cap (0: 2k)."""
    total: int = 65536
    n: int = 1 << 16
    k: int = 64
    op: str = "min"
    a1_cap: int = 0
    seed0: int = 0

    def relaxations(self, count: int) -> int:
        a1 = self.a1_cap if self.a1_cap > 0 else 2 * self.k
        return count * (self.n - a1) * self.k  # k per computed cell (commands.cpp:94)

    def table_size(self) -> int:
        return self.n


@dataclass
class McmBatchSpec:
    """MCM batch (BASELINE config 5a): n, dims range."""
    total: int = 65536
    n: int = 64
    dims_min: int = 1
    dims_max: int = 100
    seed0: int = 0

    def relaxations(self, count: int) -> int:
        return count * (self.n ** 3 - self.n) // 6  # D terms per cell, summed

    def table_size(self) -> int:
        return cell_count(self.n) + 1


class BatchShard:
    """This rank's partition of a batch, resident on one GPU.

    Host inputs are generated once; `upload()` copies them to HBM (pinned
    staging), `execute()` launches the solver kernel on `stream`, `digests()`
    hashes every table on the device.  Tensors are torch CUDA tensors (torch is
    the allocator/stream plumbing; every byte of the tables is produced by the
    pipedp kernels)."""

    def __init__(self, spec, rank: int = 0, world: int = 1, device: int = 0):
        import torch
        self.spec, self.rank, self.world, self.device = spec, rank, world, device
        self.lo, self.hi = shard_range(spec.total, rank, world)
        self.count = self.hi - self.lo
        self.dev = torch.device("cuda", device)
        self.sdp = isinstance(spec, SdpBatchSpec)
        if self.sdp:
            offs, init = generate_sdp_batch(spec.n, spec.k, spec.seed0 + self.lo, self.count,
                                            False, spec.a1_cap)
            self.a1 = init.shape[1]
            self.h_offsets, self.h_init = offs, init
            # an empty shard (world > total) has no plan: execute/digests skip it
            self.plan = SdpPlan(self.count, spec.n, spec.k, self.a1, offs.reshape(-1), init.reshape(-1),
                                spec.op, device) if self.count else None
            self.h_in = torch.from_numpy(init.reshape(-1)).pin_memory()
            self.d_in = torch.empty_like(self.h_in, device=self.dev)
            self.d_cells = torch.empty(self.count * spec.n, dtype=torch.int64, device=self.dev)
            self.d_split = None
        else:
            dims = generate_mcm_batch(spec.n, spec.seed0 + self.lo, self.count, spec.dims_min, spec.dims_max)
            self.h_dims = dims
            self.plan = McmPlan(self.count, spec.n, dims.reshape(-1), device=device) if self.count else None
            size = self.count * spec.table_size()
            self.h_in = torch.from_numpy(dims.reshape(-1)).pin_memory()
            self.d_in = None
            self.d_cells = torch.empty(size, dtype=torch.int64, device=self.dev)
            self.d_split = torch.empty(size, dtype=torch.int64, device=self.dev)
        self.d_digest = torch.empty(max(self.count, 1), dtype=torch.int64, device=self.dev)

    # -- data path ------------------------------------------------------------
    def upload(self, stream) -> int:
        """H2D of this shard's per-step inputs; returns the bytes copied."""
        import torch
        with torch.cuda.stream(stream):
            if self.d_in is not None:
                self.d_in.copy_(self.h_in, non_blocking=True)
        return self.h_in.numel() * 8 if self.d_in is not None else 0

    def execute(self, stream) -> None:
        if self.count == 0:
            return
        h = stream.cuda_stream
        if self.sdp:
            self.plan.execute(self.d_in.data_ptr(), self.d_cells.data_ptr(), h)
        else:
            self.plan.execute(self.d_cells.data_ptr(), self.d_split.data_ptr(), h)

    def launches_per_execute(self) -> int:
        return self.plan.describe()[2] if self.count else 0

    def digests(self, stream, split: bool = False):
        """FNV-1a table_digest of every instance's cells (or split) table, on device."""
        if self.count == 0:
            return self.d_digest[:0]
        src = self.d_split if split else self.d_cells
        digest_device(src.data_ptr(), self.spec.table_size(), self.count, self.d_digest.data_ptr(),
                      stream.cuda_stream)
        return self.d_digest[: self.count]

    def relaxations(self) -> int:
        return self.spec.relaxations(self.count)


def gather_digests(local, total: int, group=None) -> Optional[np.ndarray]:
    """All ranks' digests in global instance order on rank 0 (None elsewhere).
    Reporting only -- call after the timed region."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local.cpu().numpy().view(np.uint64).copy()
    world = dist.get_world_size(group)
    width = -(-total // world)  # max shard size
    buf = torch.zeros(width, dtype=torch.int64, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if dist.get_rank(group) != 0:
        return None
    out = []
    for r, p in enumerate(parts):
        lo, hi = shard_range(total, r, world)
        out.append(p[: hi - lo].cpu().numpy())
    return np.concatenate(out).view(np.uint64)
