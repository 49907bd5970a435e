"""Multi-process (one rank per GPU) batched solves over torch.distributed.

The product's multi-GPU path for a job launched with torchrun: each rank owns
the contiguous shard shard_range(total, world, rank) of the instance space
(bmpc_shard_range, the same split bmpc_multi uses inside one process), solves
it with its own launches — no data-path collective, the reference's
independent-solves pool (parallel_sweep, tools/bench.cpp:259-269) — and the
only exchange is the final gather of every shard's packed trajectories to rank
0 (NCCL over NVLink on GPUs; gloo on CPU for the multi-process tests).

Packed layout (the device pack kernel, bmpc_batch_pack_results, and pack_host
below): per instance [x (node * nx) | u (node * nu)], instances in global
order.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import shard_range


def pack_host(x: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Host twin of the device pack kernel: x [count, n, nx], u [count, n, nu]
    -> [count, n * (nx + nu)]."""
    count = x.shape[0]
    return np.concatenate([x.reshape(count, -1), u.reshape(count, -1)], axis=1)


def unpack(packed, count: int, n: int, nx: int, nu: int):
    """Inverse of the pack layout: [count * n * (nx + nu)] -> (x, u)."""
    a = np.asarray(packed, dtype=np.float64).reshape(count, n * (nx + nu))
    return a[:, :n * nx].reshape(count, n, nx), a[:, n * nx:].reshape(count, n, nu)


def gather_packed(local, total: int, per: int, world: int, rank: int, group=None):
    """Gather every rank's packed shard (torch tensor [shard * per]) to rank 0
    and return the [total * per] tensor in global instance order there (None
    elsewhere). Shards may differ by one instance: they travel padded to the
    largest shard (dist.gather needs equal sizes) and are trimmed on rank 0."""
    import torch
    import torch.distributed as dist

    sizes = [shard_range(total, world, g)[1] for g in range(world)]
    cap = max(sizes) * per
    send = local
    if local.numel() < cap:
        send = torch.zeros(cap, dtype=local.dtype, device=local.device)
        send[:local.numel()] = local
    recv = [torch.empty(cap, dtype=local.dtype, device=local.device) for _ in range(world)] if rank == 0 else None
    dist.gather(send, recv, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([recv[g][:sizes[g] * per] for g in range(world)])


class ShardedBatch:
    """This rank's shard of a job of `total` independent instances:
    problems_for(begin, n) builds the shard's problems (global indices
    begin..begin+n-1). solve() launches the shard; gather() packs it on the
    device and gathers every rank's shard to rank 0."""

    def __init__(self, ctx, problems_for, total: int, world: int, rank: int, batch_cls=None, max_records: int = 0):
        from . import Batch

        self.total, self.world, self.rank = total, world, rank
        self.begin, self.count = shard_range(total, world, rank)
        self.problems = problems_for(self.begin, self.count)
        self.batch = (batch_cls or Batch)(ctx, self.problems, max_records=max_records)
        self.n, self.nx, self.nu = self.batch.n, self.batch.nx, self.batch.nu
        self.per = self.n * (self.nx + self.nu)
        self._buf = None

    def set_models(self) -> int:
        return self.batch.set_models()

    def solve(self, options=None):
        self.batch.solve(options)

    def gather(self, device=None, group=None):
        import torch

        if self._buf is None:
            self._buf = torch.empty(self.count * self.per, dtype=torch.float64, device=device)
        self.batch.pack_results(self._buf.data_ptr())
        return gather_packed(self._buf, self.total, self.per, self.world, self.rank, group)
