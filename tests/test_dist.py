"""CPU, world_size 2 over gloo: the product's multi-process batching path
(paper_2506_13624_b200.sharding, what bench.py runs over NCCL for --gpus N):
each rank owns the contiguous shard bmpc_shard_range(total, world, rank) of
the instance space (the C-ABI split bmpc_multi uses too), solves it on its own
(no data-path collective), packs it in the device pack kernel's layout and the
final gather reassembles every instance, in global order, on rank 0 (padded
shards when the split is uneven). The per-instance solve itself needs a GPU,
so the ranks here carry a stand-in batch whose packed rows encode (global
index, node, component); the GPU tests check the real pack kernel writes that
same layout (test_gpu_multi.py)."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, NX, NU = 7, 4, 2


def fake_solution(gidx):
    x = np.array([[gidx * 1000 + k * 10 + j for j in range(NX)] for k in range(N)], np.float64)
    u = -np.array([[gidx * 1000 + k * 10 + j for j in range(NU)] for k in range(N)], np.float64)
    return x, u


class FakeBatch:
    """Stand-in for Batch on a CPU rank: pack_results writes the shard's
    packed rows (sharding.pack_host layout) to the given address."""

    def __init__(self, ctx, problems, max_records=0):
        self.gidx = list(problems)
        self.n, self.nx, self.nu = N, NX, NU

    def set_models(self):
        return 0

    def solve(self, options=None):
        pass

    def pack_results(self, ptr):
        from paper_2506_13624_b200.sharding import pack_host
        xs, us = zip(*[fake_solution(g) for g in self.gidx])
        rows = np.ascontiguousarray(pack_host(np.stack(xs), np.stack(us)))
        ctypes.memmove(ptr, rows.ctypes.data, rows.nbytes)
        return rows.nbytes


def _worker(rank, world, total, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_13624_b200.sharding import ShardedBatch

    sb = ShardedBatch(None, lambda b, n: list(range(b, b + n)), total, world, rank, batch_cls=FakeBatch)
    sb.solve()
    out = sb.gather(device="cpu")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py: max-over-ranks timing
    if rank == 0:
        q.put((out.numpy().copy(), float(t.item()), (sb.begin, sb.count)))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("total", [6, 7])  # even and uneven shards
def test_sharded_solve_and_gather_world2(total):
    from paper_2506_13624_b200.sharding import unpack

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, total, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax, shard0 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    assert shard0 == (0, total // 2)
    x, u = unpack(gathered, total, N, NX, NU)
    for g in range(total):
        xe, ue = fake_solution(g)
        np.testing.assert_array_equal(x[g], xe)
        np.testing.assert_array_equal(u[g], ue)


def test_shards_are_contiguous_disjoint_and_cover():
    import paper_2506_13624_b200 as B

    for total in (1, 7, 4096, 4096 * 8, 12345):
        for world in (1, 2, 3, 4, 8):
            spans = [B.shard_range(total, world, g) for g in range(world)]
            assert spans[0][0] == 0
            for (b0, n0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + n0 == b1
            assert spans[-1][0] + spans[-1][1] == total
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    with pytest.raises(B.BmpcError):
        B.shard_range(10, 2, 2)


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
