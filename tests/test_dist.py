"""CPU, world_size 2 over gloo: the multi-GPU batching contract of bench.py —
each rank owns a contiguous slice of the instance space (seeds 42 + rank *
count + i), solves it independently (no data-path collective), and the final
gather concatenates every rank's packed [x | u] on rank 0 in rank order. The
solver here is the CPU oracle (the product path needs a GPU); the partition
and gather logic is the same code shape bench.py runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

COUNT = 2


def shard_seeds(rank, count):
    return [42 + rank * count + i for i in range(count)]


def packed_solutions(seeds):
    import _oracle as O
    import paper_2506_13624_b200 as B
    out = []
    for s in seeds:
        p = B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2, perturb_seed=s)
        r = O.solve_problem(p)
        out.append(np.concatenate([r["x"].ravel(), r["u"].ravel()]))
    return np.stack(out)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = torch.from_numpy(packed_solutions(shard_seeds(rank, COUNT)))
    recv = [torch.empty_like(local) for _ in range(world)] if rank == 0 else None
    dist.gather(local, recv, dst=0)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py: max-over-ranks timing
    if rank == 0:
        q.put((torch.cat(recv).numpy(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_solve_and_gather_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    expect = packed_solutions([s for r in range(world) for s in shard_seeds(r, COUNT)])
    np.testing.assert_array_equal(gathered, expect)


def test_shards_are_disjoint_and_cover():
    for world in (1, 2, 4, 8):
        seeds = [s for r in range(world) for s in shard_seeds(r, 4096)]
        assert len(set(seeds)) == len(seeds) == world * 4096
        assert min(seeds) == 42 and max(seeds) == 42 + world * 4096 - 1


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
