"""Multi-device batched solves through the library (bmpc_multi_*): several
contexts, contiguous shards, concurrent launches, and the final gather into
one device buffer (the pack kernel storing straight into the first context's
device memory). On a one-GPU box the contexts share device 0 — every shard's
kernels are independent (no cross-shard waiting), so this is the same code
path a multi-GPU node runs, minus the peer mapping."""
import numpy as np
import pytest
import torch

import paper_2506_13624_b200 as B
from paper_2506_13624_b200.sharding import pack_host, unpack

pytestmark = pytest.mark.gpu


def test_multi_matches_single_batch_and_gathers():
    spec = B.intersection_spec(63, 10.0, 0.1)
    probs = [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + i) for i in range(48)]
    ctxs = [B.Context(0), B.Context(0), B.Context(0)]
    mb = B.MultiBatch(ctxs, probs)
    assert [mb.shard(g) for g in range(3)] == [(0, 16), (16, 16), (32, 16)]
    mb.set_models()
    mb.solve()
    x = np.zeros((48, mb.n, mb.nx))
    u = np.zeros((48, mb.n, mb.nu))
    reps, _ = mb.results(x, u)
    single = B.Batch(B.Context(0), probs)
    single.set_models()
    single.solve()
    xs = np.zeros_like(x)
    us = np.zeros_like(u)
    reps_s, _ = single.results(xs, us)
    assert [r.inner_iterations for r in reps] == [r.inner_iterations for r in reps_s]
    np.testing.assert_array_equal(x, xs)  # same kernels, same launch shape per instance
    np.testing.assert_array_equal(u, us)
    dst = torch.empty(48 * mb.n * (mb.nx + mb.nu), dtype=torch.float64, device="cuda:0")
    nbytes = mb.gather(dst.data_ptr())
    assert nbytes == dst.numel() * 8
    packed = dst.cpu().numpy()
    np.testing.assert_array_equal(packed.reshape(48, -1), pack_host(x, u))
    xg, ug = unpack(packed, 48, mb.n, mb.nx, mb.nu)
    np.testing.assert_array_equal(xg, x)
    np.testing.assert_array_equal(ug, u)


def test_solve_batch_one_shot_and_uneven_shards():
    spec = B.intersection_spec(20, 4.0, 0.4)
    probs = [B.build_intersection_case(spec, 2, 2, perturb_seed=7 + i) for i in range(5)]
    mb = B.MultiBatch([B.Context(0), B.Context(0)], probs)
    assert [mb.shard(g) for g in range(2)] == [(0, 2), (2, 3)]
    mb.set_models()
    mb.solve()
    reps, _ = mb.results()
    for p, r in zip(probs, reps):
        ref = B.solve(p, ctx=B.Context(0))
        assert r.inner_iterations == ref.report.inner_iterations
        assert r.status == ref.report.status
