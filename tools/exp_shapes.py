"""Experiment: grid-barrier cost; single-instance latency vs block size;
batch throughput vs block shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_13624_b200 as B

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = B.Context(0, stream=s.cuda_stream)
for blocks, threads in [(148, 256), (296, 256), (148, 128), (148, 1024)]:
    print("grid sync", blocks, threads, "%.2f us" % B.debug_grid_sync_us(blocks, threads, 2000, ctx), flush=True)


def timed(bt):
    bt.solve()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    bt.solve()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)
bt = B.Batch(ctx, [p])
bt.set_models()
for shape in [(256, 1), (512, 1), (1024, 1), (256, 2)]:
    bt.set_launch(*shape)
    ms = timed(bt)
    r, _ = bt.results()
    print("cfg0 single", shape, bt.info(), "%.2f ms" % ms, r[0].inner_iterations, flush=True)
cnt = 4096
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=42 + i) for i in range(cnt)]
bt = B.Batch(ctx, probs)
bt.set_models()
for shape in [(256, 1), (256, 2), (512, 1)]:
    bt.set_launch(*shape)
    ms = timed(bt)
    print("batch", shape, bt.info(), "%.1f ms" % ms, "%.0f solves/s" % (cnt / ms * 1e3), flush=True)
