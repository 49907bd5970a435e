"""Sweep per-instance block shapes on the cfg4 batch (kernel time, CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_13624_b200 as B

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = B.Context(0, stream=s.cuda_stream)
cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
shapes = [(256, 1), (256, 2), (256, 3), (256, 4), (128, 4), (128, 6), (128, 8), (512, 2)]
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=42 + i) for i in range(cnt)]
bt = B.Batch(ctx, probs)
bt.set_models()
for t, m in shapes:
    bt.set_launch(t, m)
    bt.solve()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    bt.solve()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    reps, _ = bt.results()
    passes = np.array([r.n_records + r.outer_iterations for r in reps])
    print(t, m, bt.info(), "ms %.1f" % ms, "solves/s %.0f" % (cnt / ms * 1e3),
          "conv", sum(r.status == 0 for r in reps), "passes mean %.1f max %d" % (passes.mean(), passes.max()),
          flush=True)
