"""Breakdown of the e2e step (bench.py's e2e leg): set_models / solve / results."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_13624_b200 as B

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = B.Context(0, stream=s.cuda_stream)
cnt = 4096
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=42 + i) for i in range(cnt)]
bt = B.Batch(ctx, probs)
n, nx, nu = bt.n, bt.nx, bt.nu
xh = np.empty((cnt, n, nx))
uh = np.empty((cnt, n, nu))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bt.set_models()
    ctx.synchronize()
    t1 = time.perf_counter()
    bt.solve()
    ctx.synchronize()
    t2 = time.perf_counter()
    bt.results(xh, uh, want_reports=False)
    t3 = time.perf_counter()
    bt.results(xh, uh, want_reports=True)
    t4 = time.perf_counter()
    print(f"set_models {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, results(no reports) {1e3*(t3-t2):.1f} ms, "
          f"results(reports) {1e3*(t4-t3):.1f} ms")
