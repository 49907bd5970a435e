"""Is the cfg4 batch bounded by throughput or by its slowest instances?
Prints kernel time, per-instance device time stats and the straggler positions."""
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
shape = sys.argv[2] if len(sys.argv) > 2 else "default"
t, m = (int(v) for v in shape.split("x")) if shape != "default" else (0, 8)
same = len(sys.argv) > 3 and sys.argv[3] == "same"  # identical instances: no tail, steady-state throughput
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=None if same else 42 + i)
         for i in range(cnt)]
bt = B.Batch(ctx, probs)
bt.set_models()
if shape != "default":
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
tt = np.array([r.times["total_s"] for r in reps]) * 1e3
passes = np.array([r.n_records + r.outer_iterations for r in reps])
slots = 148 * m
print(f"{shape}: kernel {ms:.1f} ms; instance ms mean {tt.mean():.2f} p50 {np.median(tt):.2f} "
      f"p99 {np.percentile(tt, 99):.2f} max {tt.max():.2f}; sum/slots {tt.sum() / slots:.1f} ms; "
      f"us/pass mean {1e3 * (tt / passes).mean():.1f}")
top = np.argsort(-tt)[:8]
try:
    print("slowest:", [(int(i), round(float(tt[i]), 1), int(passes[i])) for i in top], flush=True)
except BrokenPipeError:
    pass
