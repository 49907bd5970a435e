"""cfg4 batch step time under the current BMPC_* schedule knobs (e.g.
BMPC_MAIN_BUDGET, BMPC_PROBE): best of 3 device-timed solves of the 4,096
bench instances, plus a hash of every instance's (status, inner, outer) so
settings can be checked to give identical results."""
import hashlib
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
spec = B.intersection_spec(63, 10.0, 0.1)
bt = B.Batch(ctx, [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + i) for i in range(cnt)])
bt.set_models()
bt.solve()
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    bt.solve()
    e1.record(s)
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
x = np.zeros((cnt, bt.n, bt.nx))
reps, _ = bt.results(x, None, as_array=True)
key = np.stack([reps["status"], reps["inner_iterations"], reps["outer_iterations"]]).astype(np.int64)
xh = hashlib.sha1(x.tobytes()).hexdigest()[:12]
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("BMPC_"))
print(f"RESULT [{tag}] {best:.1f} ms  counts {hashlib.sha1(key.tobytes()).hexdigest()[:12]} x {xh}")
