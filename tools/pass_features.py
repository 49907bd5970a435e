"""Dump per-instance pass counts and first-iteration features of the cfg4 batch
(does anything cheap predict the heavy-tailed pass counts?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_13624_b200 as B

cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = B.Context(0)
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=42 + i) for i in range(cnt)]
bt = B.Batch(ctx, probs, max_records=1000)
bt.set_models()
bt.solve()
reps, _ = bt.results()
out = {"passes": np.array([r.n_records + r.outer_iterations for r in reps]),
       "outer": np.array([r.outer_iterations for r in reps]),
       "status": np.array([r.status for r in reps]),
       "x0": np.array([p.initial_state for p in probs])}
K = 60  # first K records of every instance (zero-padded)
first = {k: [] for k in ("outer", "cost", "violation", "defect_l1", "regularization", "alpha", "accepted")}
for i in range(cnt):
    rec = bt.records(i, 1000)
    for k in first:
        v = np.asarray(rec[k], dtype=float)[:K]
        first[k].append(np.pad(v, (0, K - len(v))))
for k, v in first.items():
    out["rec_" + k] = np.array(v)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/pass_features.npz", **out)
print("saved", {k: v.shape for k, v in out.items()})
