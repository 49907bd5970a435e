"""Dump every cfg4 instance's full IterationRecord history (for choosing the
batch schedule's ordering keys offline): gpurun_out/tail_features.npz."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import numpy as np

import paper_2506_13624_b200 as B

count, maxr = 4096, 1000
spec = B.intersection_spec(63, 10.0, 0.1)
probs = [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + i) for i in range(count)]
ctx = B.Context(0)
bt = B.Batch(ctx, probs, max_records=maxr)
bt.set_models()
bt.solve()
reps, _ = bt.results(as_array=True)
recs = (B._Record * maxr)()
n = C.c_int()
fields = ["outer", "accepted", "cost", "cost_al", "violation", "alpha", "regularization", "defect_l1", "mu"]
out = {f: np.full((count, maxr), np.nan) for f in fields}
for i in range(count):
    B._check(B.lib().bmpc_batch_records(bt._h, i, recs, maxr, C.byref(n)))
    a = np.ctypeslib.as_array(recs)[: n.value]
    for f in fields:
        out[f][i, : n.value] = a[f]
np.savez_compressed("gpurun_out/tail_features.npz", passes=reps["n_records"], status=reps["status"],
                    outer_iterations=reps["outer_iterations"], **out)
print("done", reps["n_records"].max())
