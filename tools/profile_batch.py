"""Batch solve for ncu: N instances of perturbed cfg0 at a block shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_13624_b200 as B

cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 592
shape = sys.argv[2] if len(sys.argv) > 2 else "default"
ctx = B.Context(0)
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=42 + i) for i in range(cnt)]
bt = B.Batch(ctx, probs)
bt.set_models()
if shape != "default":
    bt.set_launch(*(int(v) for v in shape.split("x")))
bt.solve()
reps, _ = bt.results()
p = np.array([r.n_records + r.outer_iterations for r in reps])
print("passes mean %.1f p50 %d p90 %d p99 %d max %d" % (p.mean(), np.median(p), np.percentile(p, 90),
                                                         np.percentile(p, 99), p.max()))
print("top passes", sorted(p)[-12:])
