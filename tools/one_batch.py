"""One cfg4 batch solve (4096 perturbed cfg0 instances), for launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
spec = B.intersection_spec(63, 10.0, 0.1)
bt = B.Batch(B.Context(0), [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + i) for i in range(n)])
bt.set_models()
bt.solve()
bt.results()
