"""hypmsilqr (condensed P2) vs pmsilqr single-solve device latency."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

ctx = B.Context(0)
cases = [("cfg0", B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)),
         ("cfg2 late 2x3", B.build_multistage_case(B.multistage_spec(100, [(1, 2), (26, 2), (51, 2)]))),
         ("cfg2 late 4x3", B.build_multistage_case(B.multistage_spec(100, [(1, 4), (26, 4), (51, 4)]))),
         ("int N=300", B.build_intersection_case(B.intersection_spec(300, 10.0, 0.1), 2, 2))]
for name, p in cases:
    for solver in ("scan-tree-riccati", "scan-condensed"):
        o = B.SolverOptions()
        o.backward = solver
        r = B.solve(p, o, ctx=ctx)
        r = B.solve(p, o, ctx=ctx)
        print(f"{name:14s} {solver:18s} inner {r.report.inner_iterations:3d} total {r.report.times['total_s'] * 1e3:8.2f} ms")
