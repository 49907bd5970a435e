"""Single-solve device phase times (PhaseTimes, solver.hpp:563-570) per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

ctx = B.Context(0)
cases = [("cfg0", B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)),
         ("cfg1-500", B.build_intersection_case(B.intersection_spec(500, 10.0, 0.1), 2, 2)),
         ("cfg1-1000", B.build_intersection_case(B.intersection_spec(1000, 10.0, 0.1), 2, 2)),
         ("cfg3", B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)])))]
only = sys.argv[1:] or [c[0] for c in cases]
for name, p in cases:
    if name not in only:
        continue
    B.solve(p, ctx=ctx)
    r = B.solve(p, ctx=ctx).report
    passes = r.n_records + r.outer_iterations
    t = r.times
    print(f"{name:10s} nodes={p.tree.node_count:6d} status={r.status_name} inner={r.inner_iterations} "
          f"outer={r.outer_iterations} passes~{passes} total={1e3*t['total_s']:.2f}ms per-pass: "
          + " ".join(f"{k[:-2]}={1e6*v/passes:.1f}us" for k, v in t.items() if k != 'total_s'), flush=True)
