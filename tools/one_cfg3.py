"""One cfg3-spread solve (256 scenarios, N=500, 59,598 nodes) on the whole GPU
(cooperative grid kernel), for ncu captures of the grid path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

p = B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)]))
r = B.solve(p, ctx=B.Context(0))
print(r.report.status_name, r.report.inner_iterations, r.report.outer_iterations)
