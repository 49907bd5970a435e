"""Single-instance latency of cfg0 (and a few tail cfg4 instances) per block
shape, chunked backward sweep on / off (BMPC_CHUNK_BWD): device time of one
batch launch of ONE instance, CUDA events via the report's total time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

ctx = B.Context(0)
spec = B.intersection_spec(63, 10.0, 0.1)
cases = [("cfg0", B.build_intersection_case(spec, 2, 2)),
         ("cfg4#1602", B.build_intersection_case(spec, 2, 2, perturb_seed=42 + 1602)),
         ("cfg4#601", B.build_intersection_case(spec, 2, 2, perturb_seed=42 + 601))]
for shape in [(64, 4), (128, 2), (128, 3), (256, 1), (512, 1)]:
    for name, p in cases:
        bt = B.Batch(ctx, [p], max_records=1000)
        bt.set_models()
        bt.set_launch(*shape)
        best = 1e9
        for _ in range(3):
            bt.solve()
            reps, _ = bt.results()
            best = min(best, reps[0].times["total_s"])
        r = reps[0]
        passes = r.n_records + r.outer_iterations
        print(f"{shape[0]}x{shape[1]} chunk={os.environ.get('BMPC_CHUNK_BWD', '1')} {name:10s} inner {r.inner_iterations:4d} "
              f"passes {passes:4d}  {best * 1e3:8.2f} ms  {best * 1e6 / passes:7.1f} us/pass")
