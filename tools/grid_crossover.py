"""Single-solve latency, one thread block (CTA mode) vs the whole GPU (grid
mode), over the cfg1 horizon sweep: run once per BMPC_GRID_MIN_NODES value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

ctx = B.Context(0)
for N in [int(a) for a in os.environ.get("HORIZONS", "63,100,127,200,255").split(",")]:
    p = B.build_intersection_case(B.intersection_spec(N), 2, 2)
    bt = B.Batch(ctx, [p])
    bt.set_models()
    ts = []
    for _ in range(3):
        bt.solve()
        r, _ = bt.results()
        ts.append(r[0].times["total_s"] * 1e3)
    print("grid_min=%s N=%d nodes=%d mode=%s total_ms=%.3f inner=%d" % (
        os.environ.get("BMPC_GRID_MIN_NODES", "1024"), N, p.tree.node_count,
        "grid" if p.tree.node_count > int(os.environ.get("BMPC_GRID_MIN_NODES", "1024")) else "cta",
        min(ts), r[0].inner_iterations), flush=True)
