"""Per-phase device time of single solves (diagnostic, --phase timers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_13624_b200 as B

ctx = B.Context(0)
cases = [("cfg0", B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)),
         ("cfg1-1000", B.build_intersection_case(B.intersection_spec(1000, 10.0, 0.1), 2, 2)),
         ("cfg3", B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)])))]
for name, p in cases:
    bt = B.Batch(ctx, [p])
    bt.set_models()
    bt.solve()
    ctx.synchronize()
    B.batch_set_profiling(bt, True)
    bt.solve()
    reps, _ = bt.results()
    r = reps[0]
    prof = B.batch_phase_profile(bt)
    passes = r.n_records + r.outer_iterations
    cps = prof.pop("sweep_cycles_per_step", None)
    wk = prof.pop("walk_cycles", (0,) * 6)
    fs = prof.pop("fwd_scan_cycles", (0,) * 3)
    print(f"   forward scan cycles/pass: elements+barrier {fs[0] / passes:.0f}, run maps {fs[1] / passes:.0f}, scan+re-walk {fs[2] / passes:.0f}")
    print(f"   effective SM clock during the solve: {prof.pop('sm_mhz', 0):.0f} MHz")
    print(f"   walk cycles/pass: head_dx {wk[0] / passes:.0f}, chunks {wk[1] / passes:.0f}, depth walks {wk[2] / passes:.0f} ({wk[3] / passes:.0f} ns); element phases {wk[4] / passes:.0f}, chain (thread 0) {wk[5] / passes:.0f}")
    tot = sum(prof.values())
    if cps:
        print(f"   team sweep: {cps:.0f} cycles per chain step (thread 0's team)")
    print(f"{name}: nodes={p.tree.node_count} passes~{passes} total={r.times['total_s']*1e3:.2f}ms profiled={tot:.2f}ms")
    for k, v in prof.items():
        print(f"   {k:24s} {v:8.2f} ms  {1e3*v/passes:8.1f} us/pass  {100*v/tot:5.1f}%")
