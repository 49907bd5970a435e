"""Per-phase device time of one instance inside a full steady-state batch
(identical cfg0 instances at a block shape): which phases cost under contention."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2506_13624_b200 as B

cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 592
t, m = (int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "128x4").split("x"))
ctx = B.Context(0)
probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2) for _ in range(cnt)]
bt = B.Batch(ctx, probs)
bt.set_models()
bt.set_launch(t, m)
bt.solve()
B.batch_set_profiling(bt, True)
bt.solve()
reps, _ = bt.results()
for inst in (0, cnt // 2):
    prof = B.batch_phase_profile(bt, inst)
    r = reps[inst]
    passes = r.n_records + r.outer_iterations
    cps = prof.pop("sweep_cycles_per_step", None)
    wk = prof.pop("walk_cycles", (0,) * 6)
    prof.pop("fwd_scan_cycles", None)
    print(f"   effective SM clock during the solve: {prof.pop('sm_mhz', 0):.0f} MHz")
    print(f"   walk cycles/pass: head_dx {wk[0] / passes:.0f}, chunks {wk[1] / passes:.0f}, depth walks {wk[2] / passes:.0f} ({wk[3] / passes:.0f} ns); element phases {wk[4] / passes:.0f}, chain (thread 0) {wk[5] / passes:.0f}")
    tot = sum(prof.values())
    print(f"{t}x{m} instance {inst}: passes {passes} total {r.times['total_s']*1e3:.2f} ms, sweep {cps or 0:.0f} cyc/step")
    for k, v in prof.items():
        if v > 0:
            print(f"   {k:24s} {1e3*v/passes:8.1f} us/pass  {100*v/tot:5.1f}%")
