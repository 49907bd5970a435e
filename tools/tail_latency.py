"""Single-instance latency of cfg0 and of the longest cfg4 instance (the
batch schedule's tail) across block shapes and sweep/scan choice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_13624_b200 as B

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = B.Context(0, stream=s.cuda_stream)


def timed(bt):
    bt.solve()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    bt.solve()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


spec = B.intersection_spec(63, 10.0, 0.1)
seeds = [int(a) for a in os.environ.get("SEEDS", "").split(",") if a]
cases = [("cfg0", B.build_intersection_case(spec, 2, 2))] + \
        [("seed%d" % sd, B.build_intersection_case(spec, 2, 2, perturb_seed=sd)) for sd in seeds]
shapes = [(int(a.split("x")[0]), int(a.split("x")[1])) for a in os.environ.get("SHAPES", "256x1").split(",")]
for name, p in cases:
    bt = B.Batch(ctx, [p])
    bt.set_models()
    for th, mb in shapes:
        try:
            bt.set_launch(th, mb)
        except Exception as e:  # noqa: BLE001
            print(name, th, mb, "n/a", e)
            continue
        line = []
        for sm in (0, 384):
            B.set_seq_max_len(ctx, sm)
            ms = timed(bt)
            r, _ = bt.results()
            line.append("seq<=%d: %.3fms (%d passes, %.1f us/pass)" % (sm, ms, r[0].n_records, 1e3 * ms / max(1, r[0].n_records)))
        print(name, "%dx%d" % (th, mb), " | ".join(line), flush=True)
