"""Crossover experiment: team Riccati sweep vs scan, per config."""
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


cases = [("cfg0", B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)),
         ("cfg1-500", B.build_intersection_case(B.intersection_spec(500, 10.0, 0.1), 2, 2)),
         ("cfg1-1000", B.build_intersection_case(B.intersection_spec(1000, 10.0, 0.1), 2, 2)),
         ("cfg3", B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)]))),
         ("cfg3e", B.build_multistage_case(B.multistage_spec(500, [(1, 4), (2, 4), (3, 4), (4, 4)])))]
for name, p in cases:
    bt = B.Batch(ctx, [p])
    bt.set_models()
    line = []
    for sm in (0, 64, 256, 384, 512, 768, 1024):
        B.set_seq_max_len(ctx, sm)
        ms = timed(bt)
        r, _ = bt.results()
        line.append("seq<=%d: %.2fms (%d it)" % (sm, ms, r[0].inner_iterations))
    print(name, p.tree.node_count, " | ".join(line), flush=True)
