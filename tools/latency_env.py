"""Single-solve device latency of the large configs under BMPC_* env settings
(one process per setting): python tools/latency_env.py "BMPC_FWD_SCAN_MIN=512" ..."""
import os
import subprocess
import sys

CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2506_13624_b200 as B
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = B.Context(0, stream=s.cuda_stream)
cases = [("cfg1-500", B.build_intersection_case(B.intersection_spec(500, 10.0, 0.1), 2, 2)),
         ("cfg1-1000", B.build_intersection_case(B.intersection_spec(1000, 10.0, 0.1), 2, 2)),
         ("cfg3-spread", B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)]))),
         ("cfg3-early", B.build_multistage_case(B.multistage_spec(500, [(1, 4), (2, 4), (3, 4), (4, 4)])))]
out = []
for name, p in cases:
    bt = B.Batch(ctx, [p]); bt.set_models(); bt.solve(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); bt.solve(); e1.record(s); torch.cuda.synchronize()
    r, _ = bt.results()
    out.append("%s %.1fms(%d)" % (name, e0.elapsed_time(e1), r[0].inner_iterations))
print("RESULT", os.environ.get("TAG", ""), " ".join(out))
'''
for arg in sys.argv[1:]:
    env = dict(os.environ, TAG=arg)
    for kv in arg.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print([l for l in r.stdout.splitlines() if l.startswith("RESULT")] or r.stderr[-600:], flush=True)
