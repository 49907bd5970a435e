"""cfg4 batch-solve device time (CUDA events, inputs resident, median of 3)
for the probe/main block shape given in BMPC_CTA (and any other BMPC_* env),
one process per setting: python tools/shape_sweep.py 64x8 64x6 128x4 ..."""
import os
import subprocess
import sys

CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2506_13624_b200 as B
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = B.Context(0, stream=s.cuda_stream)
spec = B.intersection_spec(63, 10.0, 0.1)
bt = B.Batch(ctx, [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + i) for i in range(4096)])
bt.set_models(); bt.solve(); torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); bt.solve(); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort()
print("RESULT %s %.2f" % (os.environ.get("BMPC_CTA", "default") + " " + os.environ.get("BMPC_MAIN_BUDGET", "-") + " " + os.environ.get("BMPC_PROBE", "-"), ts[1]))
'''
for arg in sys.argv[1:]:
    env = dict(os.environ)
    for kv in arg.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            env[k] = v
        else:
            env["BMPC_CTA"] = kv
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print([l for l in out.stdout.splitlines() if l.startswith("RESULT")] or out.stderr[-500:], flush=True)
