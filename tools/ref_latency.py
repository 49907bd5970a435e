"""Single-solve latency of the shim-built reference (oracle/_ref) on the host
cores next to the GPU latency (bench.py latency table configs). Writes
gpurun_out/ref_latency.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import _refbind as R  # noqa: E402

cases = [("cfg0 N=63 4 leaves", dict(family=0, horizon=63)),
         ("cfg1 N=500 4 leaves", dict(family=0, horizon=500)),
         ("cfg1 N=1000 4 leaves", dict(family=0, horizon=1000)),
         ("cfg2 N=100 2 leaves {1}", dict(family=2, horizon=100, branchings=[(1, 2)])),
         ("cfg2 N=100 64 leaves {1,26,51}", dict(family=2, horizon=100, branchings=[(1, 4), (26, 4), (51, 4)])),
         ("cfg3 N=500 256 leaves {1,100,200,300}",
          dict(family=2, horizon=500, branchings=[(1, 4), (100, 4), (200, 4), (300, 4)]))]
which = sys.argv[1:] or [c[0] for c in cases]
out = {"cores": os.cpu_count()}
for name, kw in cases:
    if name not in which:
        continue
    sc = R.scenario(**kw)
    res = {}
    for par in (1, 0):
        o = R.default_options()
        o.parallel = par
        t0 = time.perf_counter()
        _, _, rep, _ = R.solve(sc, o)
        res["parallel" if par else "serial"] = {"ms": 1e3 * (time.perf_counter() - t0), "inner": rep["inner_iterations"],
                                                 "outer": rep["outer_iterations"], "status": rep["status"]}
        print(name, "parallel" if par else "serial", res["parallel" if par else "serial"], flush=True)
    out[name] = res
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "ref_latency.json"), "w"), indent=1)
