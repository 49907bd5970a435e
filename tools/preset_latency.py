"""Single-solve latency of every solver preset (apply_solver_name,
tools/bench.cpp:60-83) on the GPU (device time of the one solve launch,
inputs resident) next to the shim-built reference (oracle/_ref) running the
same preset on the host (parallel=false for smsilqr/sssilqr as the preset
sets; pmsilqr with its own threads). Writes gpurun_out/preset_latency.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import _refbind as R  # noqa: E402
import paper_2506_13624_b200 as B  # noqa: E402
from paper_2506_13624_b200 import cli  # noqa: E402

PRESETS = {"pmsilqr": (0, 0, 0, 1), "smsilqr": (2, 0, 1, 0), "sssilqr": (2, 1, 1, 0)}
cases = [("cfg0 N=63 4 leaves", B.intersection_spec(63, 10.0, 0.1), "int", dict(family=0, horizon=63)),
         ("cfg1 N=500 4 leaves", B.intersection_spec(500, 10.0, 0.1), "int", dict(family=0, horizon=500)),
         ("cfg2 N=100 64 leaves {1,26,51}", B.multistage_spec(100, [(1, 4), (26, 4), (51, 4)]), "ms",
          dict(family=2, horizon=100, branchings=[(1, 4), (26, 4), (51, 4)]))]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = B.Context(0, stream=stream.cuda_stream)  # events below record on the solve's stream
out = {"cores": os.cpu_count()}
for name, spec, kind, kw in cases:
    p = B.build_intersection_case(spec, 2, 2) if kind == "int" else B.build_multistage_case(spec)
    sc = R.scenario(**kw)
    for solver, (bw, fw, ls, par) in PRESETS.items():
        o = B.SolverOptions()
        cli.apply_solver_name(solver, o)
        bt = B.Batch(ctx, [p])
        bt.set_models()
        bt.solve(o)
        torch.cuda.synchronize()
        ms = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s = torch.cuda.current_stream()
            e0.record(s)
            bt.solve(o)
            e1.record(s)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        rep, _ = bt.results(want_reports=True)
        ro = R.default_options()
        ro.backward, ro.forward, ro.line_search, ro.parallel = bw, fw, ls, par
        t0 = time.perf_counter()
        _, _, rr, _ = R.solve(sc, ro)
        ref_ms = 1e3 * (time.perf_counter() - t0)
        row = {"gpu_ms": sorted(ms)[1], "inner": rep[0].inner_iterations, "outer": rep[0].outer_iterations,
               "status": rep[0].status_name, "ref_ms": ref_ms, "ref_inner": rr["inner_iterations"],
               "ref_outer": rr["outer_iterations"], "speedup": ref_ms / sorted(ms)[1]}
        out.setdefault(name, {})[solver] = row
        print(name, solver, row, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "preset_latency.json"), "w"), indent=1)
