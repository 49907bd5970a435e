"""Generates tests/golden/preset_*.npz: full solve() outputs of the
reference's other solver presets (apply_solver_name, tools/bench.cpp:60-83)
from the UNMODIFIED reference (oracle/_ref/libbmpc_ref.so). Run in the build
container:  python tests/make_golden_presets.py

  smsilqr  backward sequential_riccati, linear rollout, sequential line search
  sssilqr  backward sequential_riccati, nonlinear rollout (single shooting),
           sequential line search (solver.hpp:463-467, problem.hpp:170-191)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import _refbind as R  # noqa: E402
from make_golden import GOLDEN, SCENARIOS  # noqa: E402

PRESETS = {"smsilqr": (2, 0, 1), "sssilqr": (2, 1, 1), "hypmsilqr": (1, 0, 0)}  # (backward, forward, line_search)
CASES = ("cfg0_intersection_63", "intersection_20_4s", "latency_0p5_63", "multistage_100_2x2",
         "cfg4_instance_seed42")


# Whole-GPU (cooperative grid) path: trees > 1024 nodes.
EXTRA = {"intersection_300": (0, 300, 10.0, (0.1, 0.0), (2, 2), (), None)}
# hypmsilqr: late branchings (large N_b) make the condensed shared segment
# (and its dense QP) large: cfg2 spread branchings at steps {1, 26, 51}.
COND_EXTRA = {"cfg2_late_2x3": (2, 100, 10.0, (0.1, 0.0), (2, 2), ((1, 2), (26, 2), (51, 2)), None),
              "cfg2_late_4x3": (2, 100, 10.0, (0.1, 0.0), (2, 2), ((1, 4), (26, 4), (51, 4)), None)}


def main():
    only = sys.argv[1:]
    for solver, (bw, fw, ls) in PRESETS.items():
        if only and solver not in only:
            continue
        for name in CASES + tuple(EXTRA) + (tuple(COND_EXTRA) if solver == "hypmsilqr" else ()):
            fam, N, T, sh, v, br, seed = {**SCENARIOS, **EXTRA, **COND_EXTRA}[name]
            sc = R.scenario(fam, N, total_time=T, shared=sh, v=v, branchings=br, perturb_seed=seed)
            o = R.default_options()
            o.backward, o.forward, o.line_search, o.parallel = bw, fw, ls, 0
            x, u, rep, rec = R.solve(sc, o)
            meta = dict(family=fam, horizon=N, total_time=T, shared=sh, v=v, branchings=br, perturb_seed=seed,
                        solver=solver, backward=bw, forward=fw, line_search=ls)
            out = "preset_%s_%s" % (solver, name)
            np.savez_compressed(os.path.join(GOLDEN, out + ".npz"), x=x, u=u, report=json.dumps(rep),
                                meta=json.dumps(meta), **{"rec_" + k: v for k, v in rec.items()})
            print(f"{out}: status={rep['status']} inner={rep['inner_iterations']} "
                  f"outer={rep['outer_iterations']} records={rep['n_records']}")


if __name__ == "__main__":
    main()
