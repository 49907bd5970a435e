"""Generates tests/golden/*.npz from the UNMODIFIED reference solver
(oracle/_ref/libbmpc_ref.so, built from /root/reference/proj headers against
the Eigen shim). Run in the build container:  python tests/make_golden.py

Fixtures: full solve() outputs (trajectory, report, every IterationRecord) of
the scenario problems the reference tests and BASELINE configs use, random
linear-quadratic instances (oracles.hpp:316, std::mt19937_64 seeds), and one
kernel-level backward_pass/linear_rollout case. The GPU tests compare the
CUDA path against these on the GPU box, where /root/reference is absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
import _gen  # noqa: E402
import _refbind as R  # noqa: E402

GOLDEN = os.path.join(HERE, "golden")

SCENARIOS = {
    # name: (family, horizon, total_time, shared, v, branchings, perturb_seed)
    "cfg0_intersection_63": (0, 63, 10.0, (0.1, 0.0), (2, 2), (), None),
    "intersection_20_4s": (0, 20, 4.0, (0.4, 0.0), (2, 2), (), None),        # test_solver.cpp:414
    "intersection_25_1x2": (0, 25, 5.0, (0.4, 0.0), (1, 2), (), None),       # test_solver.cpp:473
    "latency_0p5_63": (1, 63, 5.0, (0.05, 0.5), (2, 2), (), None),           # test_solver.cpp:537
    "multistage_100_2x2": (2, 100, 10.0, (0.1, 0.0), (2, 2), ((1, 2), (34, 2)), None),
    "cfg4_instance_seed42": (0, 63, 10.0, (0.1, 0.0), (2, 2), (), 42),
    "cfg4_instance_seed43": (0, 63, 10.0, (0.1, 0.0), (2, 2), (), 43),
}

LQ = {
    # name: (horizon, branchings, nx, nu, seed)
    "lq_6_branch2_nx3nu2": (6, ((2, 2, (0.5, 0.5)),), 3, 2, 2024),
    "lq_7_branch3_nx3nu2": (7, ((3, 2, (0.5, 0.5)),), 3, 2, 7),
    "lq_5_path_nx2nu1": (5, (), 2, 1, 11),
}


def dump_solve(name, sc, meta):
    x, u, rep, rec = R.solve(sc)
    d = R.dump(sc) if sc.family != 3 else {}
    np.savez_compressed(os.path.join(GOLDEN, name + ".npz"), x=x, u=u,
                        report=json.dumps(rep), meta=json.dumps(meta),
                        **{"rec_" + k: v for k, v in rec.items()},
                        **{("prob_" + k): v for k, v in d.items() if isinstance(v, np.ndarray)})
    print(f"{name}: status={rep['status']} inner={rep['inner_iterations']} outer={rep['outer_iterations']} "
          f"records={rep['n_records']}")


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    for name, (fam, N, T, sh, v, br, seed) in SCENARIOS.items():
        sc = R.scenario(fam, N, total_time=T, shared=sh, v=v, branchings=br, perturb_seed=seed)
        dump_solve(name, sc, dict(family=fam, horizon=N, total_time=T, shared=sh, v=v, branchings=br,
                                  perturb_seed=seed))
    for name, (N, br, nx, nu, seed) in LQ.items():
        sc = R.scenario(3, N, branchings=br, lq=(nx, nu, seed))
        x0, st, lf = R.lq_dump(sc)
        x, u, rep, rec = R.solve(sc)
        np.savez_compressed(os.path.join(GOLDEN, name + ".npz"), x=x, u=u, x0=x0, stage=st, leaf=lf,
                            report=json.dumps(rep),
                            meta=json.dumps(dict(horizon=N, branchings=br, nx=nx, nu=nu, seed=seed)),
                            **{"rec_" + k: v for k, v in rec.items()})
        print(f"{name}: status={rep['status']} inner={rep['inner_iterations']}")
    # Kernel-level LQR tree (solver.hpp:203-430) on random TreeStageModels.
    import paper_2506_13624_b200 as B

    rng = np.random.default_rng(7)
    br = ((2, 2, (0.5, 0.5)), (4, 3, (0.2, 0.3, 0.5)))
    tree = B.build_tree(6, br)
    stage, defect, leaf = _gen.random_tree_models(rng, tree, 3, 2)
    dx0 = rng.uniform(-1, 1, 3)
    out = R.lqr_tree(br, 6, 3, 2, stage, defect, leaf, 0.0, 0, dx0)
    np.savez_compressed(os.path.join(GOLDEN, "lqr_tree_two_stage_nx3nu2.npz"), stage=stage, defect=defect,
                        leaf=leaf, dx0=dx0, meta=json.dumps(dict(horizon=6, branchings=br, nx=3, nu=2)),
                        **{k: np.asarray(v) for k, v in out.items()})
    print("lqr_tree_two_stage_nx3nu2: written")
    # `bench gen` documents (bench.cpp:327-357) written by the reference's own
    # serialization (oracle/_ref/gen_ref), fixtures for the CLI's gen command.
    import gzip
    import subprocess

    for scen in ("intersection", "latency", "report", "tree"):
        doc = subprocess.run([os.path.join(os.path.dirname(HERE), "oracle", "_ref", "gen_ref"), scen],
                             check=True, capture_output=True, text=True).stdout
        with gzip.open(os.path.join(GOLDEN, "gen_%s.json.gz" % scen), "wt") as f:
            f.write(doc)
        print("gen_%s.json.gz: written" % scen)


if __name__ == "__main__":
    main()
