"""Generates the compact population fixtures that pin the benched configs:

  tests/golden/cfg4_population.npz  every one of the 4,096 cfg4 bench instances
      (build_intersection_case(intersection_spec(63, 10, 0.1), 2, 2), x0
      perturbed with std::mt19937_64(42 + i), i = 0..4095), solved by the
      UNMODIFIED reference solve() (oracle/_ref/libbmpc_ref.so, default
      pmsilqr options; parallel=false, which is scheduling-independent,
      SPEC.md:443). Per instance: status, inner / outer / record counts, final
      cost / violation / defect, the whole per-record alpha level / accepted /
      outer sequences (int8, concatenated with offsets), the final record's
      cost and merit, and the state at every leaf plus x / u sums.
  tests/golden/cfg3_early.npz       cfg3-early, multistage_spec(500,
      [(1,4),(2,4),(3,4),(4,4)]) (127,062 nodes), solved by the same
      reference: full report, every IterationRecord, and the trajectory at
      every 61st node (plus sums over all nodes).

Each reference solve is cross-checked against the plain-C oracle
(oracle/_build) while generating (identical counts and alpha sequences), so
the fixture also re-pins the restatement at population scale. Run in the build
container (needs /root/reference via oracle/_ref):

  python tests/make_golden_batch.py [cfg4|cfg3|all] [--procs 8]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
GOLDEN = os.path.join(HERE, "golden")

CFG4_COUNT = 4096
CFG4_SEED0 = 42
CFG3_EARLY = (500, ((1, 4), (2, 4), (3, 4), (4, 4)))
CFG3_STRIDE = 61


def alpha_level(a):
    """IterationRecord alpha -> level l (alpha = 2^-l), -1 for a rejected pass."""
    a = np.asarray(a, np.float64)
    out = np.full(a.shape, -1, np.int8)
    ok = a > 0
    out[ok] = np.rint(-np.log2(a[ok])).astype(np.int8)
    return out


def _cfg4_one(i):
    import _oracle as O
    import _refbind as R
    import paper_2506_13624_b200 as B

    seed = CFG4_SEED0 + i
    sc = R.scenario(0, 63, total_time=10.0, shared=(0.1, 0.0), v=(2, 2), perturb_seed=seed)
    o = R.default_options()
    o.parallel = 0
    x, u, rep, rec = R.solve(sc, o)
    # Cross-check: the C restatement on the product's own builder output.
    p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=seed)
    oc = O.solve_problem(p)
    same = (oc["status"] == rep["status"] and oc["inner_iterations"] == rep["inner_iterations"]
            and oc["outer_iterations"] == rep["outer_iterations"]
            and np.array_equal(oc["records"]["alpha"], rec["alpha"]))
    leaves = np.flatnonzero(p.tree.child_count == 0)
    return dict(i=i, status=rep["status"], inner=rep["inner_iterations"], outer=rep["outer_iterations"],
                nrec=rep["n_records"], final_cost=rep["final_cost"], final_violation=rep["final_violation"],
                final_defect=rep["final_defect_l1"], lvl=alpha_level(rec["alpha"]),
                acc=np.asarray(rec["accepted"], np.int8), out=np.asarray(rec["outer"], np.int8),
                last_cost=rec["cost"][-1], last_merit=rec["merit_after"][-1], x_leaves=x[leaves],
                x_sum=x.sum(axis=0), u_sum=u.sum(axis=0), x_abs=np.abs(x).sum(), u_abs=np.abs(u).sum(),
                oracle_same=same)


def gen_cfg4(procs):
    t0 = time.time()
    with mp.Pool(procs) as pool:
        rows = pool.map(_cfg4_one, range(CFG4_COUNT), chunksize=8)
    rows.sort(key=lambda r: r["i"])
    off = np.zeros(CFG4_COUNT + 1, np.int64)
    off[1:] = np.cumsum([len(r["lvl"]) for r in rows])
    cat = lambda k: np.concatenate([r[k] for r in rows])  # noqa: E731
    col = lambda k, dt=np.float64: np.array([r[k] for r in rows], dt)  # noqa: E731
    mismatch = [r["i"] for r in rows if not r["oracle_same"]]
    meta = dict(count=CFG4_COUNT, seed0=CFG4_SEED0, scenario="intersection_spec(63,10.0,0.1) 2x2",
                solver="reference solve(), default options, parallel=false", oracle_mismatch=mismatch,
                seconds=time.time() - t0)
    np.savez_compressed(os.path.join(GOLDEN, "cfg4_population.npz"), status=col("status", np.int8),
                        inner=col("inner", np.int32), outer=col("outer", np.int32), nrec=col("nrec", np.int32),
                        final_cost=col("final_cost"), final_violation=col("final_violation"),
                        final_defect=col("final_defect"), last_cost=col("last_cost"),
                        last_merit=col("last_merit"), rec_off=off, rec_level=cat("lvl"), rec_accepted=cat("acc"),
                        rec_outer=cat("out"), x_leaves=np.stack([r["x_leaves"] for r in rows]),
                        x_sum=np.stack([r["x_sum"] for r in rows]), u_sum=np.stack([r["u_sum"] for r in rows]),
                        x_abs=col("x_abs"), u_abs=col("u_abs"), meta=json.dumps(meta))
    inner = col("inner", np.int32)
    print(f"cfg4_population: {CFG4_COUNT} instances, inner mean {inner.mean():.1f} max {inner.max()}, "
          f"status counts {np.bincount(col('status', np.int8))}, oracle mismatches {len(mismatch)}, "
          f"{time.time() - t0:.0f} s")


ULP_SIGNS = ((1, 1, 1, 1), (-1, -1, -1, -1), (1, -1, 1, -1), (-1, 1, -1, 1))


def _cfg4_sensitivity(i):
    """The C restatement (bit-identical to the reference) on instance i with
    its measured state moved by one ulp per component (4 sign patterns):
    how far the reference's own counts move under the smallest perturbation."""
    import _oracle as O
    import paper_2506_13624_b200 as B

    p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=CFG4_SEED0 + i)
    op = O.from_bmpc(p)
    x0 = op.keep["x0"].copy()
    inner, outer, status, cost = [], [], [], []
    for sg in ULP_SIGNS:
        op.keep["x0"][:] = [np.nextafter(v, np.inf if s > 0 else -np.inf) for v, s in zip(x0, sg)]
        o = O.solve(op)
        inner.append(o["inner_iterations"])
        outer.append(o["outer_iterations"])
        status.append(o["status"])
        cost.append(o["final_cost"])
    op.keep["x0"][:] = x0
    return i, inner, outer, status, cost


def _cfg4_fma(i):
    """Instance i on the FMA-contracted twin of the C restatement (every a*b+c
    rounded once, like the GPU): its counts under a different, equally valid
    rounding of the same arithmetic."""
    os.environ["BMPC_ORACLE_VARIANT"] = "fma"
    import _oracle as O
    import paper_2506_13624_b200 as B

    p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=CFG4_SEED0 + i)
    o = O.solve_problem(p)
    return i, o["inner_iterations"], o["outer_iterations"], o["status"], o["final_cost"]


def gen_fma(procs):
    t0 = time.time()
    with mp.Pool(procs) as pool:
        rows = pool.map(_cfg4_fma, range(CFG4_COUNT), chunksize=8)
    rows.sort(key=lambda r: r[0])
    path = os.path.join(GOLDEN, "cfg4_population.npz")
    z = dict(np.load(path))
    z["fma_inner"] = np.array([r[1] for r in rows], np.int32)
    z["fma_outer"] = np.array([r[2] for r in rows], np.int32)
    z["fma_status"] = np.array([r[3] for r in rows], np.int8)
    z["fma_final_cost"] = np.array([r[4] for r in rows])
    meta = json.loads(str(z["meta"]))
    sens = np.flatnonzero(z["fma_inner"] != z["inner"])
    meta["fma_sensitive"] = int(sens.size)
    z["meta"] = json.dumps(meta)
    np.savez_compressed(path, **z)
    print(f"cfg4 fma twin: {sens.size} of {CFG4_COUNT} instances change their inner count, {time.time() - t0:.0f} s")


def gen_sensitivity(procs):
    t0 = time.time()
    with mp.Pool(procs) as pool:
        rows = pool.map(_cfg4_sensitivity, range(CFG4_COUNT), chunksize=8)
    rows.sort(key=lambda r: r[0])
    path = os.path.join(GOLDEN, "cfg4_population.npz")
    z = dict(np.load(path))
    z["ulp_inner"] = np.array([r[1] for r in rows], np.int32)
    z["ulp_outer"] = np.array([r[2] for r in rows], np.int32)
    z["ulp_status"] = np.array([r[3] for r in rows], np.int8)
    z["ulp_final_cost"] = np.array([r[4] for r in rows])
    meta = json.loads(str(z["meta"]))
    meta["ulp_signs"] = ULP_SIGNS
    sens = np.flatnonzero((z["ulp_inner"] != z["inner"][:, None]).any(axis=1))
    meta["ulp_sensitive"] = int(sens.size)
    z["meta"] = json.dumps(meta)
    np.savez_compressed(path, **z)
    print(f"cfg4 ulp sensitivity: {sens.size} of {CFG4_COUNT} instances change their inner count under a "
          f"1-ulp x0 perturbation, {time.time() - t0:.0f} s")


def gen_cfg3():
    import _oracle as O
    import _refbind as R
    import paper_2506_13624_b200 as B

    N, br = CFG3_EARLY
    t0 = time.time()
    sc = R.scenario(2, N, total_time=10.0, shared=(0.1, 0.0), v=(2, 2), branchings=br)
    o = R.default_options()
    x, u, rep, rec = R.solve(sc, o, max_records=4000)
    t_ref = time.time() - t0
    p = B.build_multistage_case(B.multistage_spec(N, list(br)))
    oc = O.solve_problem(p)
    same = (oc["status"] == rep["status"] and oc["inner_iterations"] == rep["inner_iterations"]
            and np.array_equal(oc["records"]["alpha"], rec["alpha"]))
    idx = np.arange(0, x.shape[0], CFG3_STRIDE)
    meta = dict(horizon=N, branchings=br, nodes=int(x.shape[0]), stride=CFG3_STRIDE, oracle_same=bool(same),
                oracle_x_rel=float(np.linalg.norm(oc["x"] - x) / np.linalg.norm(x)), reference_seconds=t_ref)
    np.savez_compressed(os.path.join(GOLDEN, "cfg3_early.npz"), x_sub=x[idx], u_sub=u[idx], idx=idx,
                        x_sum=x.sum(axis=0), u_sum=u.sum(axis=0), x_norm=np.linalg.norm(x), u_norm=np.linalg.norm(u),
                        report=json.dumps(rep), meta=json.dumps(meta), **{"rec_" + k: v for k, v in rec.items()})
    print(f"cfg3_early: {x.shape[0]} nodes, status {rep['status']} inner {rep['inner_iterations']} outer "
          f"{rep['outer_iterations']}, oracle same={same}, reference {t_ref:.0f} s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="?", default="all", choices=["cfg4", "cfg3", "ulp", "fma", "all"])
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    if a.which in ("cfg4", "all"):
        gen_cfg4(a.procs)
    if a.which in ("ulp", "all"):
        gen_sensitivity(a.procs)
    if a.which in ("fma", "all"):
        gen_fma(a.procs)
    if a.which in ("cfg3", "all"):
        gen_cfg3()
