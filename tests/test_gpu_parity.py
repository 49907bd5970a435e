"""GPU parity: the sm_100a solver (through the C ABI) against the oracle —
the C restatement (tests/_oracle.py, bit-identical to the reference) and the
reference's own golden outputs (tests/golden). Tolerances (north star):
trajectories / costs within 1e-8 relative (FP64, scan reassociation and FMA
change rounding); tree topology bit-exact; identical inner/outer iteration
counts and per-iteration alpha / acceptance sequences."""
import numpy as np
import pytest

import _fixtures as F
import _gen
import _oracle as O
import paper_2506_13624_b200 as B

pytestmark = pytest.mark.gpu

TOL = 1e-8


@pytest.fixture(scope="module")
def ctx():
    return B.Context(0)


def otree(t):
    return dict(parent=t.parent, first_child=t.first_child, nchild=t.child_count, weight=t.weight,
                step_begin=t.step_begin, horizon=t.horizon, last_branch_step=t.last_branch_step)


def assert_same_solve(res, ref_report, ref_x, ref_u, ref_records, tol=TOL):
    r = res.report
    assert r.status == ref_report["status"], (r.status, ref_report["status"], r.message)
    assert r.inner_iterations == ref_report["inner_iterations"]
    assert r.outer_iterations == ref_report["outer_iterations"]
    assert r.n_records == ref_report["n_records"]
    np.testing.assert_array_equal(r.iterations["alpha"], ref_records["alpha"])
    np.testing.assert_array_equal(r.iterations["accepted"], ref_records["accepted"])
    np.testing.assert_array_equal(r.iterations["outer"], ref_records["outer"])
    assert _gen.rel_err(res.trajectory.state, ref_x) <= tol
    assert _gen.rel_err(res.trajectory.input, ref_u) <= tol
    assert abs(r.final_cost - ref_report["final_cost"]) <= tol * max(1.0, abs(ref_report["final_cost"]))
    for k in ("cost", "cost_al", "merit_before", "merit_after"):
        assert _gen.rel_err(r.iterations[k], ref_records[k]) <= 1e-7, k


# ------------------------------------------------------------ kernel level
TREES = [
    (6, [(4, 2, [0.5, 0.5])]),
    (6, [(2, 2, [0.5, 0.5]), (4, 3, [0.2, 0.3, 0.5])]),
    (5, []),
    (5, [(4, 3, [0.3, 0.3, 0.4])]),                      # branching at the last step: single-leaf tails
    (40, [(3, 2, [0.5, 0.5]), (17, 2, [0.25, 0.75])]),
    (30, [(0, 2, [0.5, 0.5]), (1, 2, [0.5, 0.5])]),       # consecutive branchings (length-1 segments)
]


@pytest.mark.parametrize("grid", [False, True])
@pytest.mark.parametrize("dims", [(2, 1), (3, 2), (4, 2), (2, 4), (8, 4)])
@pytest.mark.parametrize("ti", range(len(TREES)))
def test_lqr_tree_matches_oracle(ctx, ti, dims, grid):
    horizon, br = TREES[ti]
    nx, nu = dims
    rng = np.random.default_rng(100 + ti)
    tree = B.build_tree(horizon, br)
    stage, defect, leaf = _gen.random_tree_models(rng, tree, nx, nu)
    dx0 = rng.uniform(-1, 1, nx)
    got = B.lqr_tree(tree, nx, nu, stage, defect, leaf, 0.0, dx0, grid=grid, ctx=ctx)
    ref = O.lqr_tree(otree(tree), nx, nu, stage, defect, leaf, 0.0, 0, dx0)
    assert got["error"] == ref["error"] == 0
    nl = tree.child_count > 0
    for key, mask in (("K", nl), ("k", nl), ("dx", slice(None)), ("du", nl), ("P", slice(None)),
                      ("p", slice(None))):
        assert _gen.rel_err(got[key][mask], ref[key][mask]) < 1e-9, key
    for key in ("a1", "a2", "max_feedforward"):
        assert abs(got[key] - ref[key]) <= 1e-9 * (1 + abs(ref[key])), key


@pytest.mark.parametrize("nx", [2, 4, 8])
@pytest.mark.parametrize("nu", [1, 2, 4])
@pytest.mark.parametrize("N", [8, 64, 511])
def test_scan_vs_sequential_riccati_grid(ctx, nx, nu, N):
    """verification.hpp:42-73: scan values within 1e-8 of the sequential
    Riccati recursion on every step of a path, (nx, nu, N) grid."""
    rng = np.random.default_rng(12345 + nx * 100 + nu * 10 + N)
    tree = B.build_tree(N, [])
    stage, defect, leaf = _gen.random_tree_models(rng, tree, nx, nu)
    got = B.lqr_tree(tree, nx, nu, stage, defect, leaf, ctx=ctx, grid=N > 64)
    ric = O.lqr_tree(otree(tree), nx, nu, stage, defect, leaf, 0.0, 2)
    worst = max(max(_gen.rel_err(got["P"][k], ric["P"][k]), _gen.rel_err(got["p"][k], ric["p"][k]))
                for k in range(N + 1))
    assert worst <= 1e-8
    # forward scan vs sequential rollout (verification.hpp:76-107, <= 1e-10 there
    # with shared policies; here each side uses its own policies).
    assert _gen.rel_err(got["dx"], ric["dx"]) <= 1e-8


def test_lqr_tree_regularization_and_indefinite(ctx):
    rng = np.random.default_rng(3)
    br = [(2, 2, [0.5, 0.5])]
    tree = B.build_tree(8, br)
    stage, defect, leaf = _gen.random_tree_models(rng, tree, 4, 2)
    got = B.lqr_tree(tree, 4, 2, stage, defect, leaf, 0.1, ctx=ctx)
    ref = O.lqr_tree(otree(tree), 4, 2, stage, defect, leaf, 0.1, 0)
    assert _gen.rel_err(got["K"][tree.child_count > 0], ref["K"][tree.child_count > 0]) < 1e-9
    # Indefinite terminal -> IndefiniteHessianError path (lqr_scan.hpp:150).
    leaf[tree.child_count == 0, :16] = -50.0 * np.eye(4).reshape(-1)
    got = B.lqr_tree(tree, 4, 2, stage, defect, leaf, 0.0, ctx=ctx)
    ref = O.lqr_tree(otree(tree), 4, 2, stage, defect, leaf, 0.0, 0)
    assert got["error"] != 0 and ref["error"] != 0


def test_lqr_tree_golden(ctx):
    fx = F.load("lqr_tree_two_stage_nx3nu2")
    meta = fx["meta"]
    tree = B.build_tree(meta["horizon"], [tuple(b) for b in meta["branchings"]])
    got = B.lqr_tree(tree, 3, 2, fx["stage"], fx["defect"], fx["leaf"], 0.0, fx["dx0"], ctx=ctx)
    nl = tree.child_count > 0
    for k, m in (("K", nl), ("k", nl), ("dx", slice(None)), ("du", nl)):
        assert _gen.rel_err(got[k][m], fx[k][m]) < 1e-9, k


# ------------------------------------------------------------- full solves
@pytest.mark.parametrize("name", F.scenario_names())
def test_solve_matches_reference_goldens(ctx, name):
    fx = F.load(name)
    p = F.build_product_problem(B, fx["meta"])
    res = B.solve(p, ctx=ctx)
    assert_same_solve(res, fx["report"], fx["x"], fx["u"], fx["records"])


@pytest.mark.parametrize("name", F.preset_names())
def test_solver_presets_match_reference_goldens(ctx, name):
    """smsilqr (team Riccati sweep everywhere, sequential line search) and
    sssilqr (single-shooting trials: nonlinear rollout under the feedback
    policies, solver.hpp:463-467 / problem.hpp:170-191) against the
    reference's own solves with those presets (bench.cpp:60-83)."""
    fx = F.load(name)
    meta = fx["meta"]
    p = F.build_product_problem(B, meta)
    o = B.SolverOptions()
    o.backward = ("scan-tree-riccati", "scan-condensed", "sequential-riccati")[meta["backward"]]
    o.forward = ("linear", "nonlinear")[meta["forward"]]
    o.line_search = ("parallel", "sequential")[meta["line_search"]]
    o.parallel = False
    res = B.solve(p, o, ctx=ctx)
    assert_same_solve(res, fx["report"], fx["x"], fx["u"], fx["records"])
    if meta["forward"] == 1:  # single shooting keeps the trajectory dynamically consistent
        assert res.report.final_defect_l1 <= 1e-12


@pytest.mark.parametrize("name", F.lq_names())
def test_lq_single_newton_step(ctx, name):
    """tests/acceptance_test.cpp:64-90 and test_solver.cpp:385-411."""
    fx = F.load(name)
    p = F.build_product_lq(B, fx)
    res = B.solve(p, ctx=ctx)
    assert res.report.status == B.CONVERGED and res.report.inner_iterations == 1
    assert res.report.iterations["alpha"][0] == 1.0
    assert res.report.final_defect_l1 <= 1e-10
    assert _gen.rel_err(res.trajectory.state, fx["x"]) <= 1e-9


def test_batch_perturbed_instances_match_oracle(ctx):
    """cfg4 semantics: independent perturbed instances, one block each."""
    seeds = list(range(42, 42 + 48))
    probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=s) for s in seeds]
    bt = B.Batch(ctx, probs, max_records=1000)
    bt.set_models()
    bt.solve()
    x = np.zeros((len(probs), bt.n, bt.nx))
    u = np.zeros((len(probs), bt.n, bt.nu))
    reps, _ = bt.results(x, u)
    for i, p in enumerate(probs):
        o = O.solve_problem(p)
        assert reps[i].status == o["status"]
        assert reps[i].inner_iterations == o["inner_iterations"], (i, reps[i].inner_iterations, o["inner_iterations"])
        assert reps[i].outer_iterations == o["outer_iterations"]
        np.testing.assert_array_equal(bt.records(i)["alpha"], o["records"]["alpha"])
        assert _gen.rel_err(x[i], o["x"]) <= TOL
        assert _gen.rel_err(u[i], o["u"]) <= TOL


@pytest.mark.parametrize("case", ["int_N500", "int_N1000", "ms_100_3x3", "latency_255"])
def test_grid_mode_solves_match_oracle(ctx, case):
    """Trees > 1024 nodes run on the whole GPU (cooperative grid)."""
    if case == "int_N500":
        p = B.build_intersection_case(B.intersection_spec(500, 10.0, 0.1), 2, 2)
    elif case == "int_N1000":
        p = B.build_intersection_case(B.intersection_spec(1000, 10.0, 0.1), 2, 2)
    elif case == "ms_100_3x3":
        p = B.build_multistage_case(B.multistage_spec(100, [(1, 3), (26, 3), (51, 3)]))
    else:
        p = B.build_latency_case(B.latency_spec(0.5, 255, 5.0, 0.05))
    res = B.solve(p, ctx=ctx)
    o = O.solve_problem(p)
    assert_same_solve(res, o, o["x"], o["u"], o["records"])


CFG2_STEPS = {1: [1], 2: [1, 34], 3: [1, 26, 51]}  # branch steps per depth (spread)


@pytest.mark.parametrize("depth", [1, 2, 3])
@pytest.mark.parametrize("arity", [2, 3, 4])
def test_cfg2_scenario_sweep_matches_oracle(ctx, arity, depth):
    """BASELINE cfg2: N=100, branching factor 2-4, branching depth 1-3 (2 to 64 leaves)."""
    p = B.build_multistage_case(B.multistage_spec(100, [(k, arity) for k in CFG2_STEPS[depth]]))
    assert p.tree.leaf_count() == arity ** depth
    res = B.solve(p, ctx=ctx)
    o = O.solve_problem(p)
    assert_same_solve(res, o, o["x"], o["u"], o["records"])


@pytest.mark.slow
def test_cfg3_full_size_matches_oracle(ctx):
    """BASELINE cfg3: 256 scenarios x N=500 (59,598 nodes), AL loop active."""
    p = B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)]))
    res = B.solve(p, ctx=ctx)
    assert res.report.status == B.CONVERGED
    assert res.report.outer_iterations >= 2  # the AL outer loop is active
    assert res.report.final_violation <= 1e-4
    assert res.report.final_defect_l1 <= 1e-8
    o = O.solve_problem(p)
    assert_same_solve(res, o, o["x"], o["u"], o["records"])


def test_converged_inputs_roll_out_to_states(ctx):
    """test_solver.cpp:521-534 at full cfg3-early size (127,062 nodes)."""
    p = B.build_multistage_case(B.multistage_spec(500, [(1, 4), (2, 4), (3, 4), (4, 4)]))
    res = B.solve(p, ctx=ctx)
    assert res.report.status == B.CONVERGED
    x = O.rollout(O.from_bmpc(p), res.trajectory.input)
    assert np.abs(x - res.trajectory.state).max() <= 1e-6
    ev = O.evaluate(O.from_bmpc(p), res.trajectory.state, res.trajectory.input)
    assert abs(ev["cost"] - res.report.final_cost) <= 1e-8 * abs(ev["cost"])


def test_initial_inputs_and_options(ctx):
    fx = F.load("intersection_20_4s")
    p = F.build_product_problem(B, fx["meta"])
    op = O.from_bmpc(p)
    # Warm start from the reference's own solution (solver.hpp:604-610).
    res = B.solve(p, initial_inputs=fx["u"], ctx=ctx)
    o = O.solve(op, u_init=fx["u"])
    assert_same_solve(res, o, o["x"], o["u"], o["records"])
    # Capped outer loop -> max-iter status; fewer alpha levels.
    opts = B.SolverOptions(max_outer_iterations=1, alpha_levels=4)
    res = B.solve(p, opts, ctx=ctx)
    o = O.solve(op, O.default_options(max_outer_iterations=1, alpha_levels=4))
    assert res.report.status == o["status"] == B.MAX_ITERATIONS
    assert_same_solve(res, o, o["x"], o["u"], o["records"])


def test_nonfinite_rollout_raises(ctx):
    """problem.hpp:160-162: non-finite initial rollout throws out of solve."""
    p = B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2)
    u = np.zeros((p.tree.node_count, 2))
    u[3, 0] = np.inf
    with pytest.raises(RuntimeError):
        B.solve(p, initial_inputs=u, ctx=ctx)


def test_deterministic_and_launch_shapes_agree(ctx):
    probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=s)
             for s in range(500, 516)]
    bt = B.Batch(ctx, probs)
    bt.set_models()
    outs = []
    for shape in [(256, 1), (256, 1), (128, 2), (64, 4)]:
        bt.set_launch(*shape)
        bt.solve()
        x = np.zeros((len(probs), bt.n, bt.nx))
        reps, _ = bt.results(x)
        outs.append((x, [r.inner_iterations for r in reps]))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])  # run-to-run bitwise deterministic
    for x, it in outs[2:]:
        assert it == outs[0][1]
        assert _gen.rel_err(x, outs[0][0]) <= 1e-10


def test_line_search_rounds_do_not_change_results():
    """Evaluating the step sizes in rounds (stop at the first round holding an
    accepted alpha) returns exactly what the all-at-once parallel search does."""
    probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=s)
             for s in (601, 622, 3409, 4035)]  # 3409 / 4035: long AL runs with rejected steps
    outs = {}
    for blk in (0, 1, 2, 3, 11):
        c = B.Context(0)
        B.set_line_search_block(c, blk)
        bt = B.Batch(c, probs, max_records=1000)
        bt.set_models()
        bt.solve()
        x = np.zeros((len(probs), bt.n, bt.nx))
        u = np.zeros((len(probs), bt.n, bt.nu))
        reps, _ = bt.results(x, u)
        recs = [bt.records(i) for i in range(len(probs))]
        outs[blk] = (x, u, reps, recs)
    x0, u0, r0, rec0 = outs[0]
    assert all(r.alpha_evals == 11 * r.n_records for r in r0)
    for blk, (x, u, reps, recs) in outs.items():
        np.testing.assert_array_equal(x, x0)
        np.testing.assert_array_equal(u, u0)
        for a, b, ra, rb in zip(reps, r0, recs, rec0):
            assert (a.status, a.inner_iterations, a.outer_iterations, a.n_records) == \
                (b.status, b.inner_iterations, b.outer_iterations, b.n_records)
            assert a.final_cost == b.final_cost
            for k in ra:
                np.testing.assert_array_equal(ra[k], rb[k])
        if blk == 1:  # one alpha per round: evaluations = accepted level + 1 (all 11 when rejected)
            for a, ra in zip(reps, recs):
                lv = np.where(ra["accepted"] > 0, -np.log2(np.where(ra["alpha"] > 0, ra["alpha"], 1.0)), 10)
                assert a.alpha_evals == float((lv + 1).sum())


def test_structured_expansion_matches_dense(ctx, monkeypatch):
    """Diagonal weights take the zero-skipping unicycle expansion; it must be
    bit-identical to the dense chain rule."""
    probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=s)
             for s in (7, 601, 3409)]
    probs.append(B.build_latency_case(B.latency_spec(0.5)))
    outs = []
    for dense in (False, True):
        if dense:
            monkeypatch.setenv("BMPC_DENSE_MODEL", "1")
        else:
            monkeypatch.delenv("BMPC_DENSE_MODEL", raising=False)
        res = []
        for p in probs:
            bt = B.Batch(ctx, [p], max_records=1000)
            bt.set_models()
            bt.solve()
            x = np.zeros((1, bt.n, bt.nx))
            u = np.zeros((1, bt.n, bt.nu))
            reps, _ = bt.results(x, u)
            res.append((x, u, reps[0], bt.records(0)))
        outs.append(res)
    for (xa, ua, ra, reca), (xb, ub, rb, recb) in zip(*outs):
        np.testing.assert_array_equal(xa, xb)
        np.testing.assert_array_equal(ua, ub)
        assert (ra.inner_iterations, ra.outer_iterations, ra.final_cost) == \
            (rb.inner_iterations, rb.outer_iterations, rb.final_cost)
        for k in reca:
            np.testing.assert_array_equal(reca[k], recb[k])


def test_probe_schedule_is_bit_identical():
    """Suspending every solve after a few passes, reordering and resuming it
    in a second launch gives exactly the single-launch results."""
    probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=9000 + s)
             for s in range(200)]
    outs = {}
    for probe in (0, 1, 3, 10):
        c = B.Context(0)
        B.set_schedule(c, probe)
        bt = B.Batch(c, probs, max_records=600)
        bt.set_models()
        bt.set_launch(256, 1)  # one wave = 148 instances < 200: the schedule engages
        n0 = c.launches
        bt.solve()
        launches = c.launches - n0
        x = np.zeros((len(probs), bt.n, bt.nx))
        u = np.zeros((len(probs), bt.n, bt.nu))
        reps, _ = bt.results(x, u)
        outs[probe] = (x, u, reps, [bt.records(i, 600) for i in (0, 17, 199)], launches)
    assert outs[0][4] == 1 and outs[3][4] == 4  # probe, order, main (150-pass budget), finish
    x0, u0, r0, rec0, _ = outs[0]
    for probe, (x, u, reps, recs, _) in outs.items():
        np.testing.assert_array_equal(x, x0)
        np.testing.assert_array_equal(u, u0)
        for a, b in zip(reps, r0):
            assert (a.status, a.inner_iterations, a.outer_iterations, a.n_records, a.alpha_evals) == \
                (b.status, b.inner_iterations, b.outer_iterations, b.n_records, b.alpha_evals)
            assert a.final_cost == b.final_cost and a.final_violation == b.final_violation
        for ra, rb in zip(recs, rec0):
            for k in ra:
                np.testing.assert_array_equal(ra[k], rb[k])


def test_results_as_array_matches_reports(ctx):
    probs = [B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2, perturb_seed=s) for s in range(6)]
    bt = B.Batch(ctx, probs)
    bt.set_models()
    bt.solve()
    reps, _ = bt.results()
    arr, _ = bt.results(as_array=True)
    assert len(arr) == len(reps)
    for r, a in zip(reps, arr):
        assert (r.status, r.inner_iterations, r.outer_iterations, r.n_records) == \
            (a["status"], a["inner_iterations"], a["outer_iterations"], a["n_records"])
        assert r.final_cost == a["final_cost"] and r.alpha_evals == a["alpha_evals"]


def test_set_initial_states_matches_full_upload(ctx):
    """Receding-horizon call: the scenario stays resident, only x0 changes."""
    spec = B.intersection_spec(20, 4.0, 0.4)
    pert = [B.build_intersection_case(spec, 2, 2, perturb_seed=s) for s in range(5)]
    base = [B.build_intersection_case(spec, 2, 2) for _ in range(5)]
    outs = []
    for probs, x0 in ((pert, None), (base, np.array([p.initial_state for p in pert]))):
        bt = B.Batch(ctx, probs)
        bt.set_models()
        if x0 is not None:
            assert bt.set_initial_states(x0) == 5 * 4 * 8
        bt.solve()
        x = np.zeros((5, bt.n, bt.nx))
        arr, _ = bt.results(x, as_array=True)
        outs.append((x, arr["inner_iterations"].copy(), arr["final_cost"].copy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])


def test_native_library_loaded(ctx):
    """The CUDA path is the one that ran: the in-tree .so is mapped and
    launched kernels."""
    p = B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2)
    n0 = ctx.launches
    B.solve(p, ctx=ctx)
    assert ctx.launches >= n0 + 1  # the solve (+ the result pack kernel)
    maps = open("/proc/self/maps").read()
    assert "libbmpc_b200.so" in maps


def test_single_shooting_batch_schedule_and_singles_agree():
    """sssilqr over a batch larger than one wave (probe / order / main /
    finish launches of the single-shooting kernel): bit-identical to the
    one-launch FIFO batch and to single solves, and instance 0 (seed 42)
    matches the reference's own sssilqr solve."""
    probs = [B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=42 + s)
             for s in range(400)]
    o = B.SolverOptions(backward="sequential-riccati", forward="nonlinear", line_search="sequential", parallel=False)
    outs = {}
    for probe in (0, 10):
        c = B.Context(0)
        B.set_schedule(c, probe)
        bt = B.Batch(c, probs, max_records=600)
        bt.set_models()
        bt.solve(o)
        x = np.zeros((len(probs), bt.n, bt.nx))
        u = np.zeros((len(probs), bt.n, bt.nu))
        reps, _ = bt.results(x, u)
        outs[probe] = (x, u, reps, bt.records(0, 600))
    x0, u0, r0, rec0 = outs[0]
    x1, u1, r1, _ = outs[10]
    np.testing.assert_array_equal(x1, x0)
    np.testing.assert_array_equal(u1, u0)
    assert [(a.status, a.inner_iterations, a.outer_iterations) for a in r1] == \
        [(a.status, a.inner_iterations, a.outer_iterations) for a in r0]
    fx = F.load("preset_sssilqr_cfg4_instance_seed42")
    assert (r0[0].inner_iterations, r0[0].outer_iterations) == \
        (fx["report"]["inner_iterations"], fx["report"]["outer_iterations"])
    np.testing.assert_array_equal(rec0["alpha"], fx["records"]["alpha"])
    assert _gen.rel_err(x0[0], fx["x"]) <= TOL and _gen.rel_err(u0[0], fx["u"]) <= TOL
    ctx = B.Context(0)
    for i in (0, 7, 399):
        r = B.solve(probs[i], o, ctx=ctx)
        np.testing.assert_array_equal(r.trajectory.state, x0[i])
        assert r.report.inner_iterations == r0[i].inner_iterations
