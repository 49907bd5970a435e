"""CPU: the C oracle (oracle/bmpc_oracle.c) pinned against the reference —
its golden fixtures (tests/golden, generated from oracle/_ref) and the
known-answer tests of the reference's own test suite."""
import os

import numpy as np
import pytest

import _fixtures as F
import _oracle as O

REF_SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                      "libbmpc_ref.so")


def oracle_problem_from_fixture(fx):
    """Oracle problem built from the reference's own dumped problem data."""
    meta = fx["meta"]
    br = [tuple(b) if len(b) > 2 else (b[0], b[1]) for b in meta["branchings"]]
    if meta["family"] == 0:
        v = meta["v"][0] * meta["v"][1]
        dt = meta["total_time"] / meta["horizon"]
        step = int(np.round(meta["shared"][0] / dt))
        br = [(step, v)] if v > 1 else []
    elif meta["family"] == 1:
        dt = meta["total_time"] / meta["horizon"]
        br = [(int(np.round(meta["shared"][0] / dt)), 2), (int(np.round(meta["shared"][1] / dt)), 2)]
    tree = O.build_tree(meta["horizon"], br)
    np.testing.assert_array_equal(tree["parent"], fx["prob_parent"])
    np.testing.assert_array_equal(tree["weight"], fx["prob_weight"])
    W = lambda d: np.diag(d).reshape(-1, order="F")
    veh = fx["prob_vehicles"]
    return O.Problem(tree, 1, 4, 2, fx["prob_initial_state"], dt=float(meta["total_time"] / meta["horizon"]),
                     Wx=W([1.0, 1.0, 0.1, 0.1]), Wu=W([0.5, 0.5]), Wf=W([1.0, 1.0, 0.1, 0.1]), a_max=3.0,
                     w_max=0.5, radius=3.0, nv=veh.shape[1], reference=fx["prob_reference"], vehicles=veh)


@pytest.mark.parametrize("name", F.scenario_names())
def test_oracle_reproduces_reference_goldens(name):
    fx = F.load(name)
    out = O.solve(oracle_problem_from_fixture(fx))
    rep = fx["report"]
    assert out["status"] == rep["status"]
    assert out["inner_iterations"] == rep["inner_iterations"]
    assert out["outer_iterations"] == rep["outer_iterations"]
    assert out["n_records"] == rep["n_records"]
    # Same arithmetic order as the shim-built reference: bit-identical.
    np.testing.assert_array_equal(out["x"], fx["x"])
    np.testing.assert_array_equal(out["u"], fx["u"])
    for k, v in fx["records"].items():
        np.testing.assert_array_equal(out["records"][k], v, err_msg=k)
    assert out["final_cost"] == rep["final_cost"]


@pytest.mark.parametrize("name", F.lq_names())
def test_oracle_lq_generator_and_single_newton_step(name):
    fx = F.load(name)
    meta = fx["meta"]
    tree = O.build_tree(meta["horizon"], [tuple(b) for b in meta["branchings"]])
    x0, stage, leaf = O.random_lq(meta["seed"], tree, meta["nx"], meta["nu"])
    # libstdc++ mt19937_64 + uniform_real_distribution restated bit for bit.
    np.testing.assert_array_equal(x0, fx["x0"])
    np.testing.assert_array_equal(stage, fx["stage"])
    np.testing.assert_array_equal(leaf, fx["leaf"])
    out = O.solve(O.Problem(tree, 2, meta["nx"], meta["nu"], x0, lq_stage=stage, lq_leaf=leaf))
    # tests/acceptance_test.cpp:64-90: converged in one iteration at alpha = 1.
    assert out["status"] == 0 and out["inner_iterations"] == 1
    assert out["records"]["alpha"][0] == 1.0
    assert out["final_defect_l1"] <= 1e-10
    np.testing.assert_array_equal(out["x"], fx["x"])


def test_oracle_lqr_tree_golden():
    fx = F.load("lqr_tree_two_stage_nx3nu2")
    meta = fx["meta"]
    tree = O.build_tree(meta["horizon"], [tuple(b) for b in meta["branchings"]])
    out = O.lqr_tree(tree, 3, 2, fx["stage"], fx["defect"], fx["leaf"], 0.0, 0, fx["dx0"])
    for k in ("K", "k", "P", "p", "dx", "du"):
        np.testing.assert_allclose(out[k], fx[k], rtol=0, atol=1e-13, err_msg=k)
    assert out["error"] == 0


def scalar_stage(A, B, c, Q, R, M, q, r):
    return np.array([A, B, c, Q, R, M, q, r], np.float64)


def test_kat_init_and_combine_scalar():
    # tests/test_lqr_scan.cpp:54-61 and :112-121.
    e = np.zeros(5)
    assert O.lib().bo_init_bwd_element(1, 1, O._p(scalar_stage(1, 1, 0, 1, 1, 0, 0, 0)), O._p(e)) == 0
    np.testing.assert_array_equal(e, [1.0, 0.0, 1.0, 1.0, 0.0])  # P p C A c
    out = np.zeros(5)
    a = np.array([1.0, 0.0, 1.0, 1.0, 0.0])
    assert O.lib().bo_combine_bwd(1, O._p(a), O._p(a), O._p(out)) == 0
    assert abs(out[0] - 1.5) < 1e-15 and abs(out[2] - 1.5) < 1e-15
    assert abs(abs(out[3]) - 0.5) < 1e-15 and abs(out[1]) < 1e-15 and abs(out[4]) < 1e-15


def test_kat_singular_R_is_factorization_error():
    # tests/test_lqr_scan.cpp:63-71: R = 0 is rejected.
    e = np.zeros(5)
    assert O.lib().bo_init_bwd_element(1, 1, O._p(scalar_stage(1, 1, 0, 1, 0.0, 0, 0, 0)), O._p(e)) == 2


def path_models(N, stage):
    tree = O.build_tree(N, [])
    n = N + 1
    st = np.tile(stage, (n, 1))
    return tree, st, np.zeros((n, 1))


def test_kat_long_chain_golden_ratio():
    # tests/test_lqr_scan.cpp:261-278: N = 511 scalar chain -> golden ratio.
    tree, st, df = path_models(511, scalar_stage(1, 1, 0, 1, 1, 0, 0, 0))
    leaf = np.zeros((512, 2))
    out = O.lqr_tree(tree, 1, 1, st, df, leaf)
    assert abs(out["P"][0, 0] - (1 + 5 ** 0.5) / 2) < 1e-12


def test_kat_feedback_scalar():
    # tests/test_lqr_scan.cpp:289-295: K = -0.5 with P_next = 1.
    tree, st, df = path_models(1, scalar_stage(1, 1, 0, 1, 1, 0, 0, 0))
    leaf = np.array([[0, 0], [1.0, 0.0]])
    out = O.lqr_tree(tree, 1, 1, st, df, leaf)
    assert abs(out["K"][0, 0] + 0.5) < 1e-15 and abs(out["k"][0, 0]) < 1e-15
    # tests/test_riccati.cpp:14-23: P0 = 1.5.
    assert abs(out["P"][0, 0] - 1.5) < 1e-15


def test_kat_indefinite_signals_regularization():
    # tests/test_lqr_scan.cpp:311-315: R + B'PB = -0.5 -> IndefiniteHessianError.
    tree, st, df = path_models(1, scalar_stage(1, 1, 0, 1, 0.5, 0, 0, 0))
    leaf = np.array([[0, 0], [-1.0, 0.0]])
    out = O.lqr_tree(tree, 1, 1, st, df, leaf)
    assert out["error"] == 1


def test_kat_scan_equals_sequential_riccati_grid():
    # verification.hpp:42-73 (scan vs Riccati <= 1e-8) on a reduced grid.
    rng = np.random.default_rng(12345)
    import _gen
    for nx, nu, N in [(2, 1, 8), (4, 2, 64), (8, 4, 64), (4, 2, 511)]:
        tree = O.build_tree(N, [])

        class T:  # minimal tree view for _gen
            node_count = N + 1
            child_count = tree["nchild"]
        st, df, lf = _gen.random_tree_models(rng, T, nx, nu)
        a = O.lqr_tree(tree, nx, nu, st, df, lf, 0.0, 0)
        b = O.lqr_tree(tree, nx, nu, st, df, lf, 0.0, 2)
        for i in range(N + 1):
            assert _gen.rel_err(a["P"][i], b["P"][i]) <= 1e-8
            assert _gen.rel_err(a["p"][i], b["p"][i]) <= 1e-8


def test_kat_mt19937_64_first_output():
    # std::mt19937_64 default seed 5489: first output 14514284786278117030.
    u = O.mt_uniform(5489, 1)[0]
    assert u == (14514284786278117030 / 2.0 ** 64) * 2.0 - 1.0


@pytest.mark.parametrize("horizon,br,nodes,leaves,nb", [
    (6, [(4, 2)], 9, 2, 4),                      # test_tree.cpp:27-33
    (7, [(3, 2)], 12, 2, 3),                     # :35-43 (leaves {10, 11})
    (5, [], 6, 1, -1),                           # :45-53
    (6, [(2, 2), (4, 2)], 15, 4, 4),             # :55-60
])
def test_kat_tree_counts(horizon, br, nodes, leaves, nb):
    t = O.build_tree(horizon, br)
    assert len(t["parent"]) == nodes
    assert int((t["nchild"] == 0).sum()) == leaves
    assert t["last_branch_step"] == nb
    if (horizon, nodes) == (7, 12):
        assert list(np.nonzero(t["nchild"] == 0)[0]) == [10, 11]


@pytest.mark.parametrize("horizon,br", [
    (5, [(5, 2)]), (5, [(1, 2, (0.6, 0.6))]), (5, [(1, 2, (1.2, -0.2))]), (5, [(2, 2), (2, 2)]), (0, []),
])
def test_kat_tree_rejects_invalid_specs(horizon, br):
    # tests/test_tree.cpp:151-158.
    with pytest.raises(ValueError):
        O.build_tree(horizon, br)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_perturbed():
    import _refbind as R
    import paper_2506_13624_b200 as B
    for seed in (101, 202):
        p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2, perturb_seed=seed)
        o = O.solve_problem(p)
        x, u, rep, rec = R.solve(R.scenario(0, 63, perturb_seed=seed))
        assert o["inner_iterations"] == rep["inner_iterations"]
        np.testing.assert_array_equal(o["x"], x)
