"""First GPU parity checks: kernel-level LQR tree and full solves vs the
reference (oracle/_ref). Marked gpu."""
import numpy as np
import pytest

import _gen
import _refbind as R
import paper_2506_13624_b200 as B

pytestmark = pytest.mark.gpu

TREES = [
    (6, [(4, 2, [0.5, 0.5])]),
    (6, [(2, 2, [0.5, 0.5]), (4, 3, [0.2, 0.3, 0.5])]),
    (5, []),
    (5, [(4, 3, [0.3, 0.3, 0.4])]),
    (40, [(3, 2, [0.5, 0.5]), (17, 2, [0.25, 0.75])]),
]


@pytest.mark.parametrize("grid", [False, True])
@pytest.mark.parametrize("dims", [(3, 2), (4, 2), (2, 1), (8, 4)])
@pytest.mark.parametrize("ti", range(len(TREES)))
def test_lqr_tree_matches_reference(ti, dims, grid):
    horizon, br = TREES[ti]
    nx, nu = dims
    rng = np.random.default_rng(100 + ti)
    tree = B.build_tree(horizon, br)
    stage, defect, leaf = _gen.random_tree_models(rng, tree, nx, nu)
    dx0 = rng.uniform(-1, 1, nx)
    got = B.lqr_tree(tree, nx, nu, stage, defect, leaf, 0.0, dx0, grid=grid)
    ref = R.lqr_tree(br, horizon, nx, nu, stage, defect, leaf, 0.0, 0, dx0)
    assert got["error"] == ref["error"] == 0
    nl = tree.child_count > 0
    for key, mask in (("K", nl), ("k", nl), ("dx", slice(None)), ("du", nl), ("P", slice(None)), ("p", slice(None))):
        assert _gen.rel_err(got[key][mask], ref[key][mask]) < 1e-9, key
    assert abs(got["a1"] - ref["a1"]) <= 1e-9 * (1 + abs(ref["a1"]))
    assert abs(got["a2"] - ref["a2"]) <= 1e-9 * (1 + abs(ref["a2"]))
    assert abs(got["max_feedforward"] - ref["max_feedforward"]) <= 1e-9 * (1 + ref["max_feedforward"])


def test_intersection_cfg0_matches_reference():
    p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)
    res = B.solve(p)
    x, u, rep, rec = R.solve(R.scenario(0, 63))
    print(res.report.status, res.report.inner_iterations, res.report.outer_iterations, rep)
    assert res.report.status == rep["status"] == 0
    assert res.report.inner_iterations == rep["inner_iterations"]
    assert res.report.outer_iterations == rep["outer_iterations"]
    np.testing.assert_array_equal(res.report.iterations["alpha"], rec["alpha"])
    assert _gen.rel_err(res.trajectory.state, x) < 1e-8
    assert _gen.rel_err(res.trajectory.input, u) < 1e-8
    assert abs(res.report.final_cost - rep["final_cost"]) <= 1e-8 * abs(rep["final_cost"])
