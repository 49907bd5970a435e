"""Error semantics at the drop-in boundary, against the reference's catch and
throw sites:

* nonlinear_rollout throws at the FIRST node in index order whose successor
  state is non-finite (problem.hpp:157-162);
* linearize checks every node's expansion in index order first
  ("non-finite expansion" / "non-finite terminal expansion", solver.hpp:
  102-105, 130-133), and solve() turns the exception into status error with
  that message (solver.hpp:629-636);
* Batch.results only accepts float64 C-contiguous arrays of the exact shape
  (the C call memcpys into the raw buffers)."""
import numpy as np
import pytest

import _fixtures as F
import paper_2506_13624_b200 as B

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return B.Context(0)


def test_rollout_error_reports_first_node(ctx):
    p = B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2)
    u = np.zeros((p.tree.node_count, 2))
    u[9, 0] = np.inf  # a later node fails too ...
    u[3, 0] = np.inf  # ... but node 3 comes first in index order
    with pytest.raises(RuntimeError, match=r"nonlinear_rollout: non-finite state at node 3$"):
        B.solve(p, initial_inputs=u, ctx=ctx)


def _lq(name="lq_6_branch2_nx3nu2"):
    fx = F.load(name)
    meta = fx["meta"]
    tree = B.build_tree(meta["horizon"], [tuple(b) for b in meta["branchings"]])
    return tree, meta, fx


def test_linearize_error_first_expansion_node(ctx):
    tree, meta, fx = _lq()
    nx, nu = meta["nx"], meta["nu"]
    stage = fx["stage"].copy()
    q_off = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx  # A B c Q R M | q
    stage[4, q_off] = np.nan
    stage[2, q_off] = np.nan
    p = B.lq_problem(tree, nx, nu, fx["x0"], stage, fx["leaf"])
    res = B.solve(p, ctx=ctx)
    assert res.report.status == B.ERROR
    assert res.report.message == "linearize: non-finite expansion at node 2"


def test_linearize_error_terminal_expansion(ctx):
    tree, meta, fx = _lq()
    nx, nu = meta["nx"], meta["nu"]
    leaf = fx["leaf"].copy()
    last = tree.node_count - 1  # a leaf
    leaf[last, 0] = np.nan
    p = B.lq_problem(tree, nx, nu, fx["x0"], fx["stage"], leaf)
    res = B.solve(p, ctx=ctx)
    assert res.report.status == B.ERROR
    assert res.report.message == f"linearize: non-finite terminal expansion at node {last}"


def test_batch_results_rejects_bad_buffers(ctx):
    probs = [B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2, perturb_seed=s) for s in (1, 2)]
    bt = B.Batch(ctx, probs)
    bt.set_models()
    bt.solve()
    n = bt.n
    for bad in (np.zeros((2, n, 4), np.float32), np.zeros((2, n, 3)), np.zeros((2, 4, n)).transpose(0, 2, 1),
                np.zeros(2 * n * 4)):
        with pytest.raises(ValueError):
            bt.results(bad)
    x = np.zeros((2, n, 4))
    u = np.zeros((2, n, 2))
    reps, _ = bt.results(x, u)
    assert all(r.status == B.CONVERGED for r in reps)
    assert np.isfinite(x).all() and np.abs(x).sum() > 0


def test_ctx_destroyed_before_batch_is_safe():
    """bmpc_ctx_destroy with a live batch defers the free to the last
    bmpc_batch_destroy (garbage-collected bindings may finalize in any order)."""
    c = B.Context(0)
    bt = B.Batch(c, [B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2)])
    bt.set_models()
    B.lib().bmpc_ctx_destroy(c._h)  # what Context.__del__ does
    c._h = None
    bt.solve()
    reps, _ = bt.results()
    assert reps[0].status == B.CONVERGED
    del bt  # frees the batch, then the pending ctx
