"""`bench verify` on the GPU back end (paper_2506_13624_b200.verify). CPU:
the suites' host references (sequential tree Riccati, closed-loop rollout,
dense tree-QP KKT solve) against the C restatement of the reference. GPU:
every suite passes, and the scan-sign mutation trips scan-riccati."""
import io

import numpy as np
import pytest

import _oracle as O
import paper_2506_13624_b200 as B
from paper_2506_13624_b200 import cli
from paper_2506_13624_b200 import verify as V


@pytest.mark.parametrize("br,nx,nu", [([(2, 2, [0.5, 0.5]), (4, 3, [0.2, 0.3, 0.5])], 3, 2), ([], 4, 2),
                                      ([(0, 2, [0.5, 0.5]), (1, 2, [0.5, 0.5])], 2, 1)])
def test_host_references_match_oracle(br, nx, nu):
    rng = np.random.default_rng(3)
    tree = B.build_tree(6 if br else 9, br)
    stage, defect, leaf = V.random_tree_models(rng, tree, nx, nu)
    dx0 = rng.uniform(-1, 1, nx)
    P, p, K, k = V.host_riccati(tree, nx, nu, stage, defect, leaf)
    dx, du = V.host_rollout(tree, nx, nu, stage, defect, K, k, dx0)
    ot = dict(parent=tree.parent, first_child=tree.first_child, nchild=tree.child_count, weight=tree.weight,
              step_begin=tree.step_begin, horizon=tree.horizon, last_branch_step=tree.last_branch_step)
    ref = O.lqr_tree(ot, nx, nu, stage, defect, leaf, 0.0, 2, dx0)  # sequential Riccati strategy
    nl = tree.child_count > 0
    assert V._rel(P.reshape(len(P), -1, order="C").reshape(len(P), nx, nx).transpose(0, 2, 1).reshape(len(P), -1),
                  ref["P"]) < 1e-10
    assert V._rel(K.transpose(0, 2, 1).reshape(len(K), -1)[nl], ref["K"][nl]) < 1e-10
    assert V._rel(dx, ref["dx"]) < 1e-10 and V._rel(du[nl], ref["du"][nl]) < 1e-10
    # The tree QP's minimiser is the Riccati solution (x0 = dx0).
    xq, uq = V.dense_tree_qp(tree, nx, nu, stage, defect, leaf, dx0)
    assert V._rel(xq, dx) < 1e-9 and V._rel(uq[nl], du[nl]) < 1e-9


def test_verify_cli_selection_errors():
    assert cli.verify_command(["none"], "", out=io.StringIO()) == 0
    assert cli.verify_command([], "flip-everything", err=io.StringIO()) == 2
    assert cli.verify_command(["no-such-suite"], "", err=io.StringIO()) == 2


@pytest.mark.gpu
def test_all_suites_pass_on_gpu():
    res = V.run_suites(["all"])
    names = [r.name for r in res]
    assert {"scan-vs-riccati", "forward-scan-vs-rollout", "tree-riccati-vs-dense-qp", "cross-strategy"} <= set(names)
    for r in res:
        assert r.passed, r.line()


@pytest.mark.gpu
def test_scan_sign_mutation_is_caught():
    out = io.StringIO()
    assert cli.verify_command(["scan-riccati"], "scan-sign", out=out) == 1
    assert "[FAIL] scan-vs-riccati" in out.getvalue()
