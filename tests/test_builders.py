"""CPU: the product's host-side tree and scenario builders (C ABI
bmpc_tree_build / bmpc_scenario_build) reproduce the reference's
build_tree / build_*_case outputs bit for bit (topology
bit-exact), and reject the specs the reference rejects."""
import numpy as np
import pytest

import _fixtures as F
import _oracle as O
import paper_2506_13624_b200 as B


@pytest.mark.parametrize("name", F.scenario_names())
def test_scenario_builders_bitwise_equal_reference(name):
    fx = F.load(name)
    p = F.build_product_problem(B, fx["meta"])
    a = p.arrays()
    np.testing.assert_array_equal(p.tree.parent, fx["prob_parent"])
    np.testing.assert_array_equal(p.tree.time_step, fx["prob_time_step"])
    np.testing.assert_array_equal(p.tree.weight, fx["prob_weight"])
    np.testing.assert_array_equal(a["initial_state"], fx["prob_initial_state"])
    np.testing.assert_array_equal(a["reference"], fx["prob_reference"])
    np.testing.assert_array_equal(a["vehicles"], fx["prob_vehicles"])


@pytest.mark.parametrize("horizon,br", [
    (6, [(4, 2, [0.5, 0.5])]), (7, [(3, 2, [0.5, 0.5])]), (5, []), (6, [(2, 2), (4, 3, [0.2, 0.3, 0.5])]),
    (100, [(1, 4), (26, 4), (51, 4)]), (500, [(1, 4), (2, 4), (3, 4), (4, 4)]),
])
def test_tree_equals_oracle_build_tree(horizon, br):
    t = B.build_tree(horizon, br)
    o = O.build_tree(horizon, br)
    np.testing.assert_array_equal(t.parent, o["parent"])
    np.testing.assert_array_equal(t.time_step, o["time_step"])
    np.testing.assert_array_equal(t.weight, o["weight"])
    np.testing.assert_array_equal(t.first_child, o["first_child"])
    np.testing.assert_array_equal(t.child_count, o["nchild"])
    np.testing.assert_array_equal(t.step_begin, o["step_begin"])


def test_tree_kats():
    # tests/test_tree.cpp:27-99
    t = B.build_tree(6, [(4, 2, [0.5, 0.5])])
    assert (t.node_count, t.leaf_count(), t.last_branch_step, t.horizon) == (9, 2, 4, 6)
    t = B.build_tree(7, [(3, 2, [0.5, 0.5])])
    assert t.node_count == 12 and list(t.leaves) == [10, 11]
    t = B.build_tree(6, [(2, 2, [0.5, 0.5]), (4, 2, [0.5, 0.5])])
    for k in range(t.horizon + 1):
        assert abs(t.weight[t.step_begin[k]:t.step_begin[k + 1]].sum() - 1.0) < 1e-12
    for i in range(1, t.node_count):
        assert t.parent[i] < i and t.time_step[t.parent[i]] == t.time_step[i] - 1


@pytest.mark.parametrize("horizon,br", [
    (5, [(5, 2)]), (5, [(1, 2, [0.6, 0.6])]), (5, [(1, 2, [1.2, -0.2])]), (5, [(2, 2), (2, 2)]), (0, []),
])
def test_tree_rejects_invalid_specs(horizon, br):
    with pytest.raises(ValueError):
        B.build_tree(horizon, br)


def test_scenario_rejects_invalid():
    # tests/test_models.cpp:88-89, :306-308
    with pytest.raises(ValueError):
        B.build_intersection_case(B.intersection_spec(), 2, 4)
    with pytest.raises(ValueError):
        B.build_latency_case(B.latency_spec(0.05, 255, 5.0, 0.05))


def test_intersection_shapes():
    # tests/test_models.cpp:76-90 and :135-149
    for v1, v2 in [(1, 2), (2, 2), (2, 3), (3, 3), (3, 4)]:
        p = B.build_intersection_case(B.intersection_spec(), v1, v2)
        assert p.tree.leaf_count() == v1 * v2 and p.tree.last_branch_step == 1 and p.tree.horizon == 63
    assert B.build_intersection_case(B.intersection_spec(), 1, 1).tree.last_branch_step == -1
    assert B.build_latency_case(B.latency_spec(0.5)).tree.step_begin is not None
    p1 = B.build_latency_case(B.latency_spec(0.5))
    assert p1.tree.leaf_count() == 4
    assert sorted(set(p1.tree.time_step[p1.tree.child_count > 1])) == [3, 26]
    p2 = B.build_latency_case(B.latency_spec(2.0))
    assert sorted(set(p2.tree.time_step[p2.tree.child_count > 1])) == [3, 102]


def test_config_node_counts():
    # SURVEY.md §8 node counts.
    assert B.build_intersection_case(B.intersection_spec(63, 10, 0.1), 2, 2).tree.node_count == 250
    assert B.build_intersection_case(B.intersection_spec(1000, 10, 0.1), 2, 2).tree.node_count == 3971
    assert B.build_multistage_case(B.multistage_spec(500, [(1, 4), (100, 4), (200, 4), (300, 4)])).tree.node_count \
        == 59598
    assert B.build_multistage_case(B.multistage_spec(500, [(1, 4), (2, 4), (3, 4), (4, 4)])).tree.node_count \
        == 127062
