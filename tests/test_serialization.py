"""JSON wire formats (paper_2506_13624_b200.serialization) against the
reference's serialization.hpp: its own tests (tests/test_serialization.cpp)
restated, plus documents written by the reference itself
(tests/golden/gen_{tree,report}.json.gz from oracle/_ref/gen_ref)."""
import gzip
import json
import os

import numpy as np
import pytest

import paper_2506_13624_b200 as B
from paper_2506_13624_b200 import serialization as S

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _ref_doc(name):
    with gzip.open(os.path.join(GOLDEN, "gen_%s.json.gz" % name), "rt") as f:
        return json.load(f)


def test_tree_spec_round_trip():  # test_serialization.cpp:11-23
    tree = B.build_tree(6, [(2, 2, [0.5, 0.5]), (4, 3, [0.2, 0.3, 0.5])])
    j = S.tree_spec_to_json(tree)
    assert j == _ref_doc("tree")  # the reference's own tree_spec_to_json document
    back = S.tree_from_json(json.loads(S.dumps(j)))
    assert back.node_count == tree.node_count and back.horizon == tree.horizon
    assert back.last_branch_step == tree.last_branch_step
    np.testing.assert_array_equal(back.parent, tree.parent)
    np.testing.assert_array_equal(back.leaves, tree.leaves)
    np.testing.assert_array_equal(back.weight, tree.weight)


def test_tree_spec_of_scenario_tree():
    p = B.build_latency_case(B.latency_spec(0.5, 63, 5.0, 0.05))  # branchings recovered from the topology
    j = S.tree_spec_to_json(p.tree)
    assert j["horizon"] == 63 and [(b["step"], b["arity"], b["weights"]) for b in j["branchings"]] == \
        [(1, 2, [0.5, 0.5]), (6, 2, [0.5, 0.5])]
    back = S.tree_from_json(j)
    np.testing.assert_array_equal(back.parent, p.tree.parent)


def test_solver_options_flat_keys():  # test_serialization.cpp:25-43
    o = S.solver_options_from_json({"backward": "scan-condensed", "forward": "nonlinear", "line_search": "sequential",
                                    "max_inner_iterations": 17, "tol_constraint": 1e-3, "penalty_init": 5.0})
    assert (o.backward, o.forward, o.line_search) == ("scan-condensed", "nonlinear", "sequential")
    assert o.max_inner_iterations == 17 and o.tol_constraint == 1e-3 and o.penalty_init == 5.0
    with pytest.raises(ValueError):
        S.solver_options_from_json({"not_an_option": 1})
    with pytest.raises(ValueError):
        S.solver_options_from_json({"backward": "mystery"})
    c = o._c()  # every strategy runs on the GPU (enum numbering of solver.hpp:23-26)
    assert (c.backward, c.forward, c.line_search) == (1, 1, 1)
    o.forward = "sideways"
    with pytest.raises(ValueError):
        o._c()
    back = S.solver_options_from_json(S.solver_options_to_json(B.SolverOptions(reg_init=1e-3, alpha_levels=7)))
    assert back == B.SolverOptions(reg_init=1e-3, alpha_levels=7)


def test_scenario_spec_json():  # test_serialization.cpp:45-57 (round trip of every field)
    spec = B.intersection_spec(31, 5.0, 0.2)
    j = S.scenario_spec_to_json(spec)
    assert j["horizon"] == 31 and j["total_time"] == 5.0 and j["shared_times"] == [0.2]
    assert len(j["vehicles"]) == 2 and j["ego_start"][1] == -20.0
    back = S.scenario_spec_from_json(json.loads(S.dumps(j)))
    assert S.scenario_spec_to_json(back) == j
    # Defaults are ScenarioSpec{}'s (no vehicles), not a preset's.
    d = S.scenario_spec_from_json({"horizon": 12})
    assert d.horizon == 12 and d.vehicles == () and d.total_time == 10.0 and d.shared_times == (0.1,)
    with pytest.raises(IndexError):  # the reference's .at(3) throws out_of_range
        S.scenario_spec_from_json({"ego_start": [0.0, 1.0, 2.0]})


@pytest.mark.parametrize("kind", ["intersection", "latency"])
def test_scenario_spec_from_json_builds_reference_problem(kind):
    """A scene given as JSON — its own vehicles, target speeds, weights, limits
    and timing — built by the in-library builders equals the reference
    builders' problem from the same JSON (oracle/_ref/gen_ref spec-*,
    tests/make_golden_specs.py): spec round trip and every node's step,
    parent, weight, tracking reference and vehicle predictions."""
    with gzip.open(os.path.join(GOLDEN, f"gen_spec_{kind}.json.gz"), "rt") as f:
        ref = json.load(f)
    spec = S.scenario_spec_from_json(ref["input_spec"])
    assert S.scenario_spec_to_json(spec) == ref["spec"]
    if kind == "intersection":
        p = B.build_intersection_case(spec, ref["v1_count"], ref["v2_count"])
    else:
        p = B.build_latency_case(spec)
    got = S.scenario_artifacts_to_json(p)
    assert got["tree"] == ref["problem"]["tree"]
    assert len(got["nodes"]) == len(ref["problem"]["nodes"])
    for a, b in zip(got["nodes"], ref["problem"]["nodes"]):
        assert a == b
    w = p.model
    assert tuple(w.state_weights)[::5] == spec.state_weights and w.safety_radius == spec.safety_radius
    np.testing.assert_array_equal(p.initial_state, spec.ego_start)


def test_scenario_builders_reject_bad_scenes():
    spec = B.intersection_spec()
    one = B.ScenarioSpec(vehicles=spec.vehicles[:1])
    with pytest.raises(ValueError, match="need 2 vehicles with enough targets"):
        B.build_intersection_case(one, 2, 2)
    short = B.dataclasses.replace(spec, vehicles=(spec.vehicles[0], B.SurroundingVehicle((0.0, -10.0), 1.5, 5.0,
                                                                                          (5.0, 1.0))))
    with pytest.raises(ValueError, match="need 2 vehicles with enough targets"):
        B.build_intersection_case(short, 2, 3)  # 6 leaves: the lead vehicle needs 3 target speeds
    lat = B.latency_spec(0.5)
    with pytest.raises(ValueError, match="need one vehicle with 2 targets"):
        B.build_latency_case(B.ScenarioSpec(shared_times=lat.shared_times, total_time=5.0, horizon=255,
                                            vehicles=spec.vehicles))


def test_report_iteration_arrays():  # test_serialization.cpp:59-76
    its = {k: np.zeros(2) for k in B.RECORD_FIELDS}
    its["cost"] = np.array([1.0, 0.5])
    its["alpha"] = np.array([1.0, 0.5])
    its["mu"] = np.array([1.5, 1.5])
    its["accepted"] = np.array([1, 1])
    rep = B.SolveReport(B.CONVERGED, "", 2, 1, 0.5, 0.0, 0.0, {}, its, 2)
    j = S.report_to_json(rep)
    assert j["status"] == "converged" and len(j["iterations"]["cost"]) == 2
    assert j["iterations"]["alpha"][1] == 0.5 and j["iterations"]["mu"][0] == 1.5
    assert j["iterations"]["accepted"] == [True, True]
    assert sorted(j) == sorted(_ref_doc("report"))  # same top-level schema as the reference's


def test_scenario_artifacts_dump():  # test_serialization.cpp:78-90
    p = B.build_intersection_case(B.intersection_spec(10), 1, 2)
    j = S.scenario_artifacts_to_json(p)
    assert j["tree"]["horizon"] == 10 and len(j["nodes"]) == p.tree.node_count
    assert len(j["nodes"][0]["vehicles"]) == 2
    assert abs(sum(n["weight"] for n in j["nodes"] if n["step"] == 10) - 1.0) < 1e-12


@pytest.mark.gpu
def test_report_json_matches_reference_solve():
    """report_to_json of the GPU cfg0 solve against the reference's own
    report_to_json of solve() on the same problem: identical schema, counts,
    status and acceptance / outer sequences; values within the parity bar."""
    p = B.build_intersection_case(B.intersection_spec(63, 10.0, 0.1), 2, 2)
    got = json.loads(S.dumps(S.report_to_json(B.solve(p).report)))
    want = _ref_doc("report")
    assert sorted(got) == sorted(want) and sorted(got["iterations"]) == sorted(want["iterations"])
    for k in ("status", "message", "inner_iterations", "outer_iterations"):
        assert got[k] == want[k], k
    for k in ("accepted", "outer", "alpha"):
        assert got["iterations"][k] == want["iterations"][k], k
    for k in ("cost", "cost_al", "merit_before", "merit_after"):
        np.testing.assert_allclose(got["iterations"][k], want["iterations"][k], rtol=1e-7, atol=0)
    assert abs(got["final_cost"] - want["final_cost"]) <= 1e-8 * abs(want["final_cost"])
    assert got["times"]["total_s"] > 0.0
