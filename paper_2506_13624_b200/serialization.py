"""JSON wire formats of the reference (proj/include/bmpc/serialization.hpp),
same keys and value types, for the GPU solver's Python interface:

* tree spec      tree_spec_to_json / tree_from_json        (serialization.hpp:16-35)
* solver options solver_options_from_json / _to_json       (serialization.hpp:37-85)
* solve report   report_to_json                            (serialization.hpp:88-126)
* scenario spec  scenario_spec_to_json                     (serialization.hpp:128-154)
* problem dump   scenario_artifacts_to_json                (serialization.hpp:200-219)

nlohmann::json objects are key-sorted maps, so `dumps` sorts keys; every
double round-trips exactly (shortest representation both sides).
"""
import json
import math

from . import (SCENARIO_INTERSECTION, SCENARIO_LATENCY, STATUS_NAMES, BmpcProblem, ScenarioSpec, SolveReport,
               SolverOptions, TreeTopology, build_tree)

RECORD_KEYS = ("cost", "cost_al", "defect_l1", "violation", "alpha", "mu", "merit_before", "merit_after",
               "model_decrease", "max_feedforward", "regularization", "accepted", "outer")
TIME_KEYS = ("setup_s", "backward_p1_s", "backward_p2_s", "forward_s", "line_search_s", "total_s")

_OPT_INT = ("max_inner_iterations", "max_outer_iterations", "alpha_levels")
_OPT_FLOAT = ("armijo_beta", "merit_gamma", "merit_mu0", "merit_mu_init", "defect_epsilon", "tol_defect",
              "tol_cost", "tol_feedforward", "tol_constraint", "penalty_init", "penalty_growth", "penalty_max",
              "reg_init", "reg_min", "reg_growth", "reg_decay", "reg_max")
_STRATEGY = {"backward": ("scan-tree-riccati", "scan-condensed", "sequential-riccati"),
             "forward": ("linear", "nonlinear"), "line_search": ("parallel", "sequential"),
             "scan_order": ("tree", "sequential")}
_STRATEGY_NAME = {"backward": "backward strategy", "forward": "forward mode", "line_search": "line search mode",
                  "scan_order": "scan order"}


def dumps(j, indent=None) -> str:
    return json.dumps(j, indent=indent, sort_keys=True)


# --------------------------------------------------------------------- tree
def tree_branchings(tree: TreeTopology):
    """The construction spec of a built tree (TreeTopology::branchings,
    tree.hpp:43): kept by build_tree, else recovered from the topology."""
    br = getattr(tree, "branchings", None)
    if br is not None:
        return [(int(b[0]), int(b[1]), [float(w) for w in (b[2] if len(b) > 2 else [1.0 / b[1]] * b[1])])
                for b in br]
    out = []
    for k in range(tree.horizon):
        a = tree.step_begin[k]
        if tree.child_count[a] > 1:
            f, ar = tree.first_child[a], int(tree.child_count[a])
            out.append((k, ar, [float(tree.weight[f + c] / tree.weight[a]) for c in range(ar)]))
    return out


def tree_spec_to_json(tree: TreeTopology) -> dict:
    """{"horizon": N, "branchings": [{"step", "arity", "weights"}]} (serialization.hpp:16-22)."""
    return {"horizon": int(tree.horizon),
            "branchings": [{"step": s, "arity": a, "weights": w} for s, a, w in tree_branchings(tree)]}


def tree_from_json(j: dict) -> TreeTopology:
    """tree_from_json (serialization.hpp:24-35): build_tree of the spec."""
    br = [(int(b["step"]), int(b["arity"]), [float(w) for w in b["weights"]]) for b in j.get("branchings", [])]
    return build_tree(int(j["horizon"]), br)


# ------------------------------------------------------------------ options
def solver_options_from_json(j: dict) -> SolverOptions:
    """Flat key-value options; unknown keys and strategy names raise
    ValueError (the reference throws std::invalid_argument)."""
    o = SolverOptions()
    for key, value in j.items():
        if key in _STRATEGY:
            if value not in _STRATEGY[key]:
                raise ValueError("unknown %s: %s" % (_STRATEGY_NAME[key], value))
            setattr(o, key, value)
        elif key == "parallel":
            if not isinstance(value, bool):
                raise ValueError("option parallel must be a boolean")
            o.parallel = value
        elif key in _OPT_INT:
            if isinstance(value, bool) or not isinstance(value, int):
                raise ValueError("option %s must be an integer" % key)
            setattr(o, key, value)
        elif key in _OPT_FLOAT:
            if isinstance(value, bool) or not isinstance(value, (int, float)):
                raise ValueError("option %s must be a number" % key)
            setattr(o, key, float(value))
        else:
            raise ValueError("unknown solver option: " + key)
    return o


def solver_options_to_json(o: SolverOptions) -> dict:
    """Every option under the keys solver_options_from_json reads."""
    j = {k: getattr(o, k) for k in _STRATEGY}
    j["parallel"] = bool(o.parallel)
    j.update({k: int(getattr(o, k)) for k in _OPT_INT})
    j.update({k: float(getattr(o, k)) for k in _OPT_FLOAT})
    return j


# ------------------------------------------------------------------- report
def report_to_json(report: SolveReport) -> dict:
    """Convergence report as per-iteration arrays (serialization.hpp:88-126)."""
    its = report.iterations or {}
    n = report.n_records if its else 0
    arrays = {}
    for k in RECORD_KEYS:
        v = its.get(k, [])[:n]
        arrays[k] = [bool(x) for x in v] if k == "accepted" else [int(x) for x in v] if k == "outer" else \
            [float(x) for x in v]
    return {"status": STATUS_NAMES[report.status], "message": report.message,
            "inner_iterations": int(report.inner_iterations), "outer_iterations": int(report.outer_iterations),
            "final_cost": float(report.final_cost), "final_violation": float(report.final_violation),
            "final_defect_l1": float(report.final_defect_l1), "iterations": arrays,
            "times": {k: float(report.times.get(k, 0.0)) for k in TIME_KEYS}}


# ---------------------------------------------------------------- scenarios
_SPEC_DEFAULTS = {"state_weights": [1.0, 1.0, 0.1, 0.1], "input_weights": [0.5, 0.5],
                  "terminal_weights": [1.0, 1.0, 0.1, 0.1], "accel_limit": 3.0, "yaw_rate_limit": 0.5,
                  "safety_radius": 3.0, "prediction_tau": 1.5, "reference_turn_rate": 0.4,
                  "backup_deceleration": 3.0, "continue_deceleration": 2.5}  # ScenarioSpec, scenarios.hpp:25-47


def scenario_spec_to_json(spec: ScenarioSpec) -> dict:
    """scenario_spec_to_json (serialization.hpp:128-154) of the specs the
    builders take: intersection_spec (scenarios.hpp:178-197: ego and the
    oncoming / lead vehicles) and latency_spec (scenarios.hpp:300-317)."""
    if spec.family == SCENARIO_LATENCY:
        ego = [0.0, 0.0, 0.0, 10.0]
        veh = [{"position": [30.0, 0.0], "heading": 0.0, "speed": 8.0, "target_speeds": [8.0, 0.0]}]
    elif spec.family == SCENARIO_INTERSECTION:
        ego = [0.0, -20.0, math.pi / 2.0, 5.0]
        veh = [{"position": [-3.5, 30.0], "heading": -math.pi / 2.0, "speed": 8.0,
                "target_speeds": [8.0, 2.0, 5.0, 3.5]},
               {"position": [0.0, -10.0], "heading": math.pi / 2.0, "speed": 5.0,
                "target_speeds": [5.0, 1.0, 3.0, 2.0]}]
    else:
        raise ValueError("scenario_spec_to_json: the multistage family has no reference spec")
    d = dict(_SPEC_DEFAULTS)
    d.update({"total_time": float(spec.total_time), "shared_times": [float(t) for t in spec.shared_times],
              "horizon": int(spec.horizon), "ego_start": ego, "vehicles": veh})
    return d


def scenario_artifacts_to_json(problem: BmpcProblem) -> dict:
    """Reproducibility dump of a built scenario problem: tree spec, per node
    step / parent / weight / tracking reference / predicted vehicle
    positions (serialization.hpp:200-219)."""
    a, t = problem.arrays(), problem.tree
    if "reference" not in a:
        raise ValueError("scenario_artifacts_to_json: not a scenario problem")
    veh = a.get("vehicles")
    nodes = [{"step": int(t.time_step[i]), "parent": int(t.parent[i]), "weight": float(t.weight[i]),
              "reference": [float(v) for v in a["reference"][i]],
              "vehicles": [[float(v) for v in xy] for xy in veh[i]] if veh is not None else []}
             for i in range(t.node_count)]
    return {"tree": tree_spec_to_json(t), "nodes": nodes}


__all__ = ["dumps", "tree_spec_to_json", "tree_from_json", "solver_options_from_json", "solver_options_to_json",
           "report_to_json", "scenario_spec_to_json", "scenario_artifacts_to_json", "tree_branchings",
           "RECORD_KEYS", "TIME_KEYS"]
