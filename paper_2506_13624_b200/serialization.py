"""JSON wire formats of the reference (proj/include/bmpc/serialization.hpp),
same keys and value types, for the GPU solver's Python interface:

* tree spec      tree_spec_to_json / tree_from_json        (serialization.hpp:16-35)
* solver options solver_options_from_json / _to_json       (serialization.hpp:37-85)
* solve report   report_to_json                            (serialization.hpp:88-126)
* scenario spec  scenario_spec_to_json / _from_json        (serialization.hpp:128-197)
* problem dump   scenario_artifacts_to_json                (serialization.hpp:200-219)

nlohmann::json objects are key-sorted maps, so `dumps` sorts keys; every
double round-trips exactly (shortest representation both sides).
"""
import dataclasses
import json

from . import (STATUS_NAMES, BmpcProblem, ScenarioSpec, SolveReport, SolverOptions, SurroundingVehicle,
               TreeTopology, build_tree)

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
_SPEC_SCALARS = ("accel_limit", "yaw_rate_limit", "safety_radius", "prediction_tau", "reference_turn_rate",
                 "backup_deceleration", "continue_deceleration")


def scenario_spec_to_json(spec: ScenarioSpec) -> dict:
    """scenario_spec_to_json (serialization.hpp:128-154): every field of the
    scene the builders take (timing, ego start, surrounding vehicles with
    their target speeds, tracking weights, limits, prediction constant and the
    reference shaping parameters)."""
    d = {"total_time": float(spec.total_time), "shared_times": [float(t) for t in spec.shared_times],
         "horizon": int(spec.horizon), "ego_start": [float(v) for v in spec.ego_start],
         "vehicles": [{"position": [float(v.position[0]), float(v.position[1])], "heading": float(v.heading),
                       "speed": float(v.speed), "target_speeds": [float(t) for t in v.target_speeds]}
                      for v in spec.vehicles],
         "state_weights": [float(v) for v in spec.state_weights],
         "input_weights": [float(v) for v in spec.input_weights],
         "terminal_weights": [float(v) for v in spec.terminal_weights]}
    for k in _SPEC_SCALARS:
        d[k] = float(getattr(spec, k))
    return d


def scenario_spec_from_json(j: dict) -> ScenarioSpec:
    """scenario_spec_from_json (serialization.hpp:156-197): starts from the
    ScenarioSpec defaults (scenarios.hpp:25-47: no vehicles) and takes every
    key present; vectors must have their full length (the reference's
    .at(i) throws std::out_of_range, here IndexError)."""
    spec = ScenarioSpec()
    kw = {}
    if "total_time" in j:
        kw["total_time"] = float(j["total_time"])
    if "shared_times" in j:
        kw["shared_times"] = tuple(float(t) for t in j["shared_times"])
    if "horizon" in j:
        kw["horizon"] = int(j["horizon"])
    if "ego_start" in j:
        e = j["ego_start"]
        kw["ego_start"] = (float(e[0]), float(e[1]), float(e[2]), float(e[3]))
    if "vehicles" in j:
        kw["vehicles"] = tuple(SurroundingVehicle((float(v["position"][0]), float(v["position"][1])),
                                                  float(v["heading"]), float(v["speed"]),
                                                  tuple(float(t) for t in v["target_speeds"]))
                               for v in j["vehicles"])
    for key in ("state_weights", "terminal_weights"):
        if key in j:
            w = j[key]
            kw[key] = (float(w[0]), float(w[1]), float(w[2]), float(w[3]))
    if "input_weights" in j:
        w = j["input_weights"]
        kw["input_weights"] = (float(w[0]), float(w[1]))
    for k in _SPEC_SCALARS:
        if k in j:
            kw[k] = float(j[k])
    return dataclasses.replace(spec, **kw)


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
           "report_to_json", "scenario_spec_to_json", "scenario_spec_from_json", "scenario_artifacts_to_json",
           "tree_branchings",
           "RECORD_KEYS", "TIME_KEYS"]
