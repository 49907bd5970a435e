"""bmpc_b200 — B200-native branch MPC (parallel tree iLQR + augmented Lagrangian).

Python mirror of the reference's solve-path interface
(/root/reference/proj/include/bmpc: build_tree tree.hpp:61, the scenario
builders scenarios.hpp:178-402, SolverOptions / solve solver.hpp:28-58,
595-780) over the C ABI in include/bmpc_b200.h. The compute runs in the
in-tree sm_100a library _lib/libbmpc_b200.so; there is no CPU fallback — if the
library is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BMPC_LIB") or os.path.join(_HERE, "_lib", "libbmpc_b200.so")  # BMPC_LIB: A/B builds

CONVERGED, MAX_ITERATIONS, ERROR = 0, 1, 2
STATUS_NAMES = {CONVERGED: "converged", MAX_ITERATIONS: "max-iter", ERROR: "error"}  # solver.hpp:538-545
MODEL_UNICYCLE, MODEL_AFFINE_QUADRATIC = 1, 2
SCENARIO_INTERSECTION, SCENARIO_LATENCY, SCENARIO_MULTISTAGE = 0, 1, 2


class BmpcError(RuntimeError):
    """A C-ABI call failed (carries the library's status code)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


# ----------------------------------------------------------------- C structs
class _Tree(C.Structure):
    _fields_ = [("node_count", C.c_int), ("horizon", C.c_int), ("last_branch_step", C.c_int),
                ("leaf_count", C.c_int), ("parent", C.POINTER(C.c_int)), ("time_step", C.POINTER(C.c_int)),
                ("weight", C.POINTER(C.c_double)), ("first_child", C.POINTER(C.c_int)),
                ("child_count", C.POINTER(C.c_int)), ("step_begin", C.POINTER(C.c_int)),
                ("leaves", C.POINTER(C.c_int))]


class _Model(C.Structure):
    _fields_ = [("kind", C.c_int), ("state_dim", C.c_int), ("input_dim", C.c_int),
                ("initial_state", C.c_void_p), ("dt", C.c_double), ("state_weights", C.c_double * 16),
                ("input_weights", C.c_double * 4), ("terminal_weights", C.c_double * 16),
                ("accel_limit", C.c_double), ("yaw_rate_limit", C.c_double), ("safety_radius", C.c_double),
                ("num_vehicles", C.c_int), ("reference", C.c_void_p), ("vehicle_position", C.c_void_p),
                ("lq_stage", C.c_void_p), ("lq_leaf", C.c_void_p)]


class _Vehicle(C.Structure):
    _fields_ = [("position", C.c_double * 2), ("heading", C.c_double), ("speed", C.c_double),
                ("n_targets", C.c_int), ("target_speeds", C.c_double * 8)]


class _SpecC(C.Structure):  # bmpc_scenario_spec
    _fields_ = [("total_time", C.c_double), ("n_shared", C.c_int), ("shared_times", C.c_double * 2),
                ("horizon", C.c_int), ("ego_start", C.c_double * 4), ("n_vehicles", C.c_int),
                ("vehicles", _Vehicle * 4), ("state_weights", C.c_double * 4), ("input_weights", C.c_double * 2),
                ("terminal_weights", C.c_double * 4)] + \
               [(n, C.c_double) for n in ("accel_limit", "yaw_rate_limit", "safety_radius", "prediction_tau",
                                          "reference_turn_rate", "backup_deceleration", "continue_deceleration")]


class _Scenario(C.Structure):
    _fields_ = [("family", C.c_int), ("horizon", C.c_int), ("total_time", C.c_double),
                ("shared_time", C.c_double * 2), ("v1", C.c_int), ("v2", C.c_int), ("n_branchings", C.c_int),
                ("branch_step", C.c_int * 8), ("branch_arity", C.c_int * 8), ("perturb", C.c_int),
                ("perturb_seed", C.c_ulonglong), ("spec", C.POINTER(_SpecC))]


class _ProblemData(C.Structure):
    _fields_ = [("tree", C.POINTER(_Tree)), ("model", _Model)]


_OPT_INT = ("max_inner_iterations", "max_outer_iterations", "alpha_levels")
_OPT_DBL = ("armijo_beta", "merit_gamma", "merit_mu0", "merit_mu_init", "defect_epsilon", "tol_defect",
            "tol_cost", "tol_feedforward", "tol_constraint", "penalty_init", "penalty_growth", "penalty_max",
            "reg_init", "reg_min", "reg_growth", "reg_decay", "reg_max")


class _Options(C.Structure):
    _fields_ = ([(n, C.c_int) for n in _OPT_INT] + [(n, C.c_double) for n in _OPT_DBL] +
                [("backward", C.c_int), ("forward", C.c_int), ("line_search", C.c_int)])


RECORD_FIELDS = ("outer", "accepted", "cost", "cost_al", "merit_before", "merit_after", "model_decrease",
                 "defect_l1", "violation", "alpha", "mu", "max_feedforward", "regularization")


class _Record(C.Structure):
    _fields_ = [("outer", C.c_int), ("accepted", C.c_int)] + [(n, C.c_double) for n in RECORD_FIELDS[2:]]


class _Report(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("status", "error_code", "error_node", "inner_iterations",
                                       "outer_iterations", "n_records")] + \
               [(n, C.c_double) for n in ("final_cost", "final_violation", "final_defect_l1")] + \
               [("times", C.c_double * 6)] + \
               [(n, C.c_double) for n in ("final_penalty", "final_mu", "final_reg")] + \
               [("message", C.c_char * 160), ("alpha_evals", C.c_double)]


_lib_handle = None


def lib():
    """The loaded sm_100a library (raises if it was not built)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (make -C paper_2506_13624_b200)")
        L = C.CDLL(LIB_PATH)
        L.bmpc_last_error.restype = C.c_char_p
        L.bmpc_version.restype = C.c_char_p
        L.bmpc_ctx_launch_count.restype = C.c_longlong
        _lib_handle = L
    return _lib_handle


def _check(rc: int):
    if rc != 0:
        raise BmpcError(rc, lib().bmpc_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- topology
class TreeTopology:
    """TreeTopology (tree.hpp:28-44) owned by the library; numpy copies of
    the index arrays are exposed with the reference's field names."""

    def __init__(self, handle: C.POINTER(_Tree), owner=None):
        self._h = handle
        self._owner = owner  # keeps a parent object (problem data) alive
        t = handle.contents
        n = t.node_count
        self.node_count = n
        self.horizon = t.horizon
        self.last_branch_step = t.last_branch_step
        self.parent = np.ctypeslib.as_array(t.parent, (n,)).copy()
        self.time_step = np.ctypeslib.as_array(t.time_step, (n,)).copy()
        self.weight = np.ctypeslib.as_array(t.weight, (n,)).copy()
        self.first_child = np.ctypeslib.as_array(t.first_child, (n,)).copy()
        self.child_count = np.ctypeslib.as_array(t.child_count, (n,)).copy()
        self.step_begin = np.ctypeslib.as_array(t.step_begin, (t.horizon + 2,)).copy()
        self.leaves = np.ctypeslib.as_array(t.leaves, (t.leaf_count,)).copy()
        self.branchings = None  # set by build_tree; scenario trees recover it (serialization.tree_branchings)

    @property
    def children(self):
        return [list(range(f, f + c)) if c else [] for f, c in zip(self.first_child, self.child_count)]

    def is_leaf(self, i: int) -> bool:
        return self.child_count[i] == 0

    def leaf_count(self) -> int:
        return len(self.leaves)

    def __del__(self):
        if self._owner is None and getattr(self, "_h", None) is not None and _lib_handle is not None:
            _lib_handle.bmpc_tree_free(self._h)
            self._h = None


def build_tree(horizon: int, branchings: Sequence[tuple] = ()) -> TreeTopology:
    """build_tree(horizon, branchings) (tree.hpp:61). Each branching is
    (step, arity, weights) or (step, arity) for uniform weights. Raises
    ValueError on invalid specs, as the reference throws invalid_argument."""
    nb = len(branchings)
    max_a = max([b[1] for b in branchings] + [1])
    steps = np.array([b[0] for b in branchings], np.int32)
    ar = np.array([b[1] for b in branchings], np.int32)
    w = np.zeros((max(nb, 1), max_a))
    for i, b in enumerate(branchings):
        ws = b[2] if len(b) > 2 else [1.0 / b[1]] * b[1]
        if len(ws) != b[1]:
            raise ValueError("build_tree: branching needs arity >= 2 and one weight per child")
        w[i, :b[1]] = ws
    out = C.POINTER(_Tree)()
    rc = lib().bmpc_tree_build(int(horizon), nb, _ptr(steps), _ptr(ar), _ptr(w), int(max_a), C.byref(out))
    if rc == -1:
        raise ValueError(lib().bmpc_last_error().decode())
    _check(rc)
    t = TreeTopology(out)
    t.branchings = [(int(b[0]), int(b[1]), [float(v) for v in (b[2] if len(b) > 2 else [1.0 / b[1]] * b[1])])
                    for b in branchings]  # construction spec (TreeTopology::branchings, tree.hpp:43)
    return t


# ----------------------------------------------------------------- problems
@dataclasses.dataclass
class SurroundingVehicle:
    """SurroundingVehicle (scenarios.hpp:15-22): constant heading, speed
    converging toward the per-scenario target."""
    position: tuple = (0.0, 0.0)
    heading: float = 0.0
    speed: float = 0.0
    target_speeds: tuple = ()


@dataclasses.dataclass
class ScenarioSpec:
    """ScenarioSpec (scenarios.hpp:25-47) with the reference's defaults, plus
    the multistage builder's branchings. `family` records which preset made
    the spec; the builder called decides the family."""
    family: int = SCENARIO_INTERSECTION
    horizon: int = 63
    total_time: float = 10.0
    shared_times: tuple = (0.1,)
    branchings: tuple = ()  # multistage: ((step, arity), ...)
    ego_start: tuple = (0.0, -20.0, math.pi / 2.0, 5.0)
    vehicles: tuple = ()
    state_weights: tuple = (1.0, 1.0, 0.1, 0.1)
    input_weights: tuple = (0.5, 0.5)
    terminal_weights: tuple = (1.0, 1.0, 0.1, 0.1)
    accel_limit: float = 3.0
    yaw_rate_limit: float = 0.5
    safety_radius: float = 3.0
    prediction_tau: float = 1.5
    reference_turn_rate: float = 0.4
    backup_deceleration: float = 3.0
    continue_deceleration: float = 2.5

    def dt(self) -> float:
        return self.total_time / self.horizon

    def _c(self) -> "_SpecC":
        c = _SpecC()
        c.total_time = float(self.total_time)
        if not 1 <= len(self.shared_times) <= 2:
            raise ValueError("ScenarioSpec: one or two shared times")
        c.n_shared = len(self.shared_times)
        for i, t in enumerate(self.shared_times):
            c.shared_times[i] = float(t)
        c.horizon = int(self.horizon)
        for i in range(4):
            c.ego_start[i] = float(self.ego_start[i])
        if len(self.vehicles) > 4:
            raise ValueError("ScenarioSpec: at most 4 surrounding vehicles")
        c.n_vehicles = len(self.vehicles)
        for k, v in enumerate(self.vehicles):
            cv = c.vehicles[k]
            cv.position[0], cv.position[1] = float(v.position[0]), float(v.position[1])
            cv.heading, cv.speed = float(v.heading), float(v.speed)
            if len(v.target_speeds) > 8:
                raise ValueError("ScenarioSpec: at most 8 target speeds per vehicle")
            cv.n_targets = len(v.target_speeds)
            for i, t in enumerate(v.target_speeds):
                cv.target_speeds[i] = float(t)
        for i in range(4):
            c.state_weights[i] = float(self.state_weights[i])
            c.terminal_weights[i] = float(self.terminal_weights[i])
        for i in range(2):
            c.input_weights[i] = float(self.input_weights[i])
        for k in ("accel_limit", "yaw_rate_limit", "safety_radius", "prediction_tau", "reference_turn_rate",
                  "backup_deceleration", "continue_deceleration"):
            setattr(c, k, float(getattr(self, k)))
        return c


def intersection_spec(horizon: int = 63, total_time: float = 10.0, shared_time: float = 0.1) -> ScenarioSpec:
    """intersection_spec (scenarios.hpp:178-197): the ego turns left across an
    oncoming vehicle while following a slower lead vehicle."""
    return ScenarioSpec(SCENARIO_INTERSECTION, horizon, total_time, (shared_time,),
                        ego_start=(0.0, -20.0, math.pi / 2.0, 5.0),
                        vehicles=(SurroundingVehicle((-3.5, 30.0), -math.pi / 2.0, 8.0, (8.0, 2.0, 5.0, 3.5)),
                                  SurroundingVehicle((0.0, -10.0), math.pi / 2.0, 5.0, (5.0, 1.0, 3.0, 2.0))))


def latency_spec(shared_time_1: float, horizon: int = 255, total_time: float = 5.0,
                 shared_time_0: float = 0.05) -> ScenarioSpec:
    """latency_spec (scenarios.hpp:300-317): cruising behind a lead vehicle."""
    return ScenarioSpec(SCENARIO_LATENCY, horizon, total_time, (shared_time_0, shared_time_1),
                        ego_start=(0.0, 0.0, 0.0, 10.0),
                        vehicles=(SurroundingVehicle((30.0, 0.0), 0.0, 8.0, (8.0, 0.0)),))


def multistage_spec(horizon: int, branchings: Sequence[tuple], total_time: float = 10.0,
                    base: Optional[ScenarioSpec] = None) -> ScenarioSpec:
    """cfg2/cfg3 trees: one uniform branching (step, arity) per stage; at stage
    j vehicle j mod 2 reveals its speed target. The scene
    is intersection_spec's unless `base` gives another one."""
    base = base or intersection_spec(horizon, total_time, 0.1)
    return dataclasses.replace(base, family=SCENARIO_MULTISTAGE, horizon=horizon, total_time=total_time,
                               branchings=tuple(tuple(b) for b in branchings))


class BmpcProblem:
    """BmpcProblem (problem.hpp:44-63) as a tree + device model descriptor."""

    def __init__(self, tree: TreeTopology, model: _Model, keep=(), data_handle=None):
        self.tree = tree
        self.model = model
        self._keep = keep
        self._data = data_handle
        self.state_dim = model.state_dim
        self.input_dim = model.input_dim

    @property
    def initial_state(self) -> np.ndarray:
        return np.ctypeslib.as_array(C.cast(self.model.initial_state, C.POINTER(C.c_double)),
                                     (self.state_dim,)).copy()

    def arrays(self) -> dict:
        """Per-node scenario data (reference / vehicle predictions)."""
        n = self.tree.node_count
        out = {"initial_state": self.initial_state}
        if self.model.kind == MODEL_UNICYCLE:
            out["reference"] = np.ctypeslib.as_array(C.cast(self.model.reference, C.POINTER(C.c_double)),
                                                     (n, 4)).copy()
            nv = self.model.num_vehicles
            if nv:
                out["vehicles"] = np.ctypeslib.as_array(
                    C.cast(self.model.vehicle_position, C.POINTER(C.c_double)), (n, nv, 2)).copy()
            out["dt"] = self.model.dt
        return out

    def __del__(self):
        if getattr(self, "_data", None) is not None and _lib_handle is not None:
            _lib_handle.bmpc_problem_data_free(self._data)
            self._data = None


def _build_scenario(spec: ScenarioSpec, family: int, v1=2, v2=2, perturb_seed=None) -> BmpcProblem:
    s = _Scenario()
    s.family = family
    spec_c = spec._c()
    s.spec = C.pointer(spec_c)
    s.horizon = spec.horizon
    s.total_time = spec.total_time
    st = list(spec.shared_times) + [0.0, 0.0]
    s.shared_time[0], s.shared_time[1] = st[0], st[1]
    s.v1, s.v2 = v1, v2
    s.n_branchings = len(spec.branchings)
    for i, b in enumerate(spec.branchings):
        s.branch_step[i], s.branch_arity[i] = b[0], b[1]
    s.perturb = 0 if perturb_seed is None else 1
    s.perturb_seed = 0 if perturb_seed is None else int(perturb_seed)
    out = C.POINTER(_ProblemData)()
    rc = lib().bmpc_scenario_build(C.byref(s), C.byref(out))
    if rc == -1:
        raise ValueError(lib().bmpc_last_error().decode())
    _check(rc)
    d = out.contents
    tree = TreeTopology(d.tree, owner=out)
    return BmpcProblem(tree, d.model, data_handle=out)


def build_intersection_case(spec: ScenarioSpec, v1_count: int, v2_count: int, perturb_seed=None) -> BmpcProblem:
    """build_intersection_case (scenarios.hpp:219-295) of any scene (two
    vehicles with enough target speeds)."""
    return _build_scenario(spec, SCENARIO_INTERSECTION, v1_count, v2_count, perturb_seed)


def build_latency_case(spec: ScenarioSpec, perturb_seed=None) -> BmpcProblem:
    """build_latency_case (scenarios.hpp:321-402) of any scene (one vehicle
    with two target speeds, two shared times)."""
    return _build_scenario(spec, SCENARIO_LATENCY, perturb_seed=perturb_seed)


def build_multistage_case(spec: ScenarioSpec, perturb_seed=None) -> BmpcProblem:
    return _build_scenario(spec, SCENARIO_MULTISTAGE, perturb_seed=perturb_seed)


def lq_problem(tree: TreeTopology, nx: int, nu: int, x0: np.ndarray, stage: np.ndarray,
               leaf: np.ndarray) -> BmpcProblem:
    """Affine-quadratic problem (the data random_lq_problem captures,
    oracles.hpp:316-365): stage [node][A B c Q R M q r], leaf [node][P p],
    all blocks column-major."""
    x0 = np.ascontiguousarray(x0, np.float64)
    stage = np.ascontiguousarray(stage, np.float64)
    leaf = np.ascontiguousarray(leaf, np.float64)
    m = _Model()
    m.kind = MODEL_AFFINE_QUADRATIC
    m.state_dim, m.input_dim = nx, nu
    m.initial_state = x0.ctypes.data
    m.lq_stage = stage.ctypes.data
    m.lq_leaf = leaf.ctypes.data
    return BmpcProblem(tree, m, keep=(x0, stage, leaf))


# ------------------------------------------------------------------ options
@dataclasses.dataclass
class SolverOptions:
    """SolverOptions (solver.hpp:28-58) — pmsilqr defaults."""
    max_inner_iterations: int = 100
    max_outer_iterations: int = 10
    alpha_levels: int = 11
    armijo_beta: float = 1e-4
    merit_gamma: float = 0.5
    merit_mu0: float = 1.0
    merit_mu_init: float = 1.0
    defect_epsilon: float = 1e-8
    tol_defect: float = 1e-8
    tol_cost: float = 1e-8
    tol_feedforward: float = 1e-6
    tol_constraint: float = 1e-4
    penalty_init: float = 10.0
    penalty_growth: float = 10.0
    penalty_max: float = 1e8
    reg_init: float = 0.0
    reg_min: float = 1e-6
    reg_growth: float = 10.0
    reg_decay: float = 10.0
    reg_max: float = 1e10
    # Strategy enums (solver.hpp:23-33, JSON spellings of serialization.hpp:40-61),
    # all on the GPU: "scan-tree-riccati" = tree-segmented scan / team sweep per
    # segment length, "sequential-riccati" = team Riccati sweep on every
    # segment, "scan-condensed" = the shared segment condensed into a dense QP
    # solved on the device (hypmsilqr, condensed.hpp / solver.hpp:297-307);
    # forward "nonlinear" = single-shooting trials (nonlinear rollout under the
    # feedback policies); line_search "sequential" = one step size per round.
    # scan_order / parallel only schedule the reference's CPU threads.
    backward: str = "scan-tree-riccati"
    forward: str = "linear"
    line_search: str = "parallel"
    scan_order: str = "tree"
    parallel: bool = True

    _ENUMS = {"backward": ("scan-tree-riccati", "scan-condensed", "sequential-riccati"),
              "forward": ("linear", "nonlinear"), "line_search": ("parallel", "sequential")}

    def _c(self) -> _Options:
        o = _Options()
        for name, _ in _Options._fields_:
            if name in self._ENUMS:
                v = getattr(self, name)
                if v not in self._ENUMS[name]:
                    raise ValueError("unknown %s strategy %r" % (name, v))
                setattr(o, name, self._ENUMS[name].index(v))
            else:
                setattr(o, name, getattr(self, name))
        return o


@dataclasses.dataclass
class SolveReport:
    """SolveReport (solver.hpp:572-582); `iterations` holds the per-iteration
    records as arrays keyed like IterationRecord."""
    status: int
    message: str
    inner_iterations: int
    outer_iterations: int
    final_cost: float
    final_violation: float
    final_defect_l1: float
    times: dict
    iterations: dict
    n_records: int
    alpha_evals: float = 0.0  # work counter: step sizes evaluated by the line search

    @property
    def status_name(self) -> str:
        return STATUS_NAMES[self.status]


@dataclasses.dataclass
class TrajectoryTree:
    state: np.ndarray  # [node][nx]
    input: np.ndarray  # [node][nu], leaf rows zero


@dataclasses.dataclass
class SolveResult:
    trajectory: TrajectoryTree
    report: SolveReport


def _report(r: _Report, recs=None, nrec=0) -> SolveReport:
    its = {}
    if recs is not None:
        k = min(nrec, len(recs))
        its = {f: np.array([getattr(recs[i], f) for i in range(k)]) for f in RECORD_FIELDS}
    names = ("setup_s", "backward_p1_s", "backward_p2_s", "forward_s", "line_search_s", "total_s")
    return SolveReport(r.status, r.message.decode(), r.inner_iterations, r.outer_iterations, r.final_cost,
                       r.final_violation, r.final_defect_l1, dict(zip(names, list(r.times))), its, r.n_records,
                       r.alpha_evals)


# ------------------------------------------------------------------ context
class Context:
    """One device + one CUDA stream (bmpc_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        _check(lib().bmpc_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device
        if stream is not None:
            _check(lib().bmpc_ctx_set_stream(self._h, C.c_void_p(stream)))

    @property
    def launches(self) -> int:
        return int(lib().bmpc_ctx_launch_count(self._h))

    def synchronize(self):
        _check(lib().bmpc_ctx_synchronize(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib_handle is not None:
            _lib_handle.bmpc_ctx_destroy(self._h)
            self._h = None


_default_ctx = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def solve(problem: BmpcProblem, options: Optional[SolverOptions] = None,
          initial_inputs: Optional[np.ndarray] = None, ctx: Optional[Context] = None,
          max_records: int = 1000) -> SolveResult:
    """solve(problem, opts, initial_inputs) (solver.hpp:595) on the GPU."""
    ctx = ctx or default_context()
    n, nx, nu = problem.tree.node_count, problem.state_dim, problem.input_dim
    x = np.zeros((n, nx))
    u = np.zeros((n, nu))
    rep = _Report()
    recs = (_Record * max(max_records, 1))()
    ii = None if initial_inputs is None else np.ascontiguousarray(initial_inputs, np.float64).reshape(n, nu)
    opts = (options or SolverOptions())._c()
    rc = lib().bmpc_solve(ctx._h, problem.tree._h, C.byref(problem.model), C.byref(opts), _ptr(ii), _ptr(x),
                          _ptr(u), C.byref(rep), recs, int(max_records))
    if rc == -4:
        raise RuntimeError(lib().bmpc_last_error().decode())
    _check(rc)
    return SolveResult(TrajectoryTree(x, u), _report(rep, recs, rep.n_records))


class Batch:
    """Device-resident batch of independent instances with one tree shape
    (bmpc_batch_*): one thread block per instance, one launch per solve."""

    def __init__(self, ctx: Context, problems: Sequence[BmpcProblem], max_records: int = 0):
        self.ctx = ctx
        self.count = len(problems)
        self.problems = list(problems)
        p0 = problems[0]
        self.n, self.nx, self.nu = p0.tree.node_count, p0.state_dim, p0.input_dim
        h = C.c_void_p()
        _check(lib().bmpc_batch_create(ctx._h, p0.tree._h, self.count, C.byref(p0.model), int(max_records),
                                       C.byref(h)))
        self._h = h
        self._models = (_Model * self.count)(*[p.model for p in problems])

    def set_launch(self, threads: int, min_blocks: int):
        """Per-instance thread-block shape (compiled variants only)."""
        _check(lib().bmpc_batch_set_launch(self._h, int(threads), int(min_blocks)))

    def set_models(self) -> int:
        b = C.c_size_t()
        _check(lib().bmpc_batch_set_models(self._h, self._models, C.byref(b)))
        return b.value

    def replicate(self):
        _check(lib().bmpc_batch_replicate(self._h))

    def solve(self, options: Optional[SolverOptions] = None):
        opts = (options or SolverOptions())._c()
        _check(lib().bmpc_batch_solve(self._h, C.byref(opts)))

    def results(self, x: Optional[np.ndarray] = None, u: Optional[np.ndarray] = None, want_reports=True,
                as_array=False):
        """Trajectories into x [count, n, nx] / u [count, n, nu] and the reports:
        SolveReport objects, or with as_array=True one zero-copy numpy structured
        array of the C bmpc_report records (fields status, inner_iterations, ...)."""
        # The C call memcpys count*n*nx / count*n*nu doubles into the raw
        # buffers: only exact float64, C-contiguous, writable arrays pass.
        for name, a, shape in (("x", x, (self.count, self.n, self.nx)), ("u", u, (self.count, self.n, self.nu))):
            if a is None:
                continue
            if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.shape != shape or \
                    not a.flags.c_contiguous or not a.flags.writeable:
                raise ValueError(f"{name} must be a writable C-contiguous float64 array of shape {shape}, got "
                                 f"{getattr(a, 'dtype', type(a))} {getattr(a, 'shape', '')}")
        reps = (_Report * self.count)() if want_reports else None
        b = C.c_size_t()
        _check(lib().bmpc_batch_results(self._h, _ptr(x), _ptr(u), reps, C.byref(b)))
        if not want_reports:
            return None, b.value
        if as_array:
            return np.ctypeslib.as_array(reps), b.value
        return [_report(r) for r in reps], b.value

    def set_scenes(self, specs, family: int = SCENARIO_INTERSECTION, v1: int = 2, v2: int = 2) -> int:
        """Device-side scene generation (bmpc_batch_set_scenes): every node's
        tracking reference and vehicle predictions, the model scalars and
        x0 = ego_start computed on the GPU from one ScenarioSpec per instance
        (or a single shared one); returns the H2D bytes (the specs only)."""
        specs = [specs] if isinstance(specs, ScenarioSpec) else list(specs)
        arr = (_SpecC * len(specs))(*[s._c() for s in specs])
        b = C.c_size_t()
        _check(lib().bmpc_batch_set_scenes(self._h, int(family), arr, len(specs), int(v1), int(v2), C.byref(b)))
        return b.value

    def scene(self, instance: int) -> dict:
        """The per-node scene data of one instance (reference, vehicles, x0)."""
        nv = self.problems[0].model.num_vehicles
        ref = np.zeros((self.n, 4))
        veh = np.zeros((self.n, nv, 2))
        x0 = np.zeros(self.nx)
        _check(lib().bmpc_batch_scene(self._h, int(instance), _ptr(ref), _ptr(veh) if nv else None, _ptr(x0)))
        return {"reference": ref, "vehicles": veh, "initial_state": x0}

    def set_initial_states(self, x0: np.ndarray) -> int:
        """Upload new initial states [count, nx] over the resident scenario data
        (bmpc_batch_set_initial_states); returns H2D bytes."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(self.count, self.nx)
        b = C.c_size_t()
        _check(lib().bmpc_batch_set_initial_states(self._h, _ptr(x0), C.byref(b)))
        return b.value

    def pack_results(self, d_dst_ptr: int) -> int:
        """Pack [x | u] of every instance into a device buffer (e.g. a torch
        tensor's data_ptr()) for the NVLink gather; returns bytes."""
        b = C.c_size_t()
        _check(lib().bmpc_batch_pack_results(self._h, C.c_void_p(d_dst_ptr), C.byref(b)))
        return b.value

    def records(self, instance: int, max_records: int = 1000) -> dict:
        recs = (_Record * max_records)()
        n = C.c_int()
        _check(lib().bmpc_batch_records(self._h, int(instance), recs, int(max_records), C.byref(n)))
        return {f: np.array([getattr(recs[i], f) for i in range(min(n.value, max_records))]) for f in RECORD_FIELDS}

    def info(self) -> dict:
        t, b, r = C.c_int(), C.c_int(), C.c_int()
        _check(lib().bmpc_batch_info(self._h, C.byref(t), C.byref(b), C.byref(r)))
        return {"threads_per_block": t.value, "blocks": b.value, "regs_per_thread": r.value}

    def __del__(self):
        if getattr(self, "_h", None) and _lib_handle is not None:
            _lib_handle.bmpc_batch_destroy(self._h)
            self._h = None


def set_lqr_strategy(ctx: Context, backward: str):
    """Backward strategy of subsequent lqr_tree calls on ctx:
    "scan-tree-riccati" (default) or "scan-condensed" (bmpc_ctx_set_lqr_strategy)."""
    code = {"scan-tree-riccati": 0, "scan-condensed": 1}[backward]
    _check(lib().bmpc_ctx_set_lqr_strategy(ctx._h, code))


def lqr_elements(op: str, nx: int, nu: int, a: np.ndarray, b: Optional[np.ndarray] = None, reg: float = 0.0,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """Batched scan-element primitives on the GPU (bmpc_lqr_elements):
    "init_bwd" of packed [A B c Q R M q r] records (rows of a), "combine_bwd"
    / "combine_fwd" of element rows a (+) b (lqr_scan.hpp:28-111, 171-173)."""
    ctx = ctx or default_context()
    code = {"init_bwd": 0, "combine_bwd": 1, "combine_fwd": 2}[op]
    a = np.ascontiguousarray(a, np.float64)
    count = a.shape[0]
    width = nx * nx + nx if code == 2 else 3 * nx * nx + 2 * nx
    bb = None if b is None else np.ascontiguousarray(b, np.float64)
    out = np.zeros((count, width))
    _check(lib().bmpc_lqr_elements(ctx._h, code, int(nx), int(nu), int(count), _ptr(a), _ptr(bb), C.c_double(reg),
                                   _ptr(out)))
    return out


def shard_range(count: int, n_shards: int, g: int) -> tuple:
    """Contiguous shard g of `count` instances over n_shards devices / ranks:
    [g*count/n, (g+1)*count/n) (bmpc_shard_range; host-only, no GPU needed)."""
    b, n = C.c_int(), C.c_int()
    _check(lib().bmpc_shard_range(int(count), int(n_shards), int(g), C.byref(b), C.byref(n)))
    return b.value, n.value


class MultiBatch:
    """Independent instances sharded contiguously over several contexts
    (devices) of ONE process (bmpc_multi_*): each device solves its shard with
    its own launches, concurrently; the final gather packs every shard's
    trajectories straight into one buffer on the first context's device over
    peer-to-peer (NVLink). The reference's analogue is the thread pool of
    independent solve() calls, parallel_sweep (tools/bench.cpp:259-269)."""

    def __init__(self, ctxs: Sequence[Context], problems: Sequence[BmpcProblem], max_records: int = 0):
        self.ctxs = list(ctxs)
        self.count = len(problems)
        self.problems = list(problems)
        p0 = problems[0]
        self.n, self.nx, self.nu = p0.tree.node_count, p0.state_dim, p0.input_dim
        arr = (C.c_void_p * len(self.ctxs))(*[c._h.value for c in self.ctxs])
        h = C.c_void_p()
        _check(lib().bmpc_multi_create(arr, len(self.ctxs), p0.tree._h, self.count, C.byref(p0.model),
                                       int(max_records), C.byref(h)))
        self._h = h
        self._models = (_Model * self.count)(*[p.model for p in problems])

    def set_models(self) -> int:
        b = C.c_size_t()
        _check(lib().bmpc_multi_set_models(self._h, self._models, C.byref(b)))
        return b.value

    def set_initial_states(self, x0: np.ndarray) -> int:
        x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(self.count, self.nx)
        b = C.c_size_t()
        _check(lib().bmpc_multi_set_initial_states(self._h, _ptr(x0), C.byref(b)))
        return b.value

    def solve(self, options: Optional[SolverOptions] = None):
        opts = (options or SolverOptions())._c()
        _check(lib().bmpc_multi_solve(self._h, C.byref(opts)))

    def gather(self, d_dst_ptr: int) -> int:
        """Pack every shard's [x | u] into the device buffer d_dst_ptr on the
        first context's device (count * n * (nx + nu) doubles); returns bytes."""
        b = C.c_size_t()
        _check(lib().bmpc_multi_gather(self._h, C.c_void_p(d_dst_ptr), C.byref(b)))
        return b.value

    def results(self, x: Optional[np.ndarray] = None, u: Optional[np.ndarray] = None):
        for name, a, shape in (("x", x, (self.count, self.n, self.nx)), ("u", u, (self.count, self.n, self.nu))):
            if a is not None and (a.dtype != np.float64 or a.shape != shape or not a.flags.c_contiguous):
                raise ValueError(f"{name} must be a C-contiguous float64 array of shape {shape}")
        reps = (_Report * self.count)()
        b = C.c_size_t()
        _check(lib().bmpc_multi_results(self._h, _ptr(x), _ptr(u), reps, C.byref(b)))
        return [_report(r) for r in reps], b.value

    def shard(self, g: int) -> tuple:
        begin, n = C.c_int(), C.c_int()
        _check(lib().bmpc_multi_shard(self._h, int(g), None, C.byref(begin), C.byref(n)))
        return begin.value, n.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib_handle is not None:
            _lib_handle.bmpc_multi_destroy(self._h)
            self._h = None


def lqr_tree(tree: TreeTopology, nx: int, nu: int, stage: np.ndarray, defect: np.ndarray, leaf: np.ndarray,
             reg: float = 0.0, dx0: Optional[np.ndarray] = None, grid: bool = False,
             ctx: Optional[Context] = None) -> dict:
    """Kernel-level backward_pass + linear_rollout + EC on TreeStageModels
    (solver.hpp:203-430), the tree-segmented scan on the GPU."""
    ctx = ctx or default_context()
    n = tree.node_count
    stage = np.ascontiguousarray(stage, np.float64)
    defect = np.ascontiguousarray(defect, np.float64)
    leaf = np.ascontiguousarray(leaf, np.float64)
    dx0 = np.zeros(nx) if dx0 is None else np.ascontiguousarray(dx0, np.float64)
    K = np.zeros((n, nu * nx))
    k = np.zeros((n, nu))
    P = np.zeros((n, nx * nx))
    p = np.zeros((n, nx))
    dx = np.zeros((n, nx))
    du = np.zeros((n, nu))
    sc = np.zeros(4)
    _check(lib().bmpc_lqr_tree(ctx._h, tree._h, nx, nu, _ptr(stage), _ptr(defect), _ptr(leaf), C.c_double(reg),
                               _ptr(dx0), int(grid), _ptr(K), _ptr(k), _ptr(P), _ptr(p), _ptr(dx), _ptr(du),
                               _ptr(sc)))
    return dict(K=K, k=k, P=P, p=p, dx=dx, du=du, max_feedforward=sc[0], a1=sc[1], a2=sc[2], error=int(sc[3]))


def fp64_peak_tflops(ctx: Optional[Context] = None) -> float:
    """Measured FP64 FMA peak of the device (DFMA microbenchmark)."""
    ctx = ctx or default_context()
    v = C.c_double()
    _check(lib().bmpc_fp64_peak_tflops(ctx._h, C.byref(v)))
    return v.value


def version() -> str:
    return lib().bmpc_version().decode()


def debug_grid_sync_us(blocks: int, threads: int, iters: int = 2000, ctx: Optional[Context] = None) -> float:
    """Microseconds per cooperative grid barrier at this launch shape."""
    ctx = ctx or default_context()
    v = C.c_double()
    _check(lib().bmpc_debug_grid_sync_us(ctx._h, int(blocks), int(threads), int(iters), C.byref(v)))
    return v.value


PHASES = ("linearize", "bwd_terminal_elements", "bwd_scan", "feedback", "fwd_elements", "fwd_scan", "fwd_sweep",
          "line_search", "merit", "step_al", "ec_du")


def batch_phase_profile(batch: "Batch", instance: int = 0) -> dict:
    """Per-phase device time (ms) of one instance after a profiled solve."""
    out = np.zeros(24)
    _check(lib().bmpc_batch_phase_profile(batch._h, int(instance), _ptr(out), 24))
    res = {name: out[i] * 1e-6 for i, name in enumerate(PHASES)}
    if out[13] > 0:  # diagnostic counters, not times
        res["sweep_cycles_per_step"] = out[12] / out[13]
    res["walk_cycles"] = (out[14], out[15], out[11], out[18], out[19], out[20])  # head_dx, chunks, depths, ns, elements, chain
    res["sm_mhz"] = 1e3 * out[16] / out[17] if out[17] > 0 else 0.0  # effective SM clock of the solve
    res["fwd_scan_cycles"] = (out[21], out[22], out[23])  # elements + barrier, run maps, scan + re-walk
    return res


def batch_set_profiling(batch: "Batch", on: bool = True):
    _check(lib().bmpc_batch_set_profiling(batch._h, int(on)))


def set_seq_max_len(ctx: Context, length: int):
    """Segments of <= length nodes use the team Riccati sweep, longer ones the
    associative scan (0 = scan everywhere)."""
    _check(lib().bmpc_ctx_set_seq_max_len(ctx._h, int(length)))


def set_line_search_block(ctx: Context, alphas: int):
    """Step sizes per line-search round (0 = all levels at once, the reference's
    parallel search); the accepted alpha and all reported values are the same."""
    _check(lib().bmpc_ctx_set_line_search_block(ctx._h, int(alphas)))


def set_schedule(ctx: Context, probe_passes: int):
    """Batch schedule: probe passes before ordering instances by their last
    constraint violation (0 = one FIFO launch). Results are identical."""
    _check(lib().bmpc_ctx_set_schedule(ctx._h, int(probe_passes)))


def debug_ric_step_cycles(steps: int = 512, prefetch: int = 1, ctx: Optional[Context] = None):
    """Cycles per isolated team Riccati step; prefetch=2 returns (total, [5 stage cycles])."""
    ctx = ctx or default_context()
    v = (C.c_double * 6)()
    _check(lib().bmpc_debug_ric_step_cycles(ctx._h, int(steps), int(prefetch), v))
    return (v[0], list(v[1:])) if prefetch >= 2 else v[0]
