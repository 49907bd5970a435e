"""ctypes binding to oracle/_ref/libbmpc_ref.so (the UNMODIFIED reference
solver compiled against the Eigen shim). Test infrastructure only: used as the
checker in tests/ and as bench.py's reference arm."""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libbmpc_ref.so")


class RefScenario(C.Structure):
    _fields_ = [("family", C.c_int), ("horizon", C.c_int), ("total_time", C.c_double),
                ("shared_time", C.c_double * 2), ("v1", C.c_int), ("v2", C.c_int),
                ("n_branchings", C.c_int), ("branch_step", C.c_int * 8), ("branch_arity", C.c_int * 8),
                ("branch_weight", (C.c_double * 16) * 8), ("perturb", C.c_int),
                ("perturb_seed", C.c_ulonglong), ("lq_nx", C.c_int), ("lq_nu", C.c_int),
                ("lq_seed", C.c_ulonglong)]


class RefOptions(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("backward", "forward", "line_search", "scan_order", "parallel",
                                       "max_inner_iterations", "max_outer_iterations", "alpha_levels")] + \
               [(n, C.c_double) for n in ("armijo_beta", "merit_gamma", "merit_mu0", "merit_mu_init",
                                          "defect_epsilon", "tol_defect", "tol_cost", "tol_feedforward",
                                          "tol_constraint", "penalty_init", "penalty_growth", "penalty_max",
                                          "reg_init", "reg_min", "reg_growth", "reg_decay", "reg_max")]


class RefReport(C.Structure):
    _fields_ = [("status", C.c_int), ("inner_iterations", C.c_int), ("outer_iterations", C.c_int),
                ("n_records", C.c_int), ("final_cost", C.c_double), ("final_violation", C.c_double),
                ("final_defect_l1", C.c_double), ("times", C.c_double * 6), ("message", C.c_char * 256)]


class RefRecord(C.Structure):
    _fields_ = [("outer", C.c_int), ("accepted", C.c_int)] + \
               [(n, C.c_double) for n in ("cost", "cost_al", "merit_before", "merit_after", "model_decrease",
                                          "defect_l1", "violation", "alpha", "mu", "max_feedforward",
                                          "regularization")]


RECORD_FIELDS = [f for f, _ in RefRecord._fields_]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def scenario(family, horizon, total_time=10.0, shared=(0.1, 0.0), v=(2, 2), branchings=(), perturb_seed=None,
             lq=(0, 0, 0)):
    s = RefScenario()
    s.family = family
    s.horizon = horizon
    s.total_time = total_time
    s.shared_time[0], s.shared_time[1] = shared
    s.v1, s.v2 = v
    s.n_branchings = len(branchings)
    for i, b in enumerate(branchings):
        step, arity = b[0], b[1]
        s.branch_step[i] = step
        s.branch_arity[i] = arity
        w = b[2] if len(b) > 2 else [1.0 / arity] * arity
        for a in range(arity):
            s.branch_weight[i][a] = w[a]
    s.perturb = 0 if perturb_seed is None else 1
    s.perturb_seed = 0 if perturb_seed is None else perturb_seed
    s.lq_nx, s.lq_nu, s.lq_seed = lq
    return s


def default_options():
    o = RefOptions()
    lib().ref_default_options(C.byref(o))
    return o


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def size(sc):
    n, nx, nu, nv = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    if lib().ref_scenario_size(C.byref(sc), C.byref(n), C.byref(nx), C.byref(nu), C.byref(nv)) != 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return n.value, nx.value, nu.value, nv.value


def dump(sc):
    n, nx, nu, nv = size(sc)
    parent = np.zeros(n, np.int32)
    ts = np.zeros(n, np.int32)
    w = np.zeros(n)
    lbs = C.c_int()
    x0 = np.zeros(nx)
    ref = np.zeros((n, 4))
    veh = np.zeros((n, max(nv, 1), 2))
    dt = C.c_double()
    if lib().ref_scenario_dump(C.byref(sc), _p(parent), _p(ts), _p(w), C.byref(lbs), _p(x0), _p(ref), _p(veh),
                               C.byref(dt)) != 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return dict(parent=parent, time_step=ts, weight=w, last_branch_step=lbs.value, initial_state=x0,
                reference=ref, vehicles=veh[:, :nv], dt=dt.value, nx=nx, nu=nu)


def solve(sc, opts=None, initial_inputs=None, max_records=2000):
    n, nx, nu, _ = size(sc)
    x = np.zeros((n, nx))
    u = np.zeros((n, nu))
    rep = RefReport()
    recs = (RefRecord * max_records)()
    ii = None if initial_inputs is None else np.ascontiguousarray(initial_inputs, np.float64)
    rc = lib().ref_scenario_solve(C.byref(sc), C.byref(opts or default_options()),
                                  None if ii is None else _p(ii), _p(x), _p(u), C.byref(rep), recs,
                                  max_records)
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())
    records = {f: np.array([getattr(recs[i], f) for i in range(min(rep.n_records, max_records))])
               for f in RECORD_FIELDS}
    report = dict(status=rep.status, inner_iterations=rep.inner_iterations,
                  outer_iterations=rep.outer_iterations, final_cost=rep.final_cost,
                  final_violation=rep.final_violation, final_defect_l1=rep.final_defect_l1,
                  times=list(rep.times), message=rep.message.decode(), n_records=rep.n_records)
    return x, u, report, records


def lqr_tree(branch_spec, horizon, nx, nu, stage, defect, leaf, reg=0.0, strategy=0, dx0=None):
    """Reference backward_pass + linear_rollout + EC on explicit
    TreeStageModels (solver.hpp:203-430). branch_spec: [(step, arity, weights)]."""
    nb = len(branch_spec)
    bs = np.array([b[0] for b in branch_spec] + [0], np.int32)
    ba = np.array([b[1] for b in branch_spec] + [0], np.int32)
    bw = np.zeros((max(nb, 1), 16))
    for i, b in enumerate(branch_spec):
        w = b[2] if len(b) > 2 else [1.0 / b[1]] * b[1]
        bw[i, :b[1]] = w
    n = stage.shape[0]
    K = np.zeros((n, nu * nx)); k = np.zeros((n, nu)); P = np.zeros((n, nx * nx)); p = np.zeros((n, nx))
    dx = np.zeros((n, nx)); du = np.zeros((n, nu)); sc = np.zeros(4)
    dx0 = np.zeros(nx) if dx0 is None else np.ascontiguousarray(dx0, np.float64)
    stage = np.ascontiguousarray(stage, np.float64); defect = np.ascontiguousarray(defect, np.float64)
    leaf = np.ascontiguousarray(leaf, np.float64)
    L = lib()
    L.ref_lqr_tree.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int] + \
        [C.c_void_p] * 3 + [C.c_double, C.c_int] + [C.c_void_p] * 8
    rc = L.ref_lqr_tree(horizon, nb, _p(bs), _p(ba), _p(bw), nx, nu, _p(stage), _p(defect), _p(leaf), reg,
                        strategy, _p(dx0), _p(K), _p(k), _p(P), _p(p), _p(dx), _p(du), _p(sc))
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return dict(K=K, k=k, P=P, p=p, dx=dx, du=du, max_feedforward=sc[0], a1=sc[1], a2=sc[2], error=int(sc[3]))


def lq_dump(sc):
    """random_lq_problem data for scenario family 3 (x0, stage, leaf)."""
    n, nx, nu, _ = size(sc)
    ss = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu
    x0 = np.zeros(nx); st = np.zeros((n, ss)); lf = np.zeros((n, nx * nx + nx))
    if lib().ref_lq_dump(C.byref(sc), _p(x0), _p(st), _p(lf)) != 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return x0, st, lf
