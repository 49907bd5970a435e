"""ctypes binding to the plain-C oracle (oracle/_build/libbmpc_oracle.so).

TEST INFRASTRUCTURE ONLY: the checker for tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg. It restates the reference algorithm
(oracle/bmpc_oracle.c, pinned against oracle/_ref and tests/golden/).
"""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "oracle", "_build", "libbmpc_oracle.so")


class BoProblem(C.Structure):
    _fields_ = [("n", C.c_int), ("horizon", C.c_int), ("last_branch_step", C.c_int),
                ("parent", C.c_void_p), ("first_child", C.c_void_p), ("nchild", C.c_void_p),
                ("weight", C.c_void_p), ("step_begin", C.c_void_p),
                ("kind", C.c_int), ("nx", C.c_int), ("nu", C.c_int), ("x0", C.c_void_p), ("dt", C.c_double),
                ("Wx", C.c_void_p), ("Wu", C.c_void_p), ("Wf", C.c_void_p),
                ("a_max", C.c_double), ("w_max", C.c_double), ("radius", C.c_double), ("nv", C.c_int),
                ("reference", C.c_void_p), ("vehicles", C.c_void_p), ("lq_stage", C.c_void_p),
                ("lq_leaf", C.c_void_p)]


class BoOptions(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("max_inner_iterations", "max_outer_iterations", "alpha_levels")] + \
               [(n, C.c_double) for n in ("armijo_beta", "merit_gamma", "merit_mu0", "merit_mu_init",
                                          "defect_epsilon", "tol_defect", "tol_cost", "tol_feedforward",
                                          "tol_constraint", "penalty_init", "penalty_growth", "penalty_max",
                                          "reg_init", "reg_min", "reg_growth", "reg_decay", "reg_max")]


REC_FIELDS = ("outer", "accepted", "cost", "cost_al", "merit_before", "merit_after", "model_decrease", "defect_l1",
              "violation", "alpha", "mu", "max_feedforward", "regularization")


class BoRecord(C.Structure):
    _fields_ = [("outer", C.c_int), ("accepted", C.c_int)] + [(n, C.c_double) for n in REC_FIELDS[2:]]


class BoReport(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("status", "error_code", "inner_iterations", "outer_iterations",
                                       "n_records")] + \
               [(n, C.c_double) for n in ("final_cost", "final_violation", "final_defect_l1")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        so = SO
        if os.environ.get("BMPC_ORACLE_VARIANT") == "fma":  # rounding-sensitivity twin (oracle/Makefile)
            so = SO.replace("libbmpc_oracle.so", "libbmpc_oracle_fma.so")
        if not os.path.exists(so):
            raise FileNotFoundError(f"{so} missing: run `make -C oracle`")
        _lib = C.CDLL(so)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_tree(horizon, branchings):
    """bo_build_tree: returns dict of tree arrays (parent, time_step, weight,
    first_child, nchild, step_begin) or raises ValueError."""
    nb = len(branchings)
    steps = np.array([b[0] for b in branchings] + [0], np.int32)
    ar = np.array([b[1] for b in branchings] + [0], np.int32)
    ma = max([b[1] for b in branchings] + [1])
    w = np.zeros((max(nb, 1), ma))
    for i, b in enumerate(branchings):
        w[i, :b[1]] = b[2] if len(b) > 2 else [1.0 / b[1]] * b[1]
    n = lib().bo_tree_size(horizon, nb, _p(steps), _p(ar))
    out = dict(parent=np.zeros(n, np.int32), time_step=np.zeros(n, np.int32), weight=np.zeros(n),
               first_child=np.zeros(n, np.int32), nchild=np.zeros(n, np.int32),
               step_begin=np.zeros(horizon + 2, np.int32))
    rc = lib().bo_build_tree(horizon, nb, _p(steps), _p(ar), _p(w), ma, *[_p(out[k]) for k in
                             ("parent", "time_step", "weight", "first_child", "nchild", "step_begin")])
    if rc < 0:
        raise ValueError("invalid tree spec")
    out["horizon"] = horizon
    out["last_branch_step"] = branchings[-1][0] if nb else -1
    return out


class Problem:
    """Holds numpy arrays alive and the BoProblem struct."""

    def __init__(self, tree: dict, kind: int, nx: int, nu: int, x0, **model):
        self.keep = {}
        s = BoProblem()
        s.n = len(tree["parent"])
        s.horizon = tree["horizon"]
        s.last_branch_step = tree["last_branch_step"]
        for k in ("parent", "first_child", "nchild", "step_begin"):
            self.keep[k] = np.ascontiguousarray(tree[k], np.int32)
            setattr(s, k, self.keep[k].ctypes.data)
        self.keep["weight"] = np.ascontiguousarray(tree["weight"], np.float64)
        s.weight = self.keep["weight"].ctypes.data
        s.kind, s.nx, s.nu = kind, nx, nu
        self.keep["x0"] = np.ascontiguousarray(x0, np.float64)
        s.x0 = self.keep["x0"].ctypes.data
        for k in ("Wx", "Wu", "Wf", "reference", "vehicles", "lq_stage", "lq_leaf"):
            if model.get(k) is not None:
                self.keep[k] = np.ascontiguousarray(model[k], np.float64)
                setattr(s, k, self.keep[k].ctypes.data)
        for k in ("dt", "a_max", "w_max", "radius"):
            if k in model:
                setattr(s, k, float(model[k]))
        s.nv = int(model.get("nv", 0))
        self.s = s
        self.n, self.nx, self.nu = s.n, nx, nu


def from_bmpc(problem) -> Problem:
    """Oracle problem from a paper_2506_13624_b200.BmpcProblem (same data)."""
    t = problem.tree
    tree = dict(parent=t.parent, first_child=t.first_child, nchild=t.child_count, weight=t.weight,
                step_begin=t.step_begin, horizon=t.horizon, last_branch_step=t.last_branch_step)
    m = problem.model
    nx, nu = problem.state_dim, problem.input_dim
    if m.kind == 1:
        a = problem.arrays()
        return Problem(tree, 1, nx, nu, a["initial_state"], dt=m.dt, Wx=np.array(m.state_weights[:]),
                       Wu=np.array(m.input_weights[:]), Wf=np.array(m.terminal_weights[:]), a_max=m.accel_limit,
                       w_max=m.yaw_rate_limit, radius=m.safety_radius, nv=m.num_vehicles,
                       reference=a["reference"], vehicles=a.get("vehicles", np.zeros((t.node_count, 0, 2))))
    stage, leaf = problem._keep[1], problem._keep[2]
    return Problem(tree, 2, nx, nu, problem.initial_state, lq_stage=stage, lq_leaf=leaf)


def default_options(**over):
    o = BoOptions()
    lib().bo_default_options(C.byref(o))
    for k, v in over.items():
        setattr(o, k, v)
    return o


def solve(prob: Problem, opts=None, u_init=None, max_recs=2000):
    x = np.zeros((prob.n, prob.nx))
    u = np.zeros((prob.n, prob.nu))
    rep = BoReport()
    recs = (BoRecord * max_recs)()
    ui = None if u_init is None else np.ascontiguousarray(u_init, np.float64)
    rc = lib().bo_solve(C.byref(prob.s), C.byref(opts or default_options()), _p(ui), _p(x), _p(u), C.byref(rep),
                        recs, max_recs)
    if rc != 0:
        raise RuntimeError("nonlinear_rollout: non-finite state")
    k = min(rep.n_records, max_recs)
    records = {f: np.array([getattr(recs[i], f) for i in range(k)]) for f in REC_FIELDS}
    return dict(x=x, u=u, status=rep.status, error_code=rep.error_code, inner_iterations=rep.inner_iterations,
                outer_iterations=rep.outer_iterations, final_cost=rep.final_cost,
                final_violation=rep.final_violation, final_defect_l1=rep.final_defect_l1, records=records,
                n_records=rep.n_records)


def solve_problem(problem, opts=None):
    """Oracle solve of a paper_2506_13624_b200.BmpcProblem."""
    return solve(from_bmpc(problem), opts)


def lqr_tree(tree: dict, nx, nu, stage, defect, leaf, reg=0.0, strategy=0, dx0=None):
    prob = Problem(tree, 2, nx, nu, np.zeros(nx))
    n = prob.n
    K = np.zeros((n, nu * nx)); k = np.zeros((n, nu)); P = np.zeros((n, nx * nx)); p = np.zeros((n, nx))
    dx = np.zeros((n, nx)); du = np.zeros((n, nu)); sc = np.zeros(4)
    dx0 = np.zeros(nx) if dx0 is None else np.ascontiguousarray(dx0, np.float64)
    args = [np.ascontiguousarray(a, np.float64) for a in (stage, defect, leaf)]
    lib().bo_lqr_tree(C.byref(prob.s), nx, nu, *[_p(a) for a in args], C.c_double(reg), strategy, _p(dx0), _p(K),
                      _p(k), _p(P), _p(p), _p(dx), _p(du), _p(sc))
    return dict(K=K, k=k, P=P, p=p, dx=dx, du=du, max_feedforward=sc[0], a1=sc[1], a2=sc[2], error=int(sc[3]))


def random_lq(seed, tree: dict, nx, nu):
    n = len(tree["parent"])
    ss = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu
    x0 = np.zeros(nx); stage = np.zeros((n, ss)); leaf = np.zeros((n, nx * nx + nx))
    nch = np.ascontiguousarray(tree["nchild"], np.int32)
    lib().bo_random_lq(C.c_ulonglong(seed), n, _p(nch), nx, nu, _p(x0), _p(stage), _p(leaf))
    return x0, stage, leaf


def mt_uniform(seed, count):
    out = np.zeros(count)
    lib().bo_mt_uniform(C.c_ulonglong(seed), count, _p(out))
    return out


def rollout(prob: Problem, u):
    x = np.zeros((prob.n, prob.nx))
    uu = np.ascontiguousarray(u, np.float64)
    if lib().bo_rollout(C.byref(prob.s), _p(uu), _p(x)) != 0:
        raise RuntimeError("nonlinear_rollout: non-finite state")
    return x


def evaluate(prob: Problem, x, u, rho=10.0):
    out = np.zeros(5)
    xx = np.ascontiguousarray(x, np.float64)
    uu = np.ascontiguousarray(u, np.float64)
    lib().bo_evaluate(C.byref(prob.s), _p(xx), _p(uu), C.c_double(rho), _p(out))
    return dict(cost=out[0], cost_al=out[1], defect_l1=out[2], max_violation=out[3], finite=bool(out[4]))
