"""Oracle-equivalence suites of the reference (testing/verification.hpp,
`bench verify`) pointed at the GPU back end. Each check runs the sm_100a
kernel-level LQR path (bmpc_lqr_tree: backward pass + linear rollout on a
tree) and compares it with an independent host-side computation written here
in numpy — a sequential Riccati recursion, a sequential closed-loop rollout,
a brute-force KKT solve of the tree QP — or with the other GPU strategy:

    scan-riccati    GPU associative scan (segments scanned) vs sequential Riccati   1e-8  (verification.hpp:42-74)
    forward         GPU forward scan vs sequential rollout of the same policies     1e-10 (:76-107)
    tree-qp         GPU tree solve vs dense KKT solve of the tree QP                 1e-7  (:225-261)
    cross-strategy  GPU scan vs GPU team sweep vs host Riccati (dx, du)              1e-6  (:263-300)

    associativity   GPU combine_bwd / combine_fwd, (a+b)+c vs a+(b+c)             1e-9  (:110-137)
    condensing      GPU condensed shared segment vs GPU tree scan vs host Riccati 1e-7  (:141-223)

`mutate="scan-sign"` flips the sign of the dynamics offsets fed to the GPU
scan only (verification.hpp:31-36); scan-riccati must then fail (harness
sanity). Random data: numpy default_rng(seed) with the reference's
distributions (oracles.hpp:39-83).
"""
import dataclasses
from typing import List, Optional, Sequence

import numpy as np

from . import Context, build_tree, default_context, lqr_elements, lqr_tree, set_lqr_strategy, set_seq_max_len

SUITES = ("scan-riccati", "forward", "associativity", "condensing", "tree-qp", "cross-strategy")
_SWEEP_ALL = 1 << 30  # seq_max_len: every segment takes the team Riccati sweep


@dataclasses.dataclass
class CheckResult:
    name: str
    passed: bool
    max_error: float
    tolerance: float
    detail: str = ""

    def line(self) -> str:
        """bench.cpp:317-320."""
        return "[%s] %s: max error %.3e (tolerance %.1e)%s%s" % (
            "PASS" if self.passed else ("SKIP" if self.tolerance == 0 else "FAIL"), self.name, self.max_error,
            self.tolerance, ", " if self.detail else "", self.detail)


# ------------------------------------------------------------------ data
def _cm(m: np.ndarray) -> np.ndarray:
    return np.asarray(m).reshape(-1, order="F")


def random_stage(rng, nx: int, nu: int) -> np.ndarray:
    """random_stage (oracles.hpp:39-54): [A B c Q R M q r], R SPD, [Q M'; M R] PSD + shift."""
    A = rng.uniform(-1, 1, (nx, nx)) / np.sqrt(nx)
    B = rng.uniform(-1, 1, (nx, nu))
    c = 0.5 * rng.uniform(-1, 1, nx)
    G = rng.uniform(-1, 1, (nx + nu, nx + nu))
    H = G @ G.T / (nx + nu) + 1e-3 * np.eye(nx + nu)
    Q, M, R = H[:nx, :nx], H[nx:, :nx], H[nx:, nx:] + 0.1 * np.eye(nu)
    return np.concatenate([_cm(A), _cm(B), c, _cm(Q), _cm(R), _cm(M), rng.uniform(-1, 1, nx), rng.uniform(-1, 1, nu)])


def random_terminal(rng, nx: int) -> np.ndarray:
    G = rng.uniform(-1, 1, (nx, nx))
    return np.concatenate([_cm(G @ G.T / nx + 1e-3 * np.eye(nx)), rng.uniform(-1, 1, nx)])


def random_tree_models(rng, tree, nx: int, nu: int):
    """random_tree_models (oracles.hpp:63-83): stages, edge offsets, leaf costs."""
    n = tree.node_count
    stage = np.zeros((n, 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu))
    defect = np.zeros((n, nx))
    leaf = np.zeros((n, nx * nx + nx))
    for i in range(n):
        if tree.child_count[i]:
            stage[i] = random_stage(rng, nx, nu)
        else:
            leaf[i] = random_terminal(rng, nx)
        if i > 0:
            defect[i] = 0.5 * rng.uniform(-1, 1, nx)
    return stage, defect, leaf


def _unpack(s: np.ndarray, nx: int, nu: int):
    o, out = 0, []
    for r, c in ((nx, nx), (nx, nu), (nx, 0), (nx, nx), (nu, nu), (nu, nx), (nx, 0), (nu, 0)):  # c = 0: vector
        out.append(s[o:o + r * c].reshape((r, c), order="F") if c else s[o:o + r].copy())
        o += r * max(c, 1)
    return out  # A B c Q R M q r


# --------------------------------------------------------- host references
def host_riccati(tree, nx: int, nu: int, stage, defect, leaf):
    """Sequential tree Riccati recursion (riccati.hpp:22-43, 97-122): values
    P, p per node and policies K, k per non-leaf node."""
    n = tree.node_count
    P, p = np.zeros((n, nx, nx)), np.zeros((n, nx))
    K, k = np.zeros((n, nu, nx)), np.zeros((n, nu))
    for i in reversed(range(n)):
        if tree.child_count[i] == 0:
            P[i] = leaf[i, :nx * nx].reshape((nx, nx), order="F")
            p[i] = leaf[i, nx * nx:]
            continue
        A, B, _, Q, R, M, q, r = _unpack(stage[i], nx, nu)
        chs = range(tree.first_child[i], tree.first_child[i] + tree.child_count[i])
        Pn = sum(P[c] for c in chs)
        pn = sum(p[c] + P[c] @ defect[c] for c in chs)
        Qxx, Qux, Quu = Q + A.T @ Pn @ A, M + B.T @ Pn @ A, R + B.T @ Pn @ B
        qx, qu = q + A.T @ pn, r + B.T @ pn
        K[i] = -np.linalg.solve(Quu, Qux)
        k[i] = -np.linalg.solve(Quu, qu)
        Pi = Qxx + Qux.T @ K[i]
        P[i] = 0.5 * (Pi + Pi.T)
        p[i] = qx + Qux.T @ k[i]
    return P, p, K, k


def host_rollout(tree, nx: int, nu: int, stage, defect, K, k, dx0):
    """Sequential closed-loop rollout (lqr_scan.hpp:190-200 sequential_rollout):
    du = K dx + k, dx_child = A dx + B du + d_child."""
    n = tree.node_count
    dx, du = np.zeros((n, nx)), np.zeros((n, nu))
    dx[0] = dx0
    for i in range(n):
        if tree.child_count[i] == 0:
            continue
        A, B = _unpack(stage[i], nx, nu)[:2]
        du[i] = K[i] @ dx[i] + k[i]
        for c in range(tree.first_child[i], tree.first_child[i] + tree.child_count[i]):
            dx[c] = A @ dx[i] + B @ du[i] + defect[c]
    return dx, du


def dense_tree_qp(tree, nx: int, nu: int, stage, defect, leaf, x0):
    """Brute-force KKT solve of the tree QP (oracles.hpp dense_tree_qp): states
    of every node, inputs of every non-leaf node."""
    n = tree.node_count
    nl = [i for i in range(n) if tree.child_count[i]]
    uidx = {i: n * nx + j * nu for j, i in enumerate(nl)}
    nz = n * nx + len(nl) * nu
    H, g = np.zeros((nz, nz)), np.zeros(nz)
    rows = []
    for i in range(n):
        xs = slice(i * nx, (i + 1) * nx)
        if tree.child_count[i] == 0:
            H[xs, xs] += leaf[i, :nx * nx].reshape((nx, nx), order="F")
            g[xs] += leaf[i, nx * nx:]
            continue
        A, B, _, Q, R, M, q, r = _unpack(stage[i], nx, nu)
        us = slice(uidx[i], uidx[i] + nu)
        H[xs, xs] += Q
        H[us, us] += R
        H[us, xs] += M
        H[xs, us] += M.T
        g[xs] += q
        g[us] += r
        for c in range(tree.first_child[i], tree.first_child[i] + tree.child_count[i]):
            row = np.zeros((nx, nz))
            row[:, c * nx:(c + 1) * nx] = np.eye(nx)
            row[:, xs] = -A
            row[:, us] = -B
            rows.append((row, defect[c]))
    E0 = np.zeros((nx, nz))
    E0[:, :nx] = np.eye(nx)
    E = np.vstack([E0] + [r for r, _ in rows])
    e = np.concatenate([x0] + [d for _, d in rows])
    kkt = np.block([[H, E.T], [E, np.zeros((E.shape[0], E.shape[0]))]])
    sol = np.linalg.solve(kkt, np.concatenate([-g, e]))
    x = sol[:n * nx].reshape(n, nx)
    u = np.zeros((n, nu))
    for i in nl:
        u[i] = sol[uidx[i]:uidx[i] + nu]
    return x, u


def _rel(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12))


def _gpu(ctx, tree, nx, nu, stage, defect, leaf, dx0, seq_max):
    set_seq_max_len(ctx, seq_max)
    try:
        return lqr_tree(tree, nx, nu, stage, defect, leaf, 0.0, dx0, ctx=ctx)
    finally:
        set_seq_max_len(ctx, -1)


# ------------------------------------------------------------------ suites
def check_scan_vs_riccati(ctx: Context, seed: int = 12345, mutate_scan_sign: bool = False) -> CheckResult:
    res = CheckResult("scan-vs-riccati", False, 0.0, 1e-8)
    rng = np.random.default_rng(seed)
    count = 0
    for nx in (2, 4, 8):
        for nu in (1, 2, 4):
            for N in (8, 64, 511):
                tree = build_tree(N, [])
                stage, defect, leaf = random_tree_models(rng, tree, nx, nu)
                P, p, _, _ = host_riccati(tree, nx, nu, stage, defect, leaf)
                fed = -defect if mutate_scan_sign else defect
                got = _gpu(ctx, tree, nx, nu, stage, fed, leaf, np.zeros(nx), 0)
                for i in range(tree.node_count):
                    res.max_error = max(res.max_error, _rel(got["P"][i].reshape((nx, nx), order="F"), P[i]),
                                        _rel(got["p"][i], p[i]))
                count += 1
    res.detail = "%d instances" % count
    res.passed = res.max_error <= res.tolerance
    return res


def check_forward_scan(ctx: Context, seed: int = 12346) -> CheckResult:
    res = CheckResult("forward-scan-vs-rollout", False, 0.0, 1e-10)
    rng = np.random.default_rng(seed)
    count = 0
    for nx in (2, 4, 8):
        for nu in (1, 2, 4):
            for N in (8, 64, 511):
                tree = build_tree(N, [])
                stage, defect, leaf = random_tree_models(rng, tree, nx, nu)
                dx0 = rng.uniform(-1, 1, nx)
                got = _gpu(ctx, tree, nx, nu, stage, defect, leaf, dx0, 0)
                K = got["K"].reshape(-1, nx, nu).transpose(0, 2, 1)  # column-major nu x nx
                dx, _ = host_rollout(tree, nx, nu, stage, defect, K, got["k"], dx0)
                res.max_error = max(res.max_error, max(_rel(got["dx"][i], dx[i]) for i in range(tree.node_count)))
                count += 1
    res.detail = "%d instances" % count
    res.passed = res.max_error <= res.tolerance
    return res


def check_tree_qp(ctx: Context, seed: int = 12349) -> CheckResult:
    res = CheckResult("tree-riccati-vs-dense-qp", False, 0.0, 1e-7)
    rng = np.random.default_rng(seed)
    trees = [build_tree(7, [(3, 2, [0.5, 0.5])]), build_tree(6, [(2, 2, [0.5, 0.5]), (4, 2, [0.4, 0.6])])]
    for tree in trees:
        nx, nu = 4, 2
        stage, defect, leaf = random_tree_models(rng, tree, nx, nu)
        x0 = rng.uniform(-1, 1, nx)
        xq, uq = dense_tree_qp(tree, nx, nu, stage, defect, leaf, x0)
        got = _gpu(ctx, tree, nx, nu, stage, defect, leaf, x0, -1)
        for i in range(tree.node_count):
            res.max_error = max(res.max_error, _rel(got["dx"][i], xq[i]))
            if tree.child_count[i]:
                res.max_error = max(res.max_error, _rel(got["du"][i], uq[i]))
    res.detail = "12-node/2-leaf and 15-node/4-leaf topologies"
    res.passed = res.max_error <= res.tolerance
    return res


# Element dims compiled for the kernel-level primitives (the reference draws
# nx in [2, 4], nu in [1, 3]; these are its combinations the library builds).
_ASSOC_DIMS = ((2, 1), (2, 2), (3, 2), (4, 1), (4, 2))


def _rel1(a, b) -> float:
    """relative_error (oracles.hpp): |a - b| / max(1, |b|)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1.0))


def check_associativity(ctx: Context, seed: int = 12347, triples: int = 1000) -> CheckResult:
    """(a (+) b) (+) c vs a (+) (b (+) c) for the backward elements of random
    stages (init_bwd_element) and for random forward affine maps, every
    combination on the GPU (bmpc_lqr_elements)."""
    res = CheckResult("associativity", False, 0.0, 1e-9)
    rng = np.random.default_rng(seed)
    per = max(1, triples // len(_ASSOC_DIMS))
    for nx, nu in _ASSOC_DIMS:
        st = np.stack([random_stage(rng, nx, nu) for _ in range(3 * per)])
        e = lqr_elements("init_bwd", nx, nu, st, ctx=ctx)
        a, b, c = e[:per], e[per:2 * per], e[2 * per:]
        left = lqr_elements("combine_bwd", nx, nu, lqr_elements("combine_bwd", nx, nu, a, b, ctx=ctx), c, ctx=ctx)
        right = lqr_elements("combine_bwd", nx, nu, a, lqr_elements("combine_bwd", nx, nu, b, c, ctx=ctx), ctx=ctx)
        n2 = nx * nx
        blocks = ((0, n2), (n2, n2 + nx), (n2 + nx, 2 * n2 + nx), (2 * n2 + nx, 3 * n2 + nx),
                  (3 * n2 + nx, 3 * n2 + 2 * nx))  # P p C A c
        for t in range(per):
            for lo, hi in blocks:
                res.max_error = max(res.max_error, _rel1(left[t, lo:hi], right[t, lo:hi]))
        f = np.concatenate([rng.uniform(-1, 1, (3 * per, nx * nx)), rng.uniform(-1, 1, (3 * per, nx))], axis=1)
        fa, fb, fc = f[:per], f[per:2 * per], f[2 * per:]
        fl = lqr_elements("combine_fwd", nx, nu, lqr_elements("combine_fwd", nx, nu, fa, fb, ctx=ctx), fc, ctx=ctx)
        fr = lqr_elements("combine_fwd", nx, nu, fa, lqr_elements("combine_fwd", nx, nu, fb, fc, ctx=ctx), ctx=ctx)
        for t in range(per):
            res.max_error = max(res.max_error, _rel1(fl[t, :n2], fr[t, :n2]), _rel1(fl[t, n2:], fr[t, n2:]))
    res.detail = "%d triples per combinator on the GPU" % (per * len(_ASSOC_DIMS))
    res.passed = res.max_error <= res.tolerance
    return res


def check_condensing(ctx: Context, seed: int = 12348) -> CheckResult:
    """The condensed shared segment (scan_condensed, solver.hpp:297-307) on
    the GPU: its open-loop inputs k = u at every shared node must equal the
    inputs of the tree Riccati solution along its rollout (the same strictly
    convex QP) — against the GPU tree scan and the host Riccati recursion —
    on the reference's three small trees and on a path condensed against a
    late branching (verification.hpp:141-223: path 1e-8, tree 1e-7)."""
    res = CheckResult("condensing", False, 0.0, 1e-7)
    rng = np.random.default_rng(seed)
    trees = [build_tree(6, [(4, 2, [0.5, 0.5])]), build_tree(5, [(2, 3, [0.3, 0.4, 0.3])]),
             build_tree(6, [(2, 2, [0.5, 0.5]), (4, 2, [0.25, 0.75])]), build_tree(7, [(6, 2, [0.5, 0.5])])]
    shared_nodes = 0
    try:
        for tree in trees:
            nx, nu = 3, 2
            stage, defect, leaf = random_tree_models(rng, tree, nx, nu)
            x0 = rng.uniform(-1, 1, nx)
            set_lqr_strategy(ctx, "scan-condensed")
            cond = lqr_tree(tree, nx, nu, stage, defect, leaf, 0.0, x0, ctx=ctx)
            set_lqr_strategy(ctx, "scan-tree-riccati")
            scan = lqr_tree(tree, nx, nu, stage, defect, leaf, 0.0, x0, ctx=ctx)
            _, _, K, k = host_riccati(tree, nx, nu, stage, defect, leaf)
            _, hdu = host_rollout(tree, nx, nu, stage, defect, K, k, x0)
            m = int(tree.step_begin[tree.last_branch_step + 1])  # nodes with step <= N_b
            for i in range(m):
                u = cond["k"][i]
                assert np.all(cond["K"][i] == 0.0), "condensed policies must be open loop"
                res.max_error = max(res.max_error, _rel1(u, scan["du"][i]), _rel1(u, hdu[i]))
            for i in range(tree.node_count):  # the rollouts coincide everywhere
                res.max_error = max(res.max_error, _rel1(cond["dx"][i], scan["dx"][i]))
            shared_nodes += m
    finally:
        set_lqr_strategy(ctx, "scan-tree-riccati")
    res.detail = "%d shared nodes on 4 trees vs GPU tree scan and host Riccati" % shared_nodes
    res.passed = res.max_error <= res.tolerance
    return res


def check_cross_strategy(ctx: Context, seed: int = 12350) -> CheckResult:
    res = CheckResult("cross-strategy", False, 0.0, 1e-6)
    rng = np.random.default_rng(seed)
    trees = [build_tree(6, [(4, 2, [0.5, 0.5])]), build_tree(6, [(2, 2, [0.5, 0.5]), (4, 3, [0.2, 0.3, 0.5])]),
             build_tree(5, [])]
    for tree in trees:
        nx, nu = 3, 2
        stage, defect, leaf = random_tree_models(rng, tree, nx, nu)
        dx0 = rng.uniform(-1, 1, nx)
        scan = _gpu(ctx, tree, nx, nu, stage, defect, leaf, dx0, 0)
        sweep = _gpu(ctx, tree, nx, nu, stage, defect, leaf, dx0, _SWEEP_ALL)
        _, _, K, k = host_riccati(tree, nx, nu, stage, defect, leaf)
        hdx, hdu = host_rollout(tree, nx, nu, stage, defect, K, k, dx0)
        for other_dx, other_du in ((sweep["dx"], sweep["du"]), (hdx, hdu)):
            for i in range(tree.node_count):
                res.max_error = max(res.max_error, _rel(other_dx[i], scan["dx"][i]))
                if tree.child_count[i]:
                    res.max_error = max(res.max_error, _rel(other_du[i], scan["du"][i]))
    res.detail = "GPU scan / GPU team sweep / host Riccati"
    res.passed = res.max_error <= res.tolerance
    return res


def run_suites(names: Sequence[str] = (), mutate: Optional[str] = None, ctx: Optional[Context] = None,
               seed: int = 12345) -> List[CheckResult]:
    """run_suites (verification.hpp:302-319): empty / "all" selects every suite."""
    if mutate not in (None, "", "scan-sign"):
        raise ValueError("unknown mutation '%s'" % mutate)
    wants = lambda n: not names or n in names or "all" in names
    if not any(wants(n) for n in SUITES):
        return []
    ctx = ctx or default_context()
    out = []
    if wants("scan-riccati"):
        out.append(check_scan_vs_riccati(ctx, seed, mutate_scan_sign=mutate == "scan-sign"))
    if wants("forward"):
        out.append(check_forward_scan(ctx, seed + 1))
    if wants("associativity"):
        out.append(check_associativity(ctx, seed + 2))
    if wants("condensing"):
        out.append(check_condensing(ctx, seed + 3))
    if wants("tree-qp"):
        out.append(check_tree_qp(ctx, seed + 4))
    if wants("cross-strategy"):
        out.append(check_cross_strategy(ctx, seed + 5))
    return out
