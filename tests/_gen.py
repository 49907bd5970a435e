"""Seeded random LQR-tree data (numpy analogue of testing::random_stage /
random_terminal / random_tree_models, oracles.hpp:39-83). Test inputs only."""
import numpy as np


def random_stage(rng, nx, nu):
    """[A B c Q R M q r] column-major, R SPD and [Q M'; M R] PSD + shift."""
    A = rng.uniform(-1, 1, (nx, nx)) / np.sqrt(nx)
    B = rng.uniform(-1, 1, (nx, nu))
    c = 0.5 * rng.uniform(-1, 1, nx)
    G = rng.uniform(-1, 1, (nx + nu, nx + nu))
    H = G @ G.T / (nx + nu) + 1e-3 * np.eye(nx + nu)
    Q, M, R = H[:nx, :nx], H[nx:, :nx], H[nx:, nx:] + 0.1 * np.eye(nu)
    q = rng.uniform(-1, 1, nx)
    r = rng.uniform(-1, 1, nu)
    f = lambda m: np.asarray(m).reshape(-1, order="F")
    return np.concatenate([f(A), f(B), c, f(Q), f(R), f(M), q, r])


def random_terminal(rng, nx):
    G = rng.uniform(-1, 1, (nx, nx))
    P = G @ G.T / nx + 1e-3 * np.eye(nx)
    return np.concatenate([P.reshape(-1, order="F"), rng.uniform(-1, 1, nx)])


def random_tree_models(rng, tree, nx, nu):
    n = tree.node_count
    ss = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu
    stage = np.zeros((n, ss))
    leaf = np.zeros((n, nx * nx + nx))
    defect = np.zeros((n, nx))
    for i in range(n):
        if tree.child_count[i]:
            stage[i] = random_stage(rng, nx, nu)
        else:
            leaf[i] = random_terminal(rng, nx)
        if i > 0:
            defect[i] = 0.5 * rng.uniform(-1, 1, nx)
    return stage, defect, leaf


def rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-12))
