"""Benchmark CLI of the reference (proj/tools/bench.cpp) on the GPU solver.

    python -m paper_2506_13624_b200.cli run --config <file>          sweep experiments, CSV output
    python -m paper_2506_13624_b200.cli verify [--suite <name> ...] [--mutate scan-sign]   oracle-equivalence suites
    python -m paper_2506_13624_b200.cli gen --scenario <name> --out <file>   scenario config dump

Same JSON run configuration (bench.cpp:31-57, solver options as
serialization.hpp:37-85), same experiments (horizon-sweep, leaf-sweep,
latency-sweep, custom; bench.cpp:164-222), same CSV schema and line format
(bench.cpp:230-263), same report-consistency check (bench.cpp:107-121), same
exit codes (2 on a bad config) and the same BMPC_OUT_DIR handling
(bench.cpp:98-105). Times in the CSV are the solver's PhaseTimes in device
time. Every solve runs on the GPU through the C ABI; there is no CPU path.

Strategy names: every preset runs on the GPU. "pmsilqr" is the tree scan;
"hypmsilqr" condenses the shared segment into a dense QP over its inputs and
solves it on the device (Cholesky, pivoted-LU fallback, condensed.hpp); "smsilqr" runs the team Riccati sweep on every segment with the
sequential line search; "sssilqr" adds single-shooting trials (nonlinear
rollout under the feedback policies, solver.hpp:463-467). `verify` runs the reference's
oracle-equivalence suites against the GPU back end (paper_2506_13624_b200.verify).
"""
import argparse
import json
import math
import os
import sys
from typing import List, Optional

import numpy as np

from . import (build_intersection_case, build_latency_case, build_tree, intersection_spec, latency_spec, lq_problem,
               solve)
from .serialization import scenario_artifacts_to_json, scenario_spec_to_json, solver_options_from_json

CSV_HEADER = ("experiment,solver,N,leaves,T_sh1,rep,iters,cost,violation,t_setup_ms,t_bp1_ms,"
              "t_bp2_ms,t_fwd_ms,t_ls_ms,t_total_ms,status")

GPU_SOLVERS = ("pmsilqr", "hypmsilqr", "smsilqr", "sssilqr")
ALL_SOLVERS = ("pmsilqr", "hypmsilqr", "smsilqr", "sssilqr")  # apply_solver_name, bench.cpp:59-85


class ConfigError(ValueError):
    pass


# ------------------------------------------------ random LQ (custom sweeps)
class MT19937_64:
    """std::mt19937_64 (libstdc++) — the generator of the `custom` experiment."""

    def __init__(self, seed: int):
        m = 0xFFFFFFFFFFFFFFFF
        self.mt = [seed & m]
        for i in range(1, 312):
            prev = self.mt[-1]
            self.mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & m)
        self.idx = 312

    def next(self) -> int:
        mt = self.mt
        if self.idx >= 312:
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def uniform(self) -> float:
        """uniform_real_distribution<double>(-1, 1): generate_canonical<double, 53>
        draws one 64-bit word."""
        r = float(self.next()) / 18446744073709551616.0
        if r >= 1.0:
            r = math.nextafter(1.0, 0.0)
        return r * 2.0 + -1.0


def _rmat(g: MT19937_64, r: int, c: int, scale: float = 1.0) -> List[List[float]]:
    """random_matrix (oracles.hpp:22-29): row-major fill."""
    return [[scale * g.uniform() for _ in range(c)] for _ in range(r)]


def _gram(G: List[List[float]], div: float) -> List[List[float]]:
    """G G' / div in the dense product's summation order."""
    n = len(G)
    H = [[0.0] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            acc = 0.0
            for l in range(len(G[0])):
                acc += G[i][l] * G[j][l]
            H[i][j] = acc / div
    return H


def random_lq_data(g: MT19937_64, tree, nx: int, nu: int):
    """testing::random_lq_problem (oracles.hpp:316-365) with random_stage /
    random_terminal (oracles.hpp:39-61): x0, stage [node][A B c Q R M q r],
    leaf [node][P p], column-major blocks."""
    x0 = np.array([g.uniform() for _ in range(nx)])
    n, m = tree.node_count, nx + nu
    ss = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu
    stage = np.zeros((n, ss))
    leaf = np.zeros((n, nx * nx + nx))
    cm = lambda M: np.asarray(M).reshape(len(M), -1).T.reshape(-1)  # column-major flatten
    for i in range(n):
        if tree.child_count[i] == 0:
            G = _rmat(g, nx, nx)
            P = _gram(G, float(nx))
            for d in range(nx):
                P[d][d] += 1e-3
            leaf[i] = np.concatenate([cm(P), [g.uniform() for _ in range(nx)]])
            continue
        A = _rmat(g, nx, nx, 1.0 / math.sqrt(float(nx)))
        B = _rmat(g, nx, nu)
        c = [0.5 * g.uniform() for _ in range(nx)]
        H = _gram(_rmat(g, m, m), float(m))
        for d in range(m):
            H[d][d] += 1e-3
        Q = [row[:nx] for row in H[:nx]]
        M = [row[:nx] for row in H[nx:]]
        R = [row[nx:] for row in H[nx:]]
        for d in range(nu):
            R[d][d] += 0.1
        q = [g.uniform() for _ in range(nx)]
        r = [g.uniform() for _ in range(nu)]
        stage[i] = np.concatenate([cm(A), cm(B), c, cm(Q), cm(R), cm(M), q, r])
    return x0, stage, leaf


# --------------------------------------------------------------------- run
def leaf_count_split(leaves: int):
    """bench.cpp:87-96."""
    return {1: (1, 1), 2: (1, 2), 4: (2, 2), 6: (2, 3), 9: (3, 3), 12: (3, 4)}.get(leaves, (0, 0))


def resolve_output(path: str) -> str:
    """BMPC_OUT_DIR prefixes relative paths (bench.cpp:98-105)."""
    d = os.environ.get("BMPC_OUT_DIR")
    if d is not None and not os.path.isabs(path):
        path = os.path.join(d, path)
    parent = os.path.dirname(path)
    if parent:
        os.makedirs(parent, exist_ok=True)
    return path


def report_consistent(rep) -> bool:
    """bench.cpp:107-121: mu never decreases; accepted steps satisfy their
    sufficient-decrease bound."""
    it = rep.iterations
    mu_prev = 0.0
    for k in range(rep.n_records):
        if it["mu"][k] + 1e-12 < mu_prev:
            return False
        mu_prev = it["mu"][k]
        if it["accepted"][k] and it["merit_after"][k] > it["merit_before"][k] + it["model_decrease"][k] + \
                1e-9 * (1.0 + abs(it["merit_before"][k])):
            return False
    return True


def apply_solver_name(name: str, o) -> None:
    """apply_solver_name (bench.cpp:59-85): the preset overrides the strategy
    keys of the options."""
    o.backward = {"pmsilqr": "scan-tree-riccati", "hypmsilqr": "scan-condensed"}.get(name, "sequential-riccati")
    o.forward = "nonlinear" if name == "sssilqr" else "linear"
    o.line_search = "parallel" if name in ("pmsilqr", "hypmsilqr") else "sequential"
    if name in ("smsilqr", "sssilqr"):
        o.parallel = False


def parse_run_config(j: dict) -> dict:
    """parse_run_config (bench.cpp:44-57) with the reference's defaults."""
    cfg = {"experiment": "horizon-sweep", "solver": "pmsilqr", "horizons": [], "leaf_counts": [4],
           "tsh1_values": [0.5], "repetitions": 1, "seed": 42, "output": "bench_results.csv",
           "parallel_sweep": False}
    for k in cfg:
        if k in j:
            cfg[k] = j[k]
    try:
        cfg["options"] = solver_options_from_json(j.get("options", {}))
    except ValueError as e:
        raise ConfigError(str(e))
    return cfg


def build_points(cfg: dict):
    """The sweep points of bench.cpp:164-222."""
    exp, pts = cfg["experiment"], []
    if exp == "horizon-sweep":
        for N in cfg["horizons"] or [63, 127, 255, 511]:
            pts.append((N, 4, 0.0, build_intersection_case(intersection_spec(N), 2, 2)))
    elif exp == "leaf-sweep":
        N = cfg["horizons"][0] if cfg["horizons"] else 255
        for leaves in cfg["leaf_counts"]:
            v1, v2 = leaf_count_split(leaves)
            if v1 == 0:
                raise ConfigError("unsupported leaf count %d" % leaves)
            pts.append((N, leaves, 0.0, build_intersection_case(intersection_spec(N), v1, v2)))
    elif exp == "latency-sweep":
        N = cfg["horizons"][0] if cfg["horizons"] else 255
        for tsh1 in cfg["tsh1_values"]:
            pts.append((N, 4, tsh1, build_latency_case(latency_spec(tsh1, N))))
    elif exp == "custom":
        N = cfg["horizons"][0] if cfg["horizons"] else 15
        g = MT19937_64(int(cfg["seed"]))
        for leaves in cfg["leaf_counts"]:
            tree = build_tree(N, [(1, leaves, [1.0 / leaves] * leaves)]) if leaves > 1 else build_tree(N, [])
            x0, stage, leaf = random_lq_data(g, tree, 4, 2)
            pts.append((N, leaves, 0.0, lq_problem(tree, 4, 2, x0, stage, leaf)))
    else:
        raise ConfigError("unknown experiment '%s'" % exp)
    return pts


def csv_line(cfg: dict, N: int, leaves: int, tsh1: float, rep: int, r) -> str:
    t = r.times
    return "%s,%s,%d,%d,%.4g,%d,%d,%.12g,%.6g,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f,%s" % (
        cfg["experiment"], cfg["solver"], N, leaves, tsh1, rep, r.inner_iterations, r.final_cost,
        r.final_violation, 1e3 * t["setup_s"], 1e3 * t["backward_p1_s"], 1e3 * t["backward_p2_s"],
        1e3 * t["forward_s"], 1e3 * t["line_search_s"], 1e3 * t["total_s"], r.status_name)


def run_command(config_path: str, out=sys.stdout, err=sys.stderr) -> int:
    """run_command (bench.cpp:123-291)."""
    try:
        with open(config_path) as f:
            text = f.read()
    except OSError:
        print("bench run: cannot open config %s" % config_path, file=err)
        return 2
    try:
        j = json.loads(text)
    except ValueError as e:
        print("bench run: bad config JSON: %s" % e, file=err)
        return 2
    try:
        cfg = parse_run_config(j)
    except (ConfigError, TypeError) as e:
        print("bench run: %s" % e, file=err)
        return 2
    if cfg["solver"] not in ALL_SOLVERS:
        print("bench run: unknown solver '%s'" % cfg["solver"], file=err)
        return 2
    apply_solver_name(cfg["solver"], cfg["options"])
    if cfg["repetitions"] < 1:
        print("bench run: repetitions must be >= 1", file=err)
        return 2
    exp = cfg["experiment"]
    if (exp == "leaf-sweep" and not cfg["leaf_counts"]) or (exp == "latency-sweep" and not cfg["tsh1_values"]) or \
            (exp == "custom" and not cfg["leaf_counts"]):
        print("bench run: empty sweep list", file=err)
        return 2
    try:
        points = build_points(cfg)
    except (ConfigError, ValueError) as e:
        print("bench run: %s" % e, file=err)
        return 2
    path = resolve_output(cfg["output"])
    try:
        csv = open(path, "w")
    except OSError:
        print("bench run: cannot write %s" % path, file=err)
        return 2
    with csv:
        csv.write(CSV_HEADER + "\n")
        # parallel_sweep: the GPU serialises solves on one stream, so points run in order.
        for N, leaves, tsh1, problem in points:
            solve(problem, cfg["options"])  # warm-up repetition, discarded (bench.cpp:236)
            for rep in range(cfg["repetitions"]):
                try:
                    res = solve(problem, cfg["options"])
                    r = res.report
                    if not report_consistent(r):
                        r.status = 2
                except RuntimeError as e:  # non-finite initial rollout (problem.hpp:160-162)
                    print("bench run: %s" % e, file=err)
                    continue
                line = csv_line(cfg, N, leaves, tsh1, rep, r)
                csv.write(line + "\n")
                print(line, file=out)
    print("wrote %s" % path, file=out)
    return 0


# --------------------------------------------------------------------- gen
def gen_command(scenario: str, out_path: str, out=sys.stdout, err=sys.stderr) -> int:
    """gen_command (bench.cpp:327-357) with scenario_artifacts_to_json
    (serialization.hpp:200-219)."""
    if scenario == "intersection":
        spec = intersection_spec()
        p = build_intersection_case(spec, 2, 2)
        doc = {"kind": "intersection", "v1_count": 2, "v2_count": 2}
    elif scenario == "latency":
        spec = latency_spec(0.5)
        p = build_latency_case(spec)
        doc = {"kind": "latency"}
    else:
        print("bench gen: unknown scenario '%s'" % scenario, file=err)
        return 2
    doc["spec"] = scenario_spec_to_json(spec)
    doc["problem"] = scenario_artifacts_to_json(p)
    path = resolve_output(out_path)
    try:
        with open(path, "w") as f:
            f.write(json.dumps(doc, indent=2, sort_keys=True) + "\n")
    except OSError:
        print("bench gen: cannot write %s" % path, file=err)
        return 2
    print("wrote %s" % path, file=out)
    return 0


def verify_command(suites: List[str], mutate: str, out=sys.stdout, err=sys.stderr) -> int:
    """verify_command (bench.cpp:297-325)."""
    from .verify import run_suites

    if mutate and mutate != "scan-sign":
        print("bench verify: unknown mutation '%s'" % mutate, file=err)
        return 2
    if suites == ["none"]:
        print("no suites selected: trivially passing", file=out)
        return 0
    results = run_suites(suites, mutate or None)
    if not results:
        print("bench verify: no suite matches the selection", file=err)
        return 2
    ok = True
    for r in results:
        print(r.line(), file=out)
        ok = ok and r.passed
    return 0 if ok else 1


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="bench", description="Branch-MPC solver benchmarks (GPU back end)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="run a sweep experiment from a JSON config")
    r.add_argument("--config", required=True)
    v = sub.add_parser("verify", help="run the oracle-equivalence suites on the GPU back end")
    v.add_argument("--suite", action="append", default=[],
                   help="scan-riccati, forward, associativity, condensing, tree-qp, cross-strategy, all, none")
    v.add_argument("--mutate", default="", help="fault injection for harness sanity (scan-sign)")
    g = sub.add_parser("gen", help="generate a scenario config with its problem dump")
    g.add_argument("--scenario", required=True)
    g.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            return run_command(a.config)
        if a.cmd == "verify":
            return verify_command(a.suite, a.mutate)
        return gen_command(a.scenario, a.out)
    except Exception as e:  # noqa: BLE001  (bench.cpp:386-389)
        print("bench: %s" % e, file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
