"""The reference's bench CLI (proj/tools/bench.cpp) on the GPU back end:
paper_2506_13624_b200.cli. CPU tests: `gen` against the reference's own
serialization (tests/golden/gen_*.json.gz from oracle/_ref/gen_ref), the
`custom` experiment's random LQ generator against the reference's problems
(golden LQ fixtures, oracles.hpp:316) and the C restatement, and the config
error paths (exit 2, bench.cpp:123-160). GPU tests: `run` sweeps, CSV schema
and values against the reference's golden solves / the oracle."""
import gzip
import io
import json
import os

import numpy as np
import pytest

import _oracle as O
import paper_2506_13624_b200 as B
from paper_2506_13624_b200 import cli

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.mark.parametrize("scen", ["intersection", "latency"])
def test_gen_matches_reference_serialization(tmp_path, scen):
    out = tmp_path / ("%s.json" % scen)
    assert cli.gen_command(scen, str(out), out=io.StringIO()) == 0
    got = json.loads(out.read_text())
    with gzip.open(os.path.join(GOLDEN, "gen_%s.json.gz" % scen), "rt") as f:
        want = json.load(f)
    assert got == want  # every number bit-identical (json floats round-trip)


def test_gen_unknown_scenario(tmp_path):
    assert cli.gen_command("roundabout", str(tmp_path / "x.json"), err=io.StringIO()) == 2


def test_mt19937_64_matches_libstdcxx():
    g = cli.MT19937_64(42)
    got = np.array([g.uniform() for _ in range(2000)])
    np.testing.assert_array_equal(got, O.mt_uniform(42, 2000))


@pytest.mark.parametrize("name", ["lq_6_branch2_nx3nu2", "lq_7_branch3_nx3nu2", "lq_5_path_nx2nu1"])
def test_random_lq_matches_reference_problems(name):
    g = _golden(name)
    meta = json.loads(str(g["meta"]))
    tree = B.build_tree(meta["horizon"], [tuple(b) for b in meta["branchings"]])
    x0, stage, leaf = cli.random_lq_data(cli.MT19937_64(meta["seed"]), tree, meta["nx"], meta["nu"])
    np.testing.assert_array_equal(x0, g["x0"])
    nl = tree.child_count > 0
    np.testing.assert_array_equal(stage[nl], g["stage"][nl])
    np.testing.assert_array_equal(leaf[~nl], g["leaf"][~nl])


def test_custom_points_match_c_restatement():
    cfg = cli.parse_run_config({"experiment": "custom", "horizons": [7], "leaf_counts": [1, 3], "seed": 5})
    g = cli.MT19937_64(5)
    for leaves in (1, 3):
        tree = B.build_tree(7, [(1, leaves, [1.0 / leaves] * leaves)]) if leaves > 1 else B.build_tree(7, [])
        x0, stage, leaf = cli.random_lq_data(g, tree, 4, 2)
        if leaves == 1:  # the first point draws from a fresh generator
            ot = dict(parent=tree.parent, nchild=tree.child_count)
            ox0, ost, olf = O.random_lq(5, ot, 4, 2)
            np.testing.assert_array_equal(x0, ox0)
            np.testing.assert_array_equal(stage[:-1], ost[:-1])
            np.testing.assert_array_equal(leaf[-1], olf[-1])
    assert cfg["repetitions"] == 1 and cfg["output"] == "bench_results.csv"


def test_solver_presets_override_strategies():
    cfg = cli.parse_run_config({"options": {"forward": "nonlinear", "line_search": "sequential"}})
    cli.apply_solver_name("pmsilqr", cfg["options"])  # bench.cpp:59-64: the preset wins
    assert (cfg["options"].forward, cfg["options"].line_search) == ("linear", "parallel")
    cfg["options"]._c()  # runs on the GPU path
    cli.apply_solver_name("sssilqr", cfg["options"])  # bench.cpp:74-79
    c = cfg["options"]._c()
    assert (c.backward, c.forward, c.line_search) == (2, 1, 1)
    assert cfg["options"].parallel is False
    cli.apply_solver_name("smsilqr", cfg["options"])
    c = cfg["options"]._c()
    assert (c.backward, c.forward, c.line_search) == (2, 0, 1)


@pytest.mark.parametrize("cfg,msg", [
    ("{not json", "bad config JSON"),
    ('{"solver": "fastest"}', "unknown solver"),
    ('{"repetitions": 0}', "repetitions must be >= 1"),
    ('{"experiment": "leaf-sweep", "leaf_counts": []}', "empty sweep list"),
    ('{"experiment": "leaf-sweep", "leaf_counts": [5]}', "unsupported leaf count 5"),
    ('{"experiment": "warp-sweep"}', "unknown experiment"),
    ('{"options": {"bogus": 1}}', "unknown solver option: bogus"),
    ('{"options": {"backward": "magic"}}', "unknown backward strategy: magic"),
])
def test_run_config_errors(tmp_path, cfg, msg):
    p = tmp_path / "c.json"
    p.write_text(cfg)
    err = io.StringIO()
    assert cli.run_command(str(p), out=io.StringIO(), err=err) == 2
    assert msg in err.getvalue()
    assert cli.run_command(str(tmp_path / "missing.json"), err=io.StringIO()) == 2


@pytest.mark.gpu
def test_run_sweeps_match_reference(tmp_path, monkeypatch):
    monkeypatch.setenv("BMPC_OUT_DIR", str(tmp_path))
    cases = [({"experiment": "horizon-sweep", "horizons": [63], "repetitions": 2, "output": "h.csv"},
              "cfg0_intersection_63"),
             ({"experiment": "latency-sweep", "horizons": [63], "tsh1_values": [0.5], "output": "l.csv",
               "options": {"max_inner_iterations": 100}}, None)]
    for cfg, golden in cases:
        p = tmp_path / "c.json"
        p.write_text(json.dumps(cfg))
        out = io.StringIO()
        assert cli.run_command(str(p), out=out, err=io.StringIO()) == 0
        lines = (tmp_path / cfg["output"]).read_text().splitlines()
        assert lines[0] == cli.CSV_HEADER
        rows = [l.split(",") for l in lines[1:]]
        assert len(rows) == cfg.get("repetitions", 1)
        for r in rows:
            assert len(r) == 16 and r[-1] == "converged"
            assert float(r[13]) > 0.0  # t_total_ms (device time)
        if golden:
            rep = json.loads(str(_golden(golden)["report"]))
            for r in rows:
                assert int(r[6]) == rep["inner_iterations"]
                assert abs(float(r[7]) - rep["final_cost"]) <= 1e-8 * abs(rep["final_cost"])
    # The latency point latency_spec(0.5, 63) (T = 5 s, T_sh0 = 0.05 s) is the
    # golden latency_0p5_63 problem (test_solver.cpp:537).
    rep = json.loads(str(_golden("latency_0p5_63")["report"]))
    row = (tmp_path / "l.csv").read_text().splitlines()[1].split(",")
    assert int(row[6]) == rep["inner_iterations"]
    assert abs(float(row[7]) - rep["final_cost"]) <= 1e-8 * abs(rep["final_cost"])


@pytest.mark.gpu
def test_run_custom_matches_oracle(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"experiment": "custom", "horizons": [15], "leaf_counts": [1], "seed": 9,
                             "output": str(tmp_path / "c.csv")}))
    assert cli.run_command(str(p), out=io.StringIO(), err=io.StringIO()) == 0
    row = (tmp_path / "c.csv").read_text().splitlines()[1].split(",")
    tree = B.build_tree(15, [])
    x0, stage, leaf = cli.random_lq_data(cli.MT19937_64(9), tree, 4, 2)
    ref = O.solve_problem(B.lq_problem(tree, 4, 2, x0, stage, leaf))
    rep = ref
    assert int(row[6]) == rep["inner_iterations"]
    assert abs(float(row[7]) - rep["final_cost"]) <= 1e-8 * max(1.0, abs(rep["final_cost"]))


@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["smsilqr", "sssilqr"])
def test_run_presets_match_reference(tmp_path, monkeypatch, solver):
    """`bench run` with the other presets (apply_solver_name, bench.cpp:60-83)
    on the GPU: the CSV row carries the reference preset's counts and cost."""
    monkeypatch.setenv("BMPC_OUT_DIR", str(tmp_path))
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"experiment": "horizon-sweep", "horizons": [63], "solver": solver, "output": "p.csv"}))
    assert cli.run_command(str(p), out=io.StringIO(), err=io.StringIO()) == 0
    row = (tmp_path / "p.csv").read_text().splitlines()[1].split(",")
    rep = json.loads(str(_golden("preset_%s_cfg0_intersection_63" % solver)["report"]))
    assert row[-1] == "converged"
    assert int(row[6]) == rep["inner_iterations"]
    assert abs(float(row[7]) - rep["final_cost"]) <= 1e-8 * max(1.0, abs(rep["final_cost"]))


@pytest.mark.gpu
def test_run_is_reproducible_except_timing(tmp_path):
    """cli_reproducible (tests/CMakeLists.txt:39-44): the same config and seed
    run twice give identical CSVs once the timing columns are cut away
    (`cut -d, -f1-9,16`: keep columns 1-9 and 16). Custom (random LQ, seeded
    mt19937_64) and scenario sweeps, with the hypmsilqr preset too."""
    cfgs = [{"experiment": "custom", "solver": "pmsilqr", "horizons": [10], "leaf_counts": [2], "repetitions": 1,
             "seed": 3},
            {"experiment": "horizon-sweep", "horizons": [31, 63], "repetitions": 2},
            {"experiment": "horizon-sweep", "horizons": [63], "solver": "hypmsilqr"}]
    for n, cfg in enumerate(cfgs):
        runs = []
        for rep in ("a", "b"):
            out = tmp_path / f"r{n}{rep}.csv"
            p = tmp_path / "c.json"
            p.write_text(json.dumps(dict(cfg, output=str(out))))
            assert cli.run_command(str(p), out=io.StringIO(), err=io.StringIO()) == 0
            lines = out.read_text().splitlines()
            runs.append([",".join(r.split(",")[:9] + [r.split(",")[15]]) for r in lines])
        assert runs[0] == runs[1]
        assert len(runs[0]) >= 2 and runs[0][1].endswith("converged")
