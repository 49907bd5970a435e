// adapter_check — test infrastructure: the C++ drop-in (include/bmpc_b200.hpp)
// against the UNMODIFIED reference solve() on the same BmpcProblem objects,
// built by the reference's own builders (compiled here against the Eigen shim,
// see Makefile). Mirrors the call sites the drop-in replaces:
// tests/acceptance_test.cpp:93-102 (cfg0), tests/test_solver.cpp:414-551
// (solver fixtures, latency case, initial inputs), README.md:134-145 (usage),
// and testing::random_lq_problem (oracles.hpp:316) for the LQ family.
//
// Prints one JSON object per case and exits 1 on any parity failure.
// Parity bar (north star): identical status / inner / outer iteration counts
// and per-iteration alpha + acceptance sequences; trajectories and final cost
// within 1e-8 relative.
#include <bmpc/bmpc.hpp>
#include <bmpc/testing/oracles.hpp>

#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "bmpc_b200.hpp"

namespace {

constexpr double kTol = 1e-8;
int failures = 0;

double traj_rel_err(const bmpc::TrajectoryTree& a, const bmpc::TrajectoryTree& b) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < b.state.size(); ++i) {
    num += (a.state[i] - b.state[i]).squaredNorm();
    den += b.state[i].squaredNorm();
    if (b.input[i].size()) {
      num += (a.input[i] - b.input[i]).squaredNorm();
      den += b.input[i].squaredNorm();
    }
  }
  return std::sqrt(num) / std::max(std::sqrt(den), 1e-12);
}

void compare(const std::string& name, const bmpc::SolveResult& got, const bmpc::SolveResult& want) {
  const auto& g = got.report;
  const auto& w = want.report;
  bool same_seq = g.iterations.size() == w.iterations.size();
  for (size_t k = 0; same_seq && k < w.iterations.size(); ++k)
    same_seq = g.iterations[k].alpha == w.iterations[k].alpha &&
               g.iterations[k].accepted == w.iterations[k].accepted && g.iterations[k].outer == w.iterations[k].outer;
  const double traj = traj_rel_err(got.trajectory, want.trajectory);
  const double cost = std::abs(g.final_cost - w.final_cost) / std::max(1.0, std::abs(w.final_cost));
  const bool ok = g.status == w.status && g.inner_iterations == w.inner_iterations &&
                  g.outer_iterations == w.outer_iterations && same_seq && traj <= kTol && cost <= kTol;
  if (!ok) ++failures;
  std::printf(
      "{\"case\": \"%s\", \"ok\": %s, \"status\": [\"%s\", \"%s\"], \"inner\": [%d, %d], \"outer\": [%d, %d], "
      "\"records\": [%zu, %zu], \"same_alpha_sequence\": %s, \"traj_rel_err\": %.3e, \"cost_rel_err\": %.3e, "
      "\"gpu_total_s\": %.6f}\n",
      name.c_str(), ok ? "true" : "false", bmpc::to_string(g.status), bmpc::to_string(w.status), g.inner_iterations,
      w.inner_iterations, g.outer_iterations, w.outer_iterations, g.iterations.size(), w.iterations.size(),
      same_seq ? "true" : "false", traj, cost, g.times.total_s);
}

void scenario_case(const std::string& name, const bmpc::ScenarioSpec& spec, bool latency, int v1, int v2,
                   const std::vector<bmpc::VectorXd>* u0 = nullptr, const bmpc::SolverOptions& opts = {}) {
  bmpc::ScenarioArtifacts art;
  const bmpc::BmpcProblem problem =
      latency ? bmpc::build_latency_case(spec, &art) : bmpc::build_intersection_case(spec, v1, v2, &art);
  const bmpc::SolveResult want = bmpc::solve(problem, opts, u0);
  const bmpc::SolveResult got = bmpc::b200::solve(problem, spec, art, opts, u0);
  compare(name, got, want);
  // The exact drop-in signature: the callbacks are probed for the scene data.
  compare(name + " [solve(problem, opts)]", bmpc::b200::solve(problem, opts, u0), want);  // was bmpc::solve
}

void lq_case(const std::string& name, int horizon, const std::vector<bmpc::TreeBranching>& br, int nx, int nu,
             uint64_t seed) {
  std::mt19937_64 rng(seed);
  const bmpc::TreeTopology tree = bmpc::build_tree(horizon, br);
  const bmpc::BmpcProblem problem = bmpc::testing::random_lq_problem(rng, tree, nx, nu);
  const bmpc::SolveResult want = bmpc::solve(problem);
  compare(name, bmpc::b200::solve_affine_quadratic(problem), want);
  compare(name + " [solve(problem)]", bmpc::b200::solve(problem), want);
}

template <class E, class F>
void expect_throw(const std::string& name, F&& f) {
  bool thrown = false;
  try {
    f();
  } catch (const E&) {
    thrown = true;
  }
  if (!thrown) ++failures;
  std::printf("{\"case\": \"%s\", \"ok\": %s}\n", name.c_str(), thrown ? "true" : "false");
}

}  // namespace

int main() {
  using bmpc::intersection_spec;
  using bmpc::latency_spec;
  // cfg0: the acceptance problem (acceptance_test.cpp:93-94).
  scenario_case("cfg0 intersection_spec(63,10,0.1) 2x2", intersection_spec(63, 10.0, 0.1), false, 2, 2);
  // Solver fixtures (test_solver.cpp:414, 474, 525, 537, 544).
  scenario_case("intersection_spec(20,4,0.4) 2x2", intersection_spec(20, 4.0, 0.4), false, 2, 2);
  scenario_case("intersection_spec(25,5,0.4) 1x2", intersection_spec(25, 5.0, 0.4), false, 1, 2);
  scenario_case("intersection_spec(25,5,0.4) 2x2", intersection_spec(25, 5.0, 0.4), false, 2, 2);
  scenario_case("latency_spec(0.5,63,5,0.05)", latency_spec(0.5, 63, 5.0, 0.05), true, 0, 0);
  scenario_case("latency_spec(1.5,63,5,0.05)", latency_spec(1.5, 63, 5.0, 0.05), true, 0, 0);
  // cfg1 points (long horizon, one-block and whole-GPU paths).
  scenario_case("cfg1 intersection_spec(255,10,0.1) 2x2", intersection_spec(255, 10.0, 0.1), false, 2, 2);
  scenario_case("cfg1 intersection_spec(500,10,0.1) 2x2", intersection_spec(500, 10.0, 0.1), false, 2, 2);
  // initial_inputs (solver.hpp:604-608).
  {
    const bmpc::ScenarioSpec spec = intersection_spec(63, 10.0, 0.1);
    const bmpc::TreeTopology tree = bmpc::build_intersection_case(spec, 2, 2).tree;
    std::vector<bmpc::VectorXd> u0(static_cast<size_t>(tree.node_count));
    for (int i = 0; i < tree.node_count; ++i)
      u0[static_cast<size_t>(i)] = tree.is_leaf(i) ? bmpc::VectorXd() : bmpc::VectorXd::Constant(2, 0.05 * (i % 3));
    scenario_case("cfg0 with initial_inputs", spec, false, 2, 2, &u0);
  }
  // Affine-quadratic family (random_lq_problem): one Newton step converges.
  lq_case("lq (4,2) N=30 2x2", 30, {{5, 2, {0.5, 0.5}}, {12, 2, {0.3, 0.7}}}, 4, 2, 7);
  lq_case("lq (3,2) N=64 3-ary", 64, {{10, 3, {0.2, 0.3, 0.5}}}, 3, 2, 11);
  lq_case("lq (2,1) N=100 path", 100, {}, 2, 1, 13);
  // Error behaviour.
  // The other presets (apply_solver_name, tools/bench.cpp:60-83).
  {
    bmpc::SolverOptions sm;
    sm.backward = bmpc::BackwardStrategy::sequential_riccati;
    sm.line_search = bmpc::LineSearchMode::sequential;
    sm.parallel = false;
    bmpc::SolverOptions ss = sm;
    ss.forward = bmpc::ForwardMode::nonlinear_rollout;
    scenario_case("smsilqr cfg0", intersection_spec(63, 10.0, 0.1), false, 2, 2, nullptr, sm);
    scenario_case("sssilqr cfg0", intersection_spec(63, 10.0, 0.1), false, 2, 2, nullptr, ss);
    scenario_case("sssilqr latency_spec(1.5,63,5,0.05)", latency_spec(1.5, 63, 5.0, 0.05), true, 0, 0, nullptr, ss);
    bmpc::SolverOptions hy;
    hy.backward = bmpc::BackwardStrategy::scan_condensed;
    scenario_case("hypmsilqr cfg0", intersection_spec(63, 10.0, 0.1), false, 2, 2, nullptr, hy);
    scenario_case("hypmsilqr intersection_spec(25,5,0.4) 2x2", intersection_spec(25, 5.0, 0.4), false, 2, 2, nullptr, hy);
  }
  expect_throw<std::invalid_argument>("mismatched artifacts rejected", [] {
    const bmpc::ScenarioSpec spec = intersection_spec(20, 4.0, 0.4);
    bmpc::ScenarioArtifacts art;
    const bmpc::BmpcProblem p = bmpc::build_intersection_case(spec, 2, 2, &art);
    art.reference.pop_back();
    bmpc::b200::solve(p, spec, art);
  });
  expect_throw<std::invalid_argument>("non-scenario constrained problem rejected by solve(problem)", [] {
    bmpc::BmpcProblem p = bmpc::build_intersection_case(intersection_spec(20, 4.0, 0.4), 2, 2);
    for (auto& c : p.constraint) {  // a different constraint form
      auto f = c.value;
      c.value = [f](const bmpc::VectorXd& x, const bmpc::VectorXd& u) {
        bmpc::VectorXd g = f(x, u);
        g(g.size() - 1) += 0.25 * x(0) * x(0);
        return g;
      };
    }
    bmpc::b200::solve(p);
  });
  // Recovered scene data equals the builders' own (bit for bit).
  {
    const bmpc::ScenarioSpec spec = intersection_spec(63, 10.0, 0.1);
    bmpc::ScenarioArtifacts art;
    const bmpc::BmpcProblem p = bmpc::build_intersection_case(spec, 2, 2, &art);
    const auto sc = bmpc::b200::detail::recover_unicycle(p);
    bool same = sc.why.empty() && sc.dt == spec.dt() && sc.a_max == spec.accel_limit &&
                sc.w_max == spec.yaw_rate_limit && sc.radius == spec.safety_radius;
    for (int i = 0; same && i < p.tree.node_count; ++i) {
      for (int j = 0; j < 4; ++j) same = same && sc.ref[4 * static_cast<size_t>(i) + j] == art.reference[static_cast<size_t>(i)](j);
      for (int v = 0; v < sc.nv; ++v)
        for (int j = 0; j < 2; ++j)
          same = same && sc.veh[(static_cast<size_t>(i) * sc.nv + v) * 2 + j] ==
                             art.vehicle_position[static_cast<size_t>(i)][static_cast<size_t>(v)](j);
    }
    if (!same) ++failures;
    std::printf("{\"case\": \"probed scene data bit-identical to the builder's\", \"ok\": %s, \"why\": \"%s\"}\n",
                same ? "true" : "false", sc.why.c_str());
  }
  std::printf("{\"failures\": %d}\n", failures);
  return failures ? 1 : 0;
}
