// flop_count — test/measurement infrastructure: the FP64 work of one inner
// pass of the UNMODIFIED reference solve path (compiled against the Eigen
// shim with -DBMPC_FLOP_COUNT, which counts every multiply / add / divide /
// sqrt its dense kernels execute), per phase and per non-leaf node, on cfg0
// (intersection_spec(63, 10, 0.1) 2x2, 250 nodes, 246 non-leaf). Freezes the
// constants bench.py uses for roofline.achieved (SURVEY.md §8d asked for
// exactly this confirmation of its hand-derived F_node = 8.6 kflop).
//
// Scalar arithmetic outside the shim (the unicycle derivative's v*cos etc.,
// the tracking cost's 0.5 * e'We) is not counted, nor are sin / cos: the
// figures are the dense-algebra work as executed, a lower bound of the total.
//
// Output: one JSON object.
#include <bmpc/bmpc.hpp>

#include <cstdio>

namespace {
unsigned long long snap() { return Eigen::flop_counter(); }
}  // namespace

int main() {
  using namespace bmpc;
  const BmpcProblem problem = build_intersection_case(intersection_spec(63, 10.0, 0.1), 2, 2);
  const TreeTopology& tree = problem.tree;
  int nl = 0;
  for (int i = 0; i < tree.node_count; ++i) nl += tree.is_leaf(i) ? 0 : 1;

  // One pass at the initial trajectory (zero inputs, nonlinear rollout), as solve() runs it.
  std::vector<VectorXd> u0(static_cast<size_t>(tree.node_count), VectorXd::Zero(problem.input_dim));
  const TrajectoryTree traj = nonlinear_rollout(problem, u0, problem.initial_state);
  const ALState al = ALState::Zero(problem, 10.0);
  SolverOptions opts;
  unsigned long long t0 = snap();
  const TreeStageModels models = linearize(problem, traj, al);
  const unsigned long long f_lin = snap() - t0;
  t0 = snap();
  const ProblemEval ev = evaluate(problem, traj, al);
  const unsigned long long f_eval = snap() - t0;
  BackwardPassOptions bp;
  bp.parallel = false;
  bp.dx0 = VectorXd::Zero(problem.state_dim);
  t0 = snap();
  const BackwardPassResult bres = backward_pass(models, bp);
  const unsigned long long f_bwd_scan = snap() - t0;
  BackwardPassOptions bs = bp;
  bs.strategy = BackwardStrategy::sequential_riccati;
  t0 = snap();
  const BackwardPassResult bseq = backward_pass(models, bs);
  const unsigned long long f_bwd_seq = snap() - t0;
  t0 = snap();
  const DeltaTrees delta = linear_rollout(models, bres.policy, bp.dx0, ScanOrder::tree, false);
  const unsigned long long f_fwd = snap() - t0;
  t0 = snap();
  const auto ec = expected_change_coefficients(models, delta);
  const unsigned long long f_ec = snap() - t0;
  // One line-search trial: x + alpha dx, u + alpha du, then evaluate.
  t0 = snap();
  {
    TrajectoryTree trial = traj;
    for (int i = 0; i < tree.node_count; ++i) {
      trial.state[static_cast<size_t>(i)] += 0.5 * delta.dx[static_cast<size_t>(i)];
      if (!tree.is_leaf(i)) trial.input[static_cast<size_t>(i)] += 0.5 * delta.du[static_cast<size_t>(i)];
    }
    (void)evaluate(problem, trial, al);
  }
  const unsigned long long f_alpha = snap() - t0;
  // A whole solve: total flops over its passes.
  opts.parallel = false;
  t0 = snap();
  const SolveResult res = solve(problem, opts);
  const unsigned long long f_solve = snap() - t0;
  const int passes = static_cast<int>(res.report.iterations.size()) + res.report.outer_iterations;
  const double per = 1.0 / nl;
  std::printf(
      "{\"problem\": \"cfg0 intersection_spec(63,10,0.1) 2x2\", \"nodes\": %d, \"nonleaf\": %d, "
      "\"per_nonleaf_node_flops\": {\"linearize\": %.1f, \"evaluate\": %.1f, \"backward_scan\": %.1f, "
      "\"backward_sequential_riccati\": %.1f, \"forward\": %.1f, \"expected_change\": %.1f, "
      "\"line_search_per_alpha\": %.1f}, "
      "\"F_pass_reference\": %.1f, \"F_pass_work_efficient\": %.1f, "
      "\"solve\": {\"flops\": %llu, \"passes\": %d, \"flops_per_pass_per_nonleaf\": %.1f}, "
      "\"note\": \"dense-algebra flops of the Eigen shim as executed; F_pass_* = linearize + 2 evaluate + "
      "backward + forward + EC + 11 line-search trials (reference: tree scan backward; work-efficient: "
      "sequential Riccati backward)\", \"check\": [%g, %g, %g]}\n",
      tree.node_count, nl, f_lin * per, f_eval * per, f_bwd_scan * per, f_bwd_seq * per, f_fwd * per, f_ec * per,
      f_alpha * per,
      (f_lin + 2 * f_eval + f_bwd_scan + f_fwd + f_ec + 11 * f_alpha) * per,
      (f_lin + 2 * f_eval + f_bwd_seq + f_fwd + f_ec + 11 * f_alpha) * per, f_solve, passes,
      static_cast<double>(f_solve) * per / passes, ev.cost, ec.first, bseq.max_feedforward);
  return 0;
}
