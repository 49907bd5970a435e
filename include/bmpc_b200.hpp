// bmpc_b200.hpp — C++ drop-in for the reference's solve path over the C ABI.
//
// `bmpc::b200::solve` has the signature and value semantics of
// `bmpc::solve(problem, opts, initial_inputs)` (/root/reference/proj/include/bmpc/solver.hpp:595-596)
// and returns the same `SolveResult` (solver.hpp:584-587), computed by the
// sm_100a solver behind include/bmpc_b200.h. Include it from the reference's
// tree (it needs <bmpc/bmpc.hpp>) and link libbmpc_b200.so.
//
// The reference's `BmpcProblem` holds `std::function` callbacks
// (problem.hpp:15-63), which cannot run on the device, so each model family the
// reference builds has one entry point that recovers the callbacks' data:
//   * scenario problems (unicycle RK4 + tracking + ego constraints,
//     scenarios.hpp:115-171): the builders' `ScenarioSpec` + `ScenarioArtifacts`
//     (scenarios.hpp:25-55) carry everything the callbacks capture;
//   * affine-quadratic problems (`testing::random_lq_problem`, oracles.hpp:316,
//     or any problem whose dynamics are affine and costs quadratic): the blocks
//     are read back through the callbacks themselves at x = 0, u = 0.
//
// Strategy options: every backward strategy (tree scan, condensed shared
// segment, sequential Riccati), forward mode (linear / nonlinear rollout) and
// line-search mode (parallel / sequential) of SolverOptions runs on the GPU
// with the reference's semantics; scan_order and parallel only schedule the
// reference's CPU threads and are ignored.
//
// Errors follow the reference: a non-finite initial rollout throws
// std::runtime_error (problem.hpp:160-162 throws out of solve); numerical
// failures come back as SolveStatus::error with the reference's message.
#pragma once

#include <bmpc/bmpc.hpp>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bmpc_b200.h"

namespace bmpc::b200 {

/// One device + stream (bmpc_ctx). Not thread-safe: one host thread per
/// Context, as the reference's solver is single-owner.
class Context {
 public:
  explicit Context(int device = 0) {
    if (bmpc_ctx_create(device, &ctx_) != BMPC_OK) throw std::runtime_error(bmpc_last_error());
  }
  ~Context() { bmpc_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  bmpc_ctx* get() const { return ctx_; }

 private:
  bmpc_ctx* ctx_{nullptr};
};

/// The calling thread's context on device 0 (created on first use).
inline Context& default_context() {
  static thread_local Context ctx(0);
  return ctx;
}

namespace detail {

/// TreeTopology (tree.hpp:28-44) in the ABI's flat form; children of a node
/// are contiguous in build_tree's BFS order (tree.hpp:96-115).
struct FlatTree {
  std::vector<int> parent, time_step, first_child, child_count, step_begin, leaves;
  std::vector<double> weight;
  bmpc_tree view{};

  explicit FlatTree(const TreeTopology& t)
      : parent(t.parent), time_step(t.time_step), first_child(t.node_count, -1), child_count(t.node_count, 0),
        step_begin(t.step_begin), leaves(t.leaves), weight(t.weight) {
    for (int i = 0; i < t.node_count; ++i) {
      const auto& ch = t.children[static_cast<size_t>(i)];
      child_count[static_cast<size_t>(i)] = static_cast<int>(ch.size());
      if (!ch.empty()) first_child[static_cast<size_t>(i)] = ch.front();
      for (size_t j = 1; j < ch.size(); ++j)
        if (ch[j] != ch[0] + static_cast<int>(j))
          throw std::invalid_argument("bmpc::b200: children of a node must be contiguous (build_tree order)");
    }
    view = bmpc_tree{t.node_count,        t.horizon,        t.last_branch_step,  t.leaf_count(),
                     parent.data(),       time_step.data(), weight.data(),       first_child.data(),
                     child_count.data(),  step_begin.data(), leaves.data()};
  }
};

/// SolverOptions (solver.hpp:28-58) -> bmpc_options; every field maps 1:1
/// (the strategy enums keep their numbering, solver.hpp:23-26).
inline bmpc_options to_abi(const SolverOptions& o) {
  bmpc_options a;
  bmpc_options_default(&a);
  a.max_inner_iterations = o.max_inner_iterations;
  a.max_outer_iterations = o.max_outer_iterations;
  a.alpha_levels = o.alpha_levels;
  a.armijo_beta = o.armijo_beta;
  a.merit_gamma = o.merit_gamma;
  a.merit_mu0 = o.merit_mu0;
  a.merit_mu_init = o.merit_mu_init;
  a.defect_epsilon = o.defect_epsilon;
  a.tol_defect = o.tol_defect;
  a.tol_cost = o.tol_cost;
  a.tol_feedforward = o.tol_feedforward;
  a.tol_constraint = o.tol_constraint;
  a.penalty_init = o.penalty_init;
  a.penalty_growth = o.penalty_growth;
  a.penalty_max = o.penalty_max;
  a.reg_init = o.reg_init;
  a.reg_min = o.reg_min;
  a.reg_growth = o.reg_growth;
  a.reg_decay = o.reg_decay;
  a.reg_max = o.reg_max;
  a.backward = static_cast<int>(o.backward);
  a.forward = static_cast<int>(o.forward);
  a.line_search = static_cast<int>(o.line_search);
  return a;
}

/// Runs bmpc_solve and rebuilds the reference's SolveResult.
inline SolveResult run(const BmpcProblem& problem, const FlatTree& tree, const bmpc_model_desc& model,
                       const SolverOptions& opts, const std::vector<VectorXd>* initial_inputs, Context* ctx) {
  const TreeTopology& t = problem.tree;
  const int n = t.node_count, nx = problem.state_dim, nu = problem.input_dim;
  const bmpc_options o = to_abi(opts);
  std::vector<double> u0;
  if (initial_inputs) {
    if (static_cast<int>(initial_inputs->size()) != n)
      throw std::invalid_argument("bmpc::b200::solve: initial_inputs must hold one entry per node");
    u0.assign(static_cast<size_t>(nu) * n, 0.0);
    for (int i = 0; i < n; ++i) {
      const VectorXd& ui = (*initial_inputs)[static_cast<size_t>(i)];
      if (t.is_leaf(i)) continue;
      if (ui.size() != nu) throw std::invalid_argument("bmpc::b200::solve: initial input of wrong size");
      for (int j = 0; j < nu; ++j) u0[static_cast<size_t>(nu) * i + j] = ui(j);
    }
  }
  std::vector<double> x(static_cast<size_t>(nx) * n), u(static_cast<size_t>(nu) * n);
  std::vector<bmpc_record> recs(static_cast<size_t>(o.max_inner_iterations) * o.max_outer_iterations + 1);
  bmpc_report rep{};
  Context& c = ctx ? *ctx : default_context();
  const int rc = bmpc_solve(c.get(), &tree.view, &model, &o, initial_inputs ? u0.data() : nullptr, x.data(),
                            u.data(), &rep, recs.data(), static_cast<int>(recs.size()));
  if (rc != BMPC_OK) {
    const std::string msg = bmpc_last_error();
    if (rc == BMPC_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == BMPC_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);  // incl. BMPC_ERR_ROLLOUT (problem.hpp:160-162)
  }

  SolveResult res;
  res.trajectory = TrajectoryTree::Zero(t, nx, nu);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < nx; ++j) res.trajectory.state[static_cast<size_t>(i)](j) = x[static_cast<size_t>(nx) * i + j];
    if (!t.is_leaf(i))
      for (int j = 0; j < nu; ++j) res.trajectory.input[static_cast<size_t>(i)](j) = u[static_cast<size_t>(nu) * i + j];
  }
  SolveReport& r = res.report;
  r.status = rep.status == BMPC_CONVERGED        ? SolveStatus::converged
             : rep.status == BMPC_MAX_ITERATIONS ? SolveStatus::max_iterations
                                                 : SolveStatus::error;
  r.message = rep.message;
  r.inner_iterations = rep.inner_iterations;
  r.outer_iterations = rep.outer_iterations;
  r.final_cost = rep.final_cost;
  r.final_violation = rep.final_violation;
  r.final_defect_l1 = rep.final_defect_l1;
  for (int k = 0; k < rep.n_records && k < static_cast<int>(recs.size()); ++k) {
    const bmpc_record& a = recs[static_cast<size_t>(k)];
    IterationRecord it;
    it.outer = a.outer;
    it.cost = a.cost;
    it.cost_al = a.cost_al;
    it.merit_before = a.merit_before;
    it.merit_after = a.merit_after;
    it.model_decrease = a.model_decrease;
    it.defect_l1 = a.defect_l1;
    it.violation = a.violation;
    it.alpha = a.alpha;
    it.mu = a.mu;
    it.max_feedforward = a.max_feedforward;
    it.regularization = a.regularization;
    it.accepted = a.accepted != 0;
    r.iterations.push_back(it);
  }
  r.times.setup_s = rep.times[0];
  r.times.backward_p1_s = rep.times[1];
  r.times.backward_p2_s = rep.times[2];
  r.times.forward_s = rep.times[3];
  r.times.line_search_s = rep.times[4];
  r.times.total_s = rep.times[5];
  return res;
}

}  // namespace detail

/// solve() for the scenario problems of scenarios.hpp (build_intersection_case,
/// build_latency_case): the problem must come from those builders with the
/// same `spec`, and `art` is the artifacts object they filled.
inline SolveResult solve(const BmpcProblem& problem, const ScenarioSpec& spec, const ScenarioArtifacts& art,
                         const SolverOptions& opts = {}, const std::vector<VectorXd>* initial_inputs = nullptr,
                         Context* ctx = nullptr) {
  const TreeTopology& t = problem.tree;
  const int n = t.node_count;
  if (problem.state_dim != 4 || problem.input_dim != 2)
    throw std::invalid_argument("bmpc::b200::solve: scenario problems are unicycle (nx 4, nu 2)");
  if (static_cast<int>(art.reference.size()) != n || static_cast<int>(art.vehicle_position.size()) != n)
    throw std::invalid_argument("bmpc::b200::solve: artifacts do not match the problem's tree");
  const detail::FlatTree tree(t);
  const int nv = n ? static_cast<int>(art.vehicle_position[0].size()) : 0;
  if (nv > 4) throw std::invalid_argument("bmpc::b200::solve: at most 4 surrounding vehicles");
  std::vector<double> ref(4 * static_cast<size_t>(n)), veh(2 * static_cast<size_t>(nv) * n), x0(4);
  for (int j = 0; j < 4; ++j) x0[static_cast<size_t>(j)] = problem.initial_state(j);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < 4; ++j) ref[4 * static_cast<size_t>(i) + j] = art.reference[static_cast<size_t>(i)](j);
    const auto& vp = art.vehicle_position[static_cast<size_t>(i)];
    if (static_cast<int>(vp.size()) != nv)
      throw std::invalid_argument("bmpc::b200::solve: vehicle count differs between nodes");
    for (int v = 0; v < nv; ++v)
      for (int j = 0; j < 2; ++j) veh[(static_cast<size_t>(i) * nv + v) * 2 + j] = vp[static_cast<size_t>(v)](j);
  }
  bmpc_model_desc m{};
  m.kind = BMPC_MODEL_UNICYCLE;
  m.state_dim = 4;
  m.input_dim = 2;
  m.initial_state = x0.data();
  m.dt = spec.dt();
  // Diagonal weights, column-major (tracking_cost / tracking_terminal_cost, problem.hpp:194-222).
  for (int j = 0; j < 4; ++j) {
    m.state_weights[5 * j] = spec.state_weights(j);
    m.terminal_weights[5 * j] = spec.terminal_weights(j);
  }
  for (int j = 0; j < 2; ++j) m.input_weights[3 * j] = spec.input_weights(j);
  m.accel_limit = spec.accel_limit;
  m.yaw_rate_limit = spec.yaw_rate_limit;
  m.safety_radius = spec.safety_radius;
  m.num_vehicles = nv;
  m.reference = ref.data();
  m.vehicle_position = veh.data();
  return detail::run(problem, tree, m, opts, initial_inputs, ctx);
}

/// solve() for affine-quadratic problems (testing::random_lq_problem,
/// oracles.hpp:316): dynamics x+ = A x + B u + c, stage cost
/// ½xᵀQx + qᵀx + ½uᵀRu + rᵀu + uᵀMx, terminal ½xᵀPx + pᵀx, no constraints.
/// The blocks are read through the problem's own callbacks at x = 0, u = 0.
inline SolveResult solve_affine_quadratic(const BmpcProblem& problem, const SolverOptions& opts = {},
                                          const std::vector<VectorXd>* initial_inputs = nullptr,
                                          Context* ctx = nullptr) {
  const TreeTopology& t = problem.tree;
  const int n = t.node_count, nx = problem.state_dim, nu = problem.input_dim;
  if (problem.has_constraints())
    throw std::invalid_argument("bmpc::b200::solve_affine_quadratic: constrained problems use the scenario path");
  const detail::FlatTree tree(t);
  const size_t rec = static_cast<size_t>(nx * nx + nx * nu + nx + nx * nx + nu * nu + nu * nx + nx + nu);
  const size_t leaf_rec = static_cast<size_t>(nx * nx + nx);
  std::vector<double> stage(rec * n, 0.0), leaf(leaf_rec * n, 0.0), x0(static_cast<size_t>(nx));
  for (int j = 0; j < nx; ++j) x0[static_cast<size_t>(j)] = problem.initial_state(j);
  const VectorXd z = VectorXd::Zero(nx), w = VectorXd::Zero(nu);
  const auto put = [](double* dst, const MatrixXd& M) {
    for (Eigen::Index c = 0; c < M.cols(); ++c)
      for (Eigen::Index r = 0; r < M.rows(); ++r) *dst++ = M(r, c);
    return dst;
  };
  for (int i = 0; i < n; ++i) {
    if (t.is_leaf(i)) {
      MatrixXd P;
      VectorXd p;
      problem.terminal_cost[static_cast<size_t>(i)].quadratic(z, P, p);
      put(put(leaf.data() + leaf_rec * i, P), p);
      continue;
    }
    MatrixXd A, B, Q, R, M;
    VectorXd q, r;
    problem.dynamics[static_cast<size_t>(i)].jacobians(z, w, A, B);
    const VectorXd c = problem.dynamics[static_cast<size_t>(i)].value(z, w);
    problem.cost[static_cast<size_t>(i)].quadratic(z, w, Q, R, M, q, r);
    double* d = stage.data() + rec * i;
    d = put(d, A);
    d = put(d, B);
    d = put(d, c);
    d = put(d, Q);
    d = put(d, R);
    d = put(d, M);
    d = put(d, q);
    put(d, r);
  }
  bmpc_model_desc m{};
  m.kind = BMPC_MODEL_AFFINE_QUADRATIC;
  m.state_dim = nx;
  m.input_dim = nu;
  m.initial_state = x0.data();
  m.lq_stage = stage.data();
  m.lq_leaf = leaf.data();
  return detail::run(problem, tree, m, opts, initial_inputs, ctx);
}

}  // namespace bmpc::b200
