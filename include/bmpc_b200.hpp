// bmpc_b200.hpp — C++ drop-in for the reference's solve path over the C ABI.
//
// `bmpc::b200::solve` has the signature and value semantics of
// `bmpc::solve(problem, opts, initial_inputs)` (/root/reference/proj/include/bmpc/solver.hpp:595-596)
// and returns the same `SolveResult` (solver.hpp:584-587), computed by the
// sm_100a solver behind include/bmpc_b200.h. Include it from the reference's
// tree (it needs <bmpc/bmpc.hpp>) and link libbmpc_b200.so.
//
// The reference's `BmpcProblem` holds `std::function` callbacks
// (problem.hpp:15-63), which cannot run on the device; the device solves the
// two model families the reference builds, and the data their callbacks
// capture is recovered from the callbacks themselves:
//   * `solve(problem, opts, initial_inputs)` — the drop-in — probes a scenario
//     problem (unicycle RK4 + tracking + ego constraints, scenarios.hpp:115-171)
//     for dt, weights, references, vehicle predictions, limits and radius, bit
//     for bit; the overload taking the builders' `ScenarioSpec` +
//     `ScenarioArtifacts` (scenarios.hpp:25-55) reads them directly;
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

#include <cmath>
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

namespace detail {

// Steps x0 by up to `span` ulps either way until pred holds (bit-exact
// recovery of a captured constant from a callback probe).
template <class Pred>
inline bool ulp_search(double x0, Pred pred, double* out, int span = 64) {
  if (pred(x0)) return *out = x0, true;
  double up = x0, dn = x0;
  for (int k = 0; k < span; ++k) {
    up = std::nextafter(up, HUGE_VAL);
    if (pred(up)) return *out = up, true;
    dn = std::nextafter(dn, -HUGE_VAL);
    if (pred(dn)) return *out = dn, true;
  }
  return false;
}

inline bool bit_equal(const VectorXd& a, const VectorXd& b) {
  if (a.size() != b.size()) return false;
  for (Eigen::Index i = 0; i < a.size(); ++i)
    if (!(a(i) == b(i))) return false;
  return true;
}

// Everything the scenario builders capture in a problem's callbacks
// (scenarios.hpp:115-171, problem.hpp:194-222), recovered through the
// callbacks themselves; empty `why` on success.
struct UnicycleScene {
  double dt{0}, a_max{0}, w_max{0}, radius{0};
  MatrixXd Wx, Wu, Wf;
  int nv{0};
  std::vector<double> ref, veh;  // [node][4], [node][nv][2]
  std::string why;
};

// A tracking reference ref with q(x) = W (x - ref): exact when W is diagonal
// (each component searched until q_j(ref) == 0), else the solved estimate.
template <class GradAt>
inline bool recover_reference(const MatrixXd& W, GradAt grad_at, double* ref) {
  const VectorXd q0 = grad_at(VectorXd::Zero(4));
  bool diag = true;
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) diag = diag && (r == c || W(r, c) == 0.0);
  if (!diag) {
    const VectorXd est = Eigen::PartialPivLU<MatrixXd>(W).solve(VectorXd(-q0));
    for (int j = 0; j < 4; ++j) ref[j] = est(j);
    return true;
  }
  VectorXd est(4);
  for (int j = 0; j < 4; ++j) est(j) = W(j, j) != 0.0 ? -q0(j) / W(j, j) : 0.0;
  for (int j = 0; j < 4; ++j) {
    if (W(j, j) == 0.0) {  // an unweighted component never enters the cost
      ref[j] = 0.0;
      continue;
    }
    if (!ulp_search(est(j), [&](double c) {
          VectorXd x = est;
          x(j) = c;
          return grad_at(x)(j) == 0.0;
        }, &ref[j]))
      return false;
  }
  return true;
}

inline UnicycleScene recover_unicycle(const BmpcProblem& p) {
  UnicycleScene sc;
  const TreeTopology& t = p.tree;
  const int n = t.node_count;
  auto bad = [&](const std::string& why) {
    sc.why = why;
    return sc;
  };
  if (p.state_dim != 4 || p.input_dim != 2) return bad("not (nx 4, nu 2)");
  if (!p.has_constraints() || static_cast<int>(p.constraint.size()) != n) return bad("no ego constraints");
  const int leaf0 = t.leaves.empty() ? -1 : t.leaves.front();
  if (leaf0 < 0 || t.is_leaf(0)) return bad("tree without a non-leaf root");
  sc.nv = p.constraint_dim(leaf0);
  if (sc.nv > 4) return bad("more than 4 surrounding vehicles");
  // dt: unicycle::step reproduced bit for bit (unicycle.hpp:36-42).
  VectorXd xs(4), us(2), xg(4), ug(2);
  xs << 0.0, 0.0, 0.0, 1.0;
  us << 0.0, 0.0;
  xg << 0.7, -1.3, 0.4, 2.5;
  ug << 0.3, -0.2;
  const VectorXd ys = p.dynamics[0].value(xs, us), yg = p.dynamics[0].value(xg, ug);
  if (!ulp_search(ys(0), [&](double c) {
        return bit_equal(unicycle::step(xs, us, c), ys) && bit_equal(unicycle::step(xg, ug, c), yg);
      }, &sc.dt))
    return bad("dynamics are not the unicycle RK4 step");
  // Weights (constant across nodes) and references.
  const VectorXd z4 = VectorXd::Zero(4), z2 = VectorXd::Zero(2);
  sc.ref.assign(4 * static_cast<size_t>(n), 0.0);
  sc.veh.assign(2 * static_cast<size_t>(sc.nv) * n, 0.0);
  bool have_w = false, have_f = false;
  for (int i = 0; i < n; ++i) {
    const bool leaf = t.is_leaf(i);
    if (p.constraint_dim(i) != sc.nv + (leaf ? 0 : 4)) return bad("constraint rows differ from ego_constraints");
    if (leaf) {
      MatrixXd P;
      VectorXd q;
      p.terminal_cost[static_cast<size_t>(i)].quadratic(z4, P, q);
      if (!have_f) sc.Wf = P, have_f = true;
      else if (!(P.rows() == 4 && (P - sc.Wf).cwiseAbs().maxCoeff() == 0.0)) return bad("terminal weights differ");
      if (!recover_reference(sc.Wf, [&](const VectorXd& x) {
            MatrixXd PP;
            VectorXd qq;
            p.terminal_cost[static_cast<size_t>(i)].quadratic(x, PP, qq);
            return qq;
          }, &sc.ref[4 * static_cast<size_t>(i)]))
        return bad("terminal cost is not a tracking cost");
    } else {
      if (!bit_equal(p.dynamics[static_cast<size_t>(i)].value(xg, ug), yg)) return bad("dynamics differ between nodes");
      MatrixXd Q, R, M;
      VectorXd q, r;
      p.cost[static_cast<size_t>(i)].quadratic(z4, z2, Q, R, M, q, r);
      if (M.size() && M.cwiseAbs().maxCoeff() != 0.0) return bad("stage cost has a cross term");
      if (!have_w) sc.Wx = Q, sc.Wu = R, have_w = true;
      else if ((Q - sc.Wx).cwiseAbs().maxCoeff() != 0.0 || (R - sc.Wu).cwiseAbs().maxCoeff() != 0.0)
        return bad("stage weights differ");
      if (!recover_reference(sc.Wx, [&](const VectorXd& x) {
            MatrixXd QQ, RR, MM;
            VectorXd qq, rr;
            p.cost[static_cast<size_t>(i)].quadratic(x, z2, QQ, RR, MM, qq, rr);
            return qq;
          }, &sc.ref[4 * static_cast<size_t>(i)]))
        return bad("stage cost is not a tracking cost");
      const VectorXd g = p.constraint[static_cast<size_t>(i)].value(z4, z2);
      if (i == 0) sc.a_max = -g(0), sc.w_max = -g(2);
      if (!(g(0) == -sc.a_max && g(1) == -sc.a_max && g(2) == -sc.w_max && g(3) == -sc.w_max))
        return bad("input box rows differ");
    }
    // Vehicles: J = -(p - v) / dist at two points gives v and the radius by
    // least squares; then each coordinate is searched until its Jacobian
    // entry is exactly zero (p == v), and the radius until r - sqrt(eps) == g(v).
    const NodeConstraint& con = p.constraint[static_cast<size_t>(i)];
    const int nb = leaf ? 0 : 4;
    for (int v = 0; v < sc.nv; ++v) {
      auto probe = [&](double px, double py, double* gv, double* jx, double* jy) {
        VectorXd x = z4;
        x(0) = px;
        x(1) = py;
        MatrixXd Jx(nb + sc.nv, 4), Ju(nb + sc.nv, 2);
        con.jacobians(x, z2, Jx, Ju);
        if (gv) *gv = con.value(x, z2)(nb + v);
        if (jx) *jx = Jx(nb + v, 0);
        if (jy) *jy = Jx(nb + v, 1);
      };
      double g0, j0x, j0y, g1, j1x, j1y;
      probe(0.0, 0.0, &g0, &j0x, &j0y);
      const double nrm = std::hypot(j0x, j0y);
      const double ox = nrm > 0 ? -j0y / nrm : 1.0, oy = nrm > 0 ? j0x / nrm : 0.0;  // perpendicular step
      probe(ox, oy, &g1, &j1x, &j1y);
      // v = x0 + J0 (r - g0) = x1 + J1 (r - g1)  =>  (J0 - J1) r = x1 - x0 + J0 g0 - J1 g1.
      const double ax = j0x - j1x, ay = j0y - j1y;
      const double bx = ox + j0x * g0 - j1x * g1, by = oy + j0y * g0 - j1y * g1;
      const double den = ax * ax + ay * ay;
      if (!(den > 0)) return bad("distance constraint not recoverable");
      const double r_est = (ax * bx + ay * by) / den;
      double vx = j0x * (r_est - g0), vy = j0y * (r_est - g0);
      double ex, ey, gv;
      if (!ulp_search(vx, [&](double c) { double jx; probe(c, vy, nullptr, &jx, nullptr); return jx == 0.0; }, &ex,
                      1 << 16) ||
          !ulp_search(vy, [&](double c) { double jy; probe(ex, c, nullptr, nullptr, &jy); return jy == 0.0; }, &ey,
                      1 << 16))
        return bad("distance constraint is not ego_constraints'");
      probe(ex, ey, &gv, nullptr, nullptr);
      double rad;
      if (!ulp_search(gv + std::sqrt(1e-6), [&](double c) { return c - std::sqrt(0.0 * 0.0 + 0.0 * 0.0 + 1e-6) == gv; },
                      &rad))
        return bad("distance constraint is not ego_constraints'");
      if (i == 0 && v == 0) sc.radius = rad;
      else if (rad != sc.radius) return bad("safety radius differs");
      sc.veh[(static_cast<size_t>(i) * sc.nv + v) * 2 + 0] = ex;
      sc.veh[(static_cast<size_t>(i) * sc.nv + v) * 2 + 1] = ey;
    }
    if (!leaf && sc.nv == 0 && i == 0) sc.radius = 0.0;
  }
  return sc;
}

}  // namespace detail

/// The drop-in: bmpc::solve(problem, opts, initial_inputs) (solver.hpp:595-596)
/// for any problem of the two families the device solves. Scenario problems
/// (unicycle RK4 + tracking costs + ego constraints, as scenarios.hpp builds
/// them) are recognized by probing their callbacks: dt, the weights, every
/// node's tracking reference, the vehicle predictions, the input limits and
/// the safety radius are recovered bit for bit (each constant searched until
/// the callback reproduces it exactly); unconstrained problems take the
/// affine-quadratic family. Anything else throws std::invalid_argument.
inline SolveResult solve(const BmpcProblem& problem, const SolverOptions& opts = {},
                         const std::vector<VectorXd>* initial_inputs = nullptr, Context* ctx = nullptr) {
  if (!problem.has_constraints()) return solve_affine_quadratic(problem, opts, initial_inputs, ctx);
  const detail::UnicycleScene sc = detail::recover_unicycle(problem);
  if (!sc.why.empty())
    throw std::invalid_argument("bmpc::b200::solve: not a unicycle scenario problem (" + sc.why + ")");
  const TreeTopology& t = problem.tree;
  const detail::FlatTree tree(t);
  std::vector<double> x0(4);
  for (int j = 0; j < 4; ++j) x0[static_cast<size_t>(j)] = problem.initial_state(j);
  bmpc_model_desc m{};
  m.kind = BMPC_MODEL_UNICYCLE;
  m.state_dim = 4;
  m.input_dim = 2;
  m.initial_state = x0.data();
  m.dt = sc.dt;
  for (int c = 0; c < 4; ++c)
    for (int r = 0; r < 4; ++r) {
      m.state_weights[r + 4 * c] = sc.Wx(r, c);
      m.terminal_weights[r + 4 * c] = sc.Wf(r, c);
    }
  for (int c = 0; c < 2; ++c)
    for (int r = 0; r < 2; ++r) m.input_weights[r + 2 * c] = sc.Wu(r, c);
  m.accel_limit = sc.a_max;
  m.yaw_rate_limit = sc.w_max;
  m.safety_radius = sc.radius;
  m.num_vehicles = sc.nv;
  m.reference = sc.ref.data();
  m.vehicle_position = sc.veh.data();
  return detail::run(problem, tree, m, opts, initial_inputs, ctx);
}

}  // namespace bmpc::b200
