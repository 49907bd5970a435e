// C-ABI wrapper around the UNMODIFIED reference solver — TEST INFRASTRUCTURE.
//
// Compiled by oracle/Makefile from the reference headers under
// /root/reference/proj/include (never copied) against oracle/eigen_shim into
// oracle/_ref/libbmpc_ref.so. Used only by tests/ (golden generation and
// pinning the C restatement), and by bench.py's reference / cpu_baseline arm.
// Nothing in the product links it.
//
// Problem families mirror the reference builders:
//   0 intersection  build_intersection_case (scenarios.hpp:296-372)
//   1 latency       build_latency_case      (scenarios.hpp:398-479)
//   2 multistage    cfg2/cfg3 builder composed only of the reference's own
//                   primitives: build_tree (tree.hpp:191), branch_choices
//                   (scenarios.hpp:138), predict_vehicles (:165),
//                   left_turn_reference (:278), ego_constraints (:206),
//                   tracking_cost (problem.hpp:194), unicycle_dynamics (:192).
//   3 lq            testing::random_lq_problem (oracles.hpp:316-365)
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "bmpc/scenarios.hpp"
#include "bmpc/solver.hpp"
#include "bmpc/testing/oracles.hpp"

namespace {

using namespace bmpc;

}  // namespace

extern "C" {

struct RefScenario {
  int family;          // 0 intersection, 1 latency, 2 multistage, 3 lq
  int horizon;
  double total_time;
  double shared_time[2];  // intersection: [0]; latency: T_sh0, T_sh1
  int v1, v2;             // intersection vehicle option counts
  int n_branchings;       // multistage / lq: explicit branchings
  int branch_step[8];
  int branch_arity[8];
  double branch_weight[8][16];  // lq only (multistage is uniform)
  int perturb;                  // 1: perturb initial_state with mt19937_64(perturb_seed)
  unsigned long long perturb_seed;
  int lq_nx, lq_nu;
  unsigned long long lq_seed;
};

struct RefOptions {
  int backward;     // 0 scan_tree_riccati, 1 scan_condensed, 2 sequential_riccati
  int forward;      // 0 linear, 1 nonlinear
  int line_search;  // 0 parallel, 1 sequential
  int scan_order;   // 0 sequential, 1 tree
  int parallel;
  int max_inner_iterations, max_outer_iterations, alpha_levels;
  double armijo_beta, merit_gamma, merit_mu0, merit_mu_init, defect_epsilon;
  double tol_defect, tol_cost, tol_feedforward, tol_constraint;
  double penalty_init, penalty_growth, penalty_max;
  double reg_init, reg_min, reg_growth, reg_decay, reg_max;
};

struct RefReport {
  int status;  // 0 converged, 1 max-iter, 2 error
  int inner_iterations, outer_iterations;
  int n_records;
  double final_cost, final_violation, final_defect_l1;
  double times[6];  // setup, bp1, bp2, forward, line_search, total (s)
  char message[256];
};

struct RefRecord {
  int outer;
  int accepted;
  double cost, cost_al, merit_before, merit_after, model_decrease, defect_l1, violation, alpha, mu,
      max_feedforward, regularization;
};

void ref_default_options(RefOptions* o) {
  const SolverOptions d;
  o->backward = static_cast<int>(d.backward);
  o->forward = static_cast<int>(d.forward);
  o->line_search = static_cast<int>(d.line_search);
  o->scan_order = static_cast<int>(d.scan_order);
  o->parallel = d.parallel ? 1 : 0;
  o->max_inner_iterations = d.max_inner_iterations;
  o->max_outer_iterations = d.max_outer_iterations;
  o->alpha_levels = d.alpha_levels;
  o->armijo_beta = d.armijo_beta;
  o->merit_gamma = d.merit_gamma;
  o->merit_mu0 = d.merit_mu0;
  o->merit_mu_init = d.merit_mu_init;
  o->defect_epsilon = d.defect_epsilon;
  o->tol_defect = d.tol_defect;
  o->tol_cost = d.tol_cost;
  o->tol_feedforward = d.tol_feedforward;
  o->tol_constraint = d.tol_constraint;
  o->penalty_init = d.penalty_init;
  o->penalty_growth = d.penalty_growth;
  o->penalty_max = d.penalty_max;
  o->reg_init = d.reg_init;
  o->reg_min = d.reg_min;
  o->reg_growth = d.reg_growth;
  o->reg_decay = d.reg_decay;
  o->reg_max = d.reg_max;
}

}  // extern "C"

namespace {

SolverOptions to_options(const RefOptions* o) {
  SolverOptions s;
  if (!o) return s;
  s.backward = static_cast<BackwardStrategy>(o->backward);
  s.forward = static_cast<ForwardMode>(o->forward);
  s.line_search = static_cast<LineSearchMode>(o->line_search);
  s.scan_order = static_cast<ScanOrder>(o->scan_order);
  s.parallel = o->parallel != 0;
  s.max_inner_iterations = o->max_inner_iterations;
  s.max_outer_iterations = o->max_outer_iterations;
  s.alpha_levels = o->alpha_levels;
  s.armijo_beta = o->armijo_beta;
  s.merit_gamma = o->merit_gamma;
  s.merit_mu0 = o->merit_mu0;
  s.merit_mu_init = o->merit_mu_init;
  s.defect_epsilon = o->defect_epsilon;
  s.tol_defect = o->tol_defect;
  s.tol_cost = o->tol_cost;
  s.tol_feedforward = o->tol_feedforward;
  s.tol_constraint = o->tol_constraint;
  s.penalty_init = o->penalty_init;
  s.penalty_growth = o->penalty_growth;
  s.penalty_max = o->penalty_max;
  s.reg_init = o->reg_init;
  s.reg_min = o->reg_min;
  s.reg_growth = o->reg_growth;
  s.reg_decay = o->reg_decay;
  s.reg_max = o->reg_max;
  return s;
}

std::vector<TreeBranching> branchings_of(const RefScenario* sc, bool uniform) {
  std::vector<TreeBranching> b;
  for (int i = 0; i < sc->n_branchings; ++i) {
    TreeBranching tb;
    tb.step = sc->branch_step[i];
    tb.arity = sc->branch_arity[i];
    for (int a = 0; a < tb.arity; ++a) {
      tb.weights.push_back(uniform ? 1.0 / tb.arity : sc->branch_weight[i][a]);
    }
    b.push_back(std::move(tb));
  }
  return b;
}

/// cfg2/cfg3 builder: intersection scene, one branching per stage j, at which
/// vehicle (j mod 2) reveals its speed-target option c_j in [0, arity). Each
/// vehicle follows its most recently revealed target (its current speed
/// before the first reveal). Everything else is build_intersection_case.
BmpcProblem build_multistage_case(const ScenarioSpec& spec, const std::vector<TreeBranching>& branchings,
                                  ScenarioArtifacts* artifacts) {
  const TreeTopology tree = build_tree(spec.horizon, branchings);
  const auto choices = detail::branch_choices(tree);
  const auto target_of = [&](size_t vehicle, int node) {
    const auto& ch = choices[static_cast<size_t>(node)];
    double target = spec.vehicles[vehicle].speed;
    for (size_t j = 0; j < ch.size(); ++j) {
      if (j % 2 == vehicle && ch[j] >= 0) target = spec.vehicles[vehicle].target_speeds.at(static_cast<size_t>(ch[j]));
    }
    return target;
  };
  const auto vehicle_states = detail::predict_vehicles(tree, spec, target_of);
  const auto reference = left_turn_reference(spec);

  BmpcProblem problem;
  problem.tree = tree;
  problem.state_dim = unicycle::kStateDim;
  problem.input_dim = unicycle::kInputDim;
  problem.initial_state = spec.ego_start;
  problem.dynamics.resize(static_cast<size_t>(tree.node_count));
  problem.cost.resize(static_cast<size_t>(tree.node_count));
  problem.terminal_cost.resize(static_cast<size_t>(tree.node_count));
  problem.constraint.resize(static_cast<size_t>(tree.node_count));
  const MatrixXd Wx = spec.state_weights.asDiagonal();
  const MatrixXd Wu = spec.input_weights.asDiagonal();
  const MatrixXd Wf = spec.terminal_weights.asDiagonal();
  if (artifacts) {
    artifacts->tree = tree;
    artifacts->reference.resize(static_cast<size_t>(tree.node_count));
    artifacts->vehicle_position.resize(static_cast<size_t>(tree.node_count));
  }
  for (int i = 0; i < tree.node_count; ++i) {
    const int k = tree.time_step[static_cast<size_t>(i)];
    std::vector<Eigen::Vector2d> positions;
    for (const auto& vs : vehicle_states[static_cast<size_t>(i)]) positions.push_back(vs.position);
    if (tree.is_leaf(i)) {
      problem.terminal_cost[static_cast<size_t>(i)] = tracking_terminal_cost(reference[static_cast<size_t>(k)], Wf);
      problem.constraint[static_cast<size_t>(i)] = detail::ego_constraints(spec, positions, false);
    } else {
      problem.dynamics[static_cast<size_t>(i)] = detail::unicycle_dynamics(spec.dt());
      problem.cost[static_cast<size_t>(i)] = tracking_cost(reference[static_cast<size_t>(k)], Wx, Wu);
      problem.constraint[static_cast<size_t>(i)] = detail::ego_constraints(spec, positions, true);
    }
    if (artifacts) {
      artifacts->reference[static_cast<size_t>(i)] = reference[static_cast<size_t>(k)];
      artifacts->vehicle_position[static_cast<size_t>(i)] = positions;
    }
  }
  return problem;
}

/// Measured-state perturbation for batched instances (cfg4): U(-0.5,0.5) m in
/// px, py; U(-0.05,0.05) rad in psi; U(-0.5,0.5) m/s in v, drawn in that order
/// from std::mt19937_64(seed).
void perturb_state(VectorXd& x0, unsigned long long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dp(-0.5, 0.5), dpsi(-0.05, 0.05), dv(-0.5, 0.5);
  x0(0) += dp(rng);
  x0(1) += dp(rng);
  x0(2) += dpsi(rng);
  x0(3) += dv(rng);
}

struct Built {
  BmpcProblem problem;
  ScenarioArtifacts art;
  ScenarioSpec spec;
  bool has_artifacts{false};
};

Built build(const RefScenario* sc) {
  Built b;
  switch (sc->family) {
    case 0: {
      b.spec = intersection_spec(sc->horizon, sc->total_time, sc->shared_time[0]);
      b.problem = build_intersection_case(b.spec, sc->v1, sc->v2, &b.art);
      b.has_artifacts = true;
      break;
    }
    case 1: {
      b.spec = latency_spec(sc->shared_time[1], sc->horizon, sc->total_time, sc->shared_time[0]);
      b.problem = build_latency_case(b.spec, &b.art);
      b.has_artifacts = true;
      break;
    }
    case 2: {
      b.spec = intersection_spec(sc->horizon, sc->total_time, 0.1);
      b.problem = build_multistage_case(b.spec, branchings_of(sc, true), &b.art);
      b.has_artifacts = true;
      break;
    }
    case 3: {
      std::mt19937_64 rng(sc->lq_seed);
      const TreeTopology tree = build_tree(sc->horizon, branchings_of(sc, false));
      b.problem = testing::random_lq_problem(rng, tree, sc->lq_nx, sc->lq_nu);
      break;
    }
    default:
      throw std::invalid_argument("unknown scenario family");
  }
  if (sc->perturb) perturb_state(b.problem.initial_state, sc->perturb_seed);
  return b;
}

void fill_report(const SolveResult& res, RefReport* rep, RefRecord* recs, int max_recs) {
  const SolveReport& r = res.report;
  rep->status = static_cast<int>(r.status);
  rep->inner_iterations = r.inner_iterations;
  rep->outer_iterations = r.outer_iterations;
  rep->n_records = static_cast<int>(r.iterations.size());
  rep->final_cost = r.final_cost;
  rep->final_violation = r.final_violation;
  rep->final_defect_l1 = r.final_defect_l1;
  rep->times[0] = r.times.setup_s;
  rep->times[1] = r.times.backward_p1_s;
  rep->times[2] = r.times.backward_p2_s;
  rep->times[3] = r.times.forward_s;
  rep->times[4] = r.times.line_search_s;
  rep->times[5] = r.times.total_s;
  std::snprintf(rep->message, sizeof rep->message, "%s", r.message.c_str());
  if (recs) {
    for (int i = 0; i < rep->n_records && i < max_recs; ++i) {
      const IterationRecord& it = r.iterations[static_cast<size_t>(i)];
      recs[i] = {it.outer,        it.accepted ? 1 : 0, it.cost,        it.cost_al,
                 it.merit_before, it.merit_after,      it.model_decrease, it.defect_l1,
                 it.violation,    it.alpha,            it.mu,           it.max_feedforward,
                 it.regularization};
    }
  }
}

thread_local std::string g_error;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

/// Sizes of a scenario: node count, state/input dims, vehicles, constraint
/// rows at non-leaf / leaf nodes.
int ref_scenario_size(const RefScenario* sc, int* nodes, int* nx, int* nu, int* nv) {
  try {
    const Built b = build(sc);
    *nodes = b.problem.tree.node_count;
    *nx = b.problem.state_dim;
    *nu = b.problem.input_dim;
    *nv = b.has_artifacts && !b.art.vehicle_position.empty()
              ? static_cast<int>(b.art.vehicle_position[0].size())
              : 0;
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

/// Tree arrays (bit-exact build_tree output) and the per-node scenario data.
int ref_scenario_dump(const RefScenario* sc, int* parent, int* time_step, double* weight, int* last_branch_step,
                      double* initial_state, double* reference, double* vehicles, double* dt) {
  try {
    const Built b = build(sc);
    const TreeTopology& t = b.problem.tree;
    for (int i = 0; i < t.node_count; ++i) {
      parent[i] = t.parent[static_cast<size_t>(i)];
      time_step[i] = t.time_step[static_cast<size_t>(i)];
      weight[i] = t.weight[static_cast<size_t>(i)];
    }
    *last_branch_step = t.last_branch_step;
    for (int j = 0; j < b.problem.state_dim; ++j) initial_state[j] = b.problem.initial_state(j);
    if (b.has_artifacts) {
      const size_t nv = b.art.vehicle_position[0].size();
      for (int i = 0; i < t.node_count; ++i) {
        for (int j = 0; j < 4; ++j) reference[4 * i + j] = b.art.reference[static_cast<size_t>(i)](j);
        for (size_t v = 0; v < nv; ++v) {
          vehicles[(i * nv + v) * 2 + 0] = b.art.vehicle_position[static_cast<size_t>(i)][v](0);
          vehicles[(i * nv + v) * 2 + 1] = b.art.vehicle_position[static_cast<size_t>(i)][v](1);
        }
      }
      *dt = b.spec.dt();
    }
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

/// random_lq_problem data, packed per node (column-major blocks):
///   non-leaf: A[nx*nx] B[nx*nu] c[nx] Q[nx*nx] R[nu*nu] M[nu*nx] q[nx] r[nu]
///   leaf:     P[nx*nx] p[nx]
/// `stage` and `leaf` are node_count * record-size arrays.
int ref_lq_dump(const RefScenario* sc, double* x0, double* stage, double* leaf) {
  try {
    std::mt19937_64 rng(sc->lq_seed);
    const TreeTopology tree = build_tree(sc->horizon, branchings_of(sc, false));
    const int nx = sc->lq_nx, nu = sc->lq_nu;
    // Same draw order as random_lq_problem (oracles.hpp:322-341).
    const VectorXd xi = testing::random_vector(rng, nx);
    for (int j = 0; j < nx; ++j) x0[j] = xi(j);
    const int ss = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu;
    const int ls = nx * nx + nx;
    for (int i = 0; i < tree.node_count; ++i) {
      if (tree.is_leaf(i)) {
        const ValueFunction vf = testing::random_terminal(rng, nx);
        double* o = leaf + static_cast<size_t>(i) * ls;
        std::memcpy(o, vf.P.data(), sizeof(double) * nx * nx);
        std::memcpy(o + nx * nx, vf.p.data(), sizeof(double) * nx);
        continue;
      }
      const StageModel s = testing::random_stage(rng, nx, nu);
      double* o = stage + static_cast<size_t>(i) * ss;
      const auto put = [&o](const MatrixXd& m) {
        std::memcpy(o, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
        o += m.size();
      };
      put(s.A), put(s.B), put(s.c), put(s.Q), put(s.R), put(s.M), put(s.q), put(s.r);
    }
    if (sc->perturb) {
      VectorXd v(nx);
      for (int j = 0; j < nx; ++j) v(j) = x0[j];
      perturb_state(v, sc->perturb_seed);
      for (int j = 0; j < nx; ++j) x0[j] = v(j);
    }
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

/// Full reference solve(). x: node_count*nx, u: node_count*nu (leaf rows 0).
int ref_scenario_solve(const RefScenario* sc, const RefOptions* opts, const double* initial_inputs, double* x,
                       double* u, RefReport* rep, RefRecord* recs, int max_recs) {
  try {
    const Built b = build(sc);
    const int n = b.problem.tree.node_count, nx = b.problem.state_dim, nu = b.problem.input_dim;
    std::vector<VectorXd> init;
    if (initial_inputs) {
      init.resize(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) {
        init[static_cast<size_t>(i)] = VectorXd(nu);
        for (int j = 0; j < nu; ++j) init[static_cast<size_t>(i)](j) = initial_inputs[i * nu + j];
      }
    }
    const SolveResult res = solve(b.problem, to_options(opts), initial_inputs ? &init : nullptr);
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < nx; ++j) x[i * nx + j] = res.trajectory.state[static_cast<size_t>(i)](j);
      for (int j = 0; j < nu; ++j)
        u[i * nu + j] = res.trajectory.input[static_cast<size_t>(i)].size() == nu
                            ? res.trajectory.input[static_cast<size_t>(i)](j)
                            : 0.0;
    }
    fill_report(res, rep, recs, max_recs);
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

/// Batched reference throughput: solves `count` instances of the scenario
/// (instance i perturbed with seed base_seed + i when sc->perturb) on
/// `threads` std::threads, each running solve() with parallel=false (the
/// reference's own parallel_sweep pattern, bench.cpp:259-269). Returns the
/// wall seconds and the number of converged instances.
int ref_batch_solve(const RefScenario* sc, const RefOptions* opts, int count, int threads, double* seconds,
                    int* converged, long long* inner_iterations) {
  try {
    std::vector<Built> problems;
    problems.reserve(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
      RefScenario s = *sc;
      s.perturb_seed = sc->perturb_seed + static_cast<unsigned long long>(i);
      problems.push_back(build(&s));
    }
    SolverOptions o = to_options(opts);
    std::atomic<int> next{0}, ok{0};
    std::atomic<long long> inner{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&] {
        for (int i = next++; i < count; i = next++) {
          const SolveResult r = solve(problems[static_cast<size_t>(i)].problem, o);
          if (r.report.status == SolveStatus::converged) ++ok;
          inner += r.report.inner_iterations;
        }
      });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *converged = ok.load();
    *inner_iterations = inner.load();
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

/// Kernel-level reference: backward_pass + linear_rollout + EC on explicit
/// TreeStageModels (riccati.hpp:77-84). stage records as in ref_lq_dump (c
/// ignored), defect: node_count*nx, leaf: node_count*(nx*nx+nx).
/// Outputs: K (node*nu*nx), k (node*nu), P (node*nx*nx), p (node*nx),
/// dx (node*nx), du (node*nu), scalars[0..3] = max_ff, a1, a2, status
/// (0 ok, 1 IndefiniteHessianError, 2 FactorizationError).
int ref_lqr_tree(int horizon, int nb, const int* bstep, const int* barity, const double* bweights, int nx, int nu,
                 const double* stage, const double* defect, const double* leaf, double reg, int strategy,
                 const double* dx0, double* K, double* k, double* P, double* p, double* dx, double* du,
                 double* scalars) {
  try {
    std::vector<TreeBranching> br;
    for (int i = 0; i < nb; ++i) {
      TreeBranching tb;
      tb.step = bstep[i];
      tb.arity = barity[i];
      tb.weights.assign(bweights + 16 * i, bweights + 16 * i + barity[i]);
      br.push_back(tb);
    }
    TreeStageModels m;
    m.topology = build_tree(horizon, br);
    const int n = m.topology.node_count;
    m.stage.resize(static_cast<size_t>(n));
    m.defect.resize(static_cast<size_t>(n));
    m.leaf_cost.resize(static_cast<size_t>(n));
    const int ss = 2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu;
    const int ls = nx * nx + nx;
    for (int i = 0; i < n; ++i) {
      if (i > 0) {
        m.defect[static_cast<size_t>(i)] = VectorXd(nx);
        std::memcpy(m.defect[static_cast<size_t>(i)].data(), defect + i * nx, sizeof(double) * nx);
      }
      if (m.topology.is_leaf(i)) {
        ValueFunction vf{MatrixXd(nx, nx), VectorXd(nx)};
        std::memcpy(vf.P.data(), leaf + static_cast<size_t>(i) * ls, sizeof(double) * nx * nx);
        std::memcpy(vf.p.data(), leaf + static_cast<size_t>(i) * ls + nx * nx, sizeof(double) * nx);
        m.leaf_cost[static_cast<size_t>(i)] = vf;
        continue;
      }
      const double* o = stage + static_cast<size_t>(i) * ss;
      StageModel s;
      const auto get = [&o](MatrixXd& mm, int r, int c) {
        mm = MatrixXd(r, c);
        std::memcpy(mm.data(), o, sizeof(double) * r * c);
        o += r * c;
      };
      MatrixXd cc, qq, rr;
      get(s.A, nx, nx), get(s.B, nx, nu), get(cc, nx, 1), get(s.Q, nx, nx), get(s.R, nu, nu), get(s.M, nu, nx),
          get(qq, nx, 1), get(rr, nu, 1);
      s.c = VectorXd::Zero(nx);
      s.q = qq;
      s.r = rr;
      m.stage[static_cast<size_t>(i)] = s;
    }
    BackwardPassOptions bo;
    bo.strategy = static_cast<BackwardStrategy>(strategy);
    bo.regularization = reg;
    bo.dx0 = VectorXd(nx);
    std::memcpy(bo.dx0.data(), dx0, sizeof(double) * nx);
    BackwardPassResult bp;
    try {
      bp = backward_pass(m, bo);
    } catch (const IndefiniteHessianError&) {
      scalars[3] = 1;
      return 0;
    } catch (const FactorizationError&) {
      scalars[3] = 2;
      return 0;
    }
    const DeltaTrees d = linear_rollout(m, bp.policy, bo.dx0);
    const auto [a1, a2] = expected_change_coefficients(m, d);
    for (int i = 0; i < n; ++i) {
      if (bp.value[static_cast<size_t>(i)].P.size() == nx * nx) {
        std::memcpy(P + i * nx * nx, bp.value[static_cast<size_t>(i)].P.data(), sizeof(double) * nx * nx);
        std::memcpy(p + i * nx, bp.value[static_cast<size_t>(i)].p.data(), sizeof(double) * nx);
      }
      std::memcpy(dx + i * nx, d.dx[static_cast<size_t>(i)].data(), sizeof(double) * nx);
      if (!m.topology.is_leaf(i)) {
        std::memcpy(K + i * nu * nx, bp.policy[static_cast<size_t>(i)].K.data(), sizeof(double) * nu * nx);
        std::memcpy(k + i * nu, bp.policy[static_cast<size_t>(i)].k.data(), sizeof(double) * nu);
        std::memcpy(du + i * nu, d.du[static_cast<size_t>(i)].data(), sizeof(double) * nu);
      }
    }
    scalars[0] = bp.max_feedforward;
    scalars[1] = a1;
    scalars[2] = a2;
    scalars[3] = 0;
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

}  // extern "C"
