// Host runtime of bmpc_b200: the C ABI (include/bmpc_b200.h), tree building,
// scenario builders, segment planning, device buffers and launches.
//
// Compiled with -ffp-contract=off so the host-side builders reproduce the
// reference builders' floating-point results bit for bit (tree weights,
// references, vehicle predictions).
#include "bmpc_b200.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "kernels.h"
#include "types.h"

using namespace bmpc_b200;

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ tree
// build_tree (tree.hpp:61-128), same validation and same arithmetic.
std::unique_ptr<bmpc_tree, void (*)(bmpc_tree*)> make_tree(int horizon, int nb, const int* steps,
                                                           const int* arities, const double* weights,
                                                           int max_arity) {
  if (horizon < 1) throw std::invalid_argument("build_tree: horizon must be >= 1");
  for (int b = 0; b < nb; ++b) {
    if (steps[b] < 0 || steps[b] >= horizon)
      throw std::invalid_argument("build_tree: branching step " + std::to_string(steps[b]) +
                                  " must lie in [0, horizon)");
    if (b > 0 && steps[b] <= steps[b - 1])
      throw std::invalid_argument("build_tree: branching steps must be strictly increasing");
    if (arities[b] < 2 || arities[b] > max_arity)
      throw std::invalid_argument("build_tree: branching needs arity >= 2 and one weight per child");
    double sum = 0.0;
    for (int a = 0; a < arities[b]; ++a) {
      const double w = weights[b * max_arity + a];
      if (!(w > 0.0)) throw std::invalid_argument("build_tree: branch weights must be positive");
      sum += w;
    }
    if (std::abs(sum - 1.0) > 1e-9)
      throw std::invalid_argument("build_tree: branch weights must sum to 1, got " + std::to_string(sum));
  }
  std::vector<int> parent{-1}, time_step{0};
  std::vector<double> weight{1.0};
  std::vector<int> step_begin(static_cast<size_t>(horizon) + 2, 0);
  std::vector<int> level{0};
  int next = 0;
  for (int k = 0; k < horizon; ++k) {
    step_begin[static_cast<size_t>(k) + 1] = static_cast<int>(parent.size());
    int br = -1;
    if (next < nb && steps[next] == k) br = next++;
    std::vector<int> next_level;
    for (int node : level) {
      const int arity = br >= 0 ? arities[br] : 1;
      for (int a = 0; a < arity; ++a) {
        const int child = static_cast<int>(parent.size());
        parent.push_back(node);
        time_step.push_back(k + 1);
        weight.push_back(weight[static_cast<size_t>(node)] * (br >= 0 ? weights[br * max_arity + a] : 1.0));
        next_level.push_back(child);
      }
    }
    level = std::move(next_level);
  }
  const int n = static_cast<int>(parent.size());
  step_begin[static_cast<size_t>(horizon) + 1] = n;

  auto* t = new bmpc_tree{};
  t->node_count = n;
  t->horizon = horizon;
  t->last_branch_step = nb == 0 ? -1 : steps[nb - 1];
  t->parent = new int[n];
  t->time_step = new int[n];
  t->weight = new double[n];
  t->first_child = new int[n];
  t->child_count = new int[n];
  t->step_begin = new int[horizon + 2];
  std::copy(parent.begin(), parent.end(), t->parent);
  std::copy(time_step.begin(), time_step.end(), t->time_step);
  std::copy(weight.begin(), weight.end(), t->weight);
  std::copy(step_begin.begin(), step_begin.end(), t->step_begin);
  for (int i = 0; i < n; ++i) {
    t->first_child[i] = -1;
    t->child_count[i] = 0;
  }
  for (int i = 1; i < n; ++i) {
    const int p = parent[static_cast<size_t>(i)];
    if (t->first_child[p] < 0) t->first_child[p] = i;
    ++t->child_count[p];
  }
  std::vector<int> leaves;
  for (int i = 0; i < n; ++i)
    if (t->child_count[i] == 0) leaves.push_back(i);
  t->leaf_count = static_cast<int>(leaves.size());
  t->leaves = new int[leaves.size()];
  std::copy(leaves.begin(), leaves.end(), t->leaves);
  return {t, bmpc_tree_free};
}

// --------------------------------------------------------------- scenarios
// ScenarioSpec defaults (scenarios.hpp:25-47).
struct Vehicle {
  double px, py, heading, speed;
  std::vector<double> targets;
};
struct Spec {
  double total_time{10.0};
  std::vector<double> shared_times{0.1};
  int horizon{63};
  double ego[4]{0.0, -20.0, M_PI / 2.0, 5.0};
  std::vector<Vehicle> vehicles;
  double state_w[4]{1.0, 1.0, 0.1, 0.1}, input_w[2]{0.5, 0.5}, terminal_w[4]{1.0, 1.0, 0.1, 0.1};
  double accel_limit{3.0}, yaw_rate_limit{0.5}, safety_radius{3.0}, prediction_tau{1.5};
  double reference_turn_rate{0.4}, backup_deceleration{3.0}, continue_deceleration{2.5};
  double dt() const { return total_time / horizon; }
};

Spec intersection_spec(int horizon, double total_time, double shared_time) {  // scenarios.hpp:178-197
  Spec s;
  s.total_time = total_time;
  s.shared_times = {shared_time};
  s.horizon = horizon;
  s.vehicles = {{-3.5, 30.0, -M_PI / 2.0, 8.0, {8.0, 2.0, 5.0, 3.5}}, {0.0, -10.0, M_PI / 2.0, 5.0, {5.0, 1.0, 3.0, 2.0}}};
  return s;
}

Spec latency_spec(double shared_time_1, int horizon, double total_time, double shared_time_0) {  // :300-314
  Spec s;
  s.total_time = total_time;
  s.shared_times = {shared_time_0, shared_time_1};
  s.horizon = horizon;
  s.ego[0] = 0.0;
  s.ego[1] = 0.0;
  s.ego[2] = 0.0;
  s.ego[3] = 10.0;
  s.vehicles = {{30.0, 0.0, 0.0, 8.0, {8.0, 0.0}}};
  return s;
}

// unicycle::step (unicycle.hpp:36-42) in the reference's operation order.
void host_unicycle_step(const double* x, const double* u, double dt, double* out) {
  auto deriv = [&](const double* y, double* d) {
    d[0] = y[3] * std::cos(y[2]);
    d[1] = y[3] * std::sin(y[2]);
    d[2] = u[1];
    d[3] = u[0];
  };
  double k1[4], k2[4], k3[4], k4[4], t[4];
  deriv(x, k1);
  for (int i = 0; i < 4; ++i) t[i] = x[i] + 0.5 * dt * k1[i];
  deriv(t, k2);
  for (int i = 0; i < 4; ++i) t[i] = x[i] + 0.5 * dt * k2[i];
  deriv(t, k3);
  for (int i = 0; i < 4; ++i) t[i] = x[i] + dt * k3[i];
  deriv(t, k4);
  for (int i = 0; i < 4; ++i) out[i] = x[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
}

// left_turn_reference (scenarios.hpp:201-214).
std::vector<std::array<double, 4>> left_turn_reference(const Spec& spec) {
  std::vector<std::array<double, 4>> ref(static_cast<size_t>(spec.horizon) + 1);
  double x[4] = {spec.ego[0], spec.ego[1], spec.ego[2], spec.ego[3]};
  const double psi_end = spec.ego[2] + M_PI / 2.0;
  const double turn_radius = spec.ego[3] / spec.reference_turn_rate;
  const double turn_start_y = -turn_radius;
  for (int k = 0; k <= spec.horizon; ++k) {
    ref[static_cast<size_t>(k)] = {x[0], x[1], x[2], x[3]};
    double omega = 0.0;
    if (x[1] >= turn_start_y && x[2] < psi_end) omega = spec.reference_turn_rate;
    const double u[2] = {0.0, omega};
    double xn[4];
    host_unicycle_step(x, u, spec.dt(), xn);
    std::copy(xn, xn + 4, x);
  }
  return ref;
}

// branch_choices (scenarios.hpp:61-77).
std::vector<std::vector<int>> branch_choices(const bmpc_tree& t, const std::vector<int>& branch_steps) {
  const size_t nb = branch_steps.size();
  std::vector<std::vector<int>> ch(static_cast<size_t>(t.node_count), std::vector<int>(nb, -1));
  for (int i = 0; i < t.node_count; ++i) {
    for (int c = 0; c < t.child_count[i]; ++c) {
      const int kid = t.first_child[i] + c;
      ch[static_cast<size_t>(kid)] = ch[static_cast<size_t>(i)];
      for (size_t b = 0; b < nb; ++b)
        if (branch_steps[b] == t.time_step[i]) ch[static_cast<size_t>(kid)][b] = c;
    }
  }
  return ch;
}

// predict_vehicles (scenarios.hpp:87-113): positions only.
template <class TargetFn>
std::vector<double> predict_vehicles(const bmpc_tree& t, const Spec& spec, const TargetFn& target_of) {
  const size_t nv = spec.vehicles.size();
  std::vector<double> pos(static_cast<size_t>(t.node_count) * nv * 2), speed(static_cast<size_t>(t.node_count) * nv);
  for (size_t v = 0; v < nv; ++v) {
    pos[v * 2 + 0] = spec.vehicles[v].px;
    pos[v * 2 + 1] = spec.vehicles[v].py;
    speed[v] = spec.vehicles[v].speed;
  }
  const double dt = spec.dt();
  for (int i = 0; i < t.node_count; ++i) {
    for (int c = 0; c < t.child_count[i]; ++c) {
      const int ch = t.first_child[i] + c;
      for (size_t v = 0; v < nv; ++v) {
        const Vehicle& veh = spec.vehicles[v];
        const size_t cur = static_cast<size_t>(i) * nv + v, nxt = static_cast<size_t>(ch) * nv + v;
        const double target = target_of(v, ch);
        const double step = dt * speed[cur];
        pos[nxt * 2 + 0] = pos[cur * 2 + 0] + step * std::cos(veh.heading);
        pos[nxt * 2 + 1] = pos[cur * 2 + 1] + step * std::sin(veh.heading);
        speed[nxt] = speed[cur] + dt * (target - speed[cur]) / spec.prediction_tau;
      }
    }
  }
  return pos;
}

struct ProblemData {
  bmpc_problem_data pub{};
  std::unique_ptr<bmpc_tree, void (*)(bmpc_tree*)> tree{nullptr, bmpc_tree_free};
  std::vector<double> x0, reference, vehicles;
};

void fill_unicycle(ProblemData& pd, const Spec& spec) {
  bmpc_model_desc& m = pd.pub.model;
  m.kind = BMPC_MODEL_UNICYCLE;
  m.state_dim = 4;
  m.input_dim = 2;
  m.dt = spec.dt();
  std::memset(m.state_weights, 0, sizeof m.state_weights);
  std::memset(m.input_weights, 0, sizeof m.input_weights);
  std::memset(m.terminal_weights, 0, sizeof m.terminal_weights);
  for (int i = 0; i < 4; ++i) {
    m.state_weights[i * 5] = spec.state_w[i];
    m.terminal_weights[i * 5] = spec.terminal_w[i];
  }
  for (int i = 0; i < 2; ++i) m.input_weights[i * 3] = spec.input_w[i];
  m.accel_limit = spec.accel_limit;
  m.yaw_rate_limit = spec.yaw_rate_limit;
  m.safety_radius = spec.safety_radius;
  m.num_vehicles = static_cast<int>(spec.vehicles.size());
  pd.x0.assign(spec.ego, spec.ego + 4);
}

// Measured-state perturbation (cfg4): U(-0.5,0.5) px, py; U(-0.05,0.05) psi;
// U(-0.5,0.5) v; std::mt19937_64(seed), drawn in that order.
void perturb(std::vector<double>& x0, unsigned long long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dp(-0.5, 0.5), dpsi(-0.05, 0.05), dv(-0.5, 0.5);
  x0[0] += dp(rng);
  x0[1] += dp(rng);
  x0[2] += dpsi(rng);
  x0[3] += dv(rng);
}

// A caller-provided ScenarioSpec (bmpc_scenario_spec).
Spec spec_from(const bmpc_scenario_spec& c) {
  Spec s;
  s.total_time = c.total_time;
  if (c.n_shared < 1 || c.n_shared > 2) throw std::invalid_argument("scenario spec: 1 or 2 shared times");
  s.shared_times.assign(c.shared_times, c.shared_times + c.n_shared);
  s.horizon = c.horizon;
  std::copy(c.ego_start, c.ego_start + 4, s.ego);
  if (c.n_vehicles < 0 || c.n_vehicles > kMaxVehicles) throw std::invalid_argument("scenario spec: at most 4 vehicles");
  for (int v = 0; v < c.n_vehicles; ++v) {
    const bmpc_vehicle& cv = c.vehicles[v];
    if (cv.n_targets < 0 || cv.n_targets > BMPC_MAX_TARGETS)
      throw std::invalid_argument("scenario spec: at most 8 target speeds per vehicle");
    s.vehicles.push_back({cv.position[0], cv.position[1], cv.heading, cv.speed,
                          std::vector<double>(cv.target_speeds, cv.target_speeds + cv.n_targets)});
  }
  std::copy(c.state_weights, c.state_weights + 4, s.state_w);
  std::copy(c.input_weights, c.input_weights + 2, s.input_w);
  std::copy(c.terminal_weights, c.terminal_weights + 4, s.terminal_w);
  s.accel_limit = c.accel_limit;
  s.yaw_rate_limit = c.yaw_rate_limit;
  s.safety_radius = c.safety_radius;
  s.prediction_tau = c.prediction_tau;
  s.reference_turn_rate = c.reference_turn_rate;
  s.backup_deceleration = c.backup_deceleration;
  s.continue_deceleration = c.continue_deceleration;
  if (!(s.horizon > 0) || !(s.total_time > 0)) throw std::invalid_argument("scenario spec: horizon and total time > 0");
  return s;
}

ProblemData* build_scenario(const bmpc_scenario& sc) {
  auto pd = std::make_unique<ProblemData>();
  Spec spec;
  std::vector<int> steps, arities;
  std::vector<double> weights;  // max_arity 16
  constexpr int kMaxA = 16;
  if (sc.family == BMPC_SCENARIO_INTERSECTION) {
    spec = sc.spec ? spec_from(*sc.spec) : intersection_spec(sc.horizon, sc.total_time, sc.shared_time[0]);
    const int leaves = sc.v1 * sc.v2;
    const bool ok = leaves == 1 || leaves == 2 || leaves == 4 || leaves == 6 || leaves == 9 || leaves == 12;
    if (!ok || sc.v1 < 1 || sc.v2 < 1)
      throw std::invalid_argument("build_intersection_case: leaf count " + std::to_string(leaves) +
                                  " not in {1, 2, 4, 6, 9, 12}");
    if (spec.vehicles.size() != 2 || static_cast<int>(spec.vehicles[0].targets.size()) < sc.v1 ||
        static_cast<int>(spec.vehicles[1].targets.size()) < sc.v2)
      throw std::invalid_argument("build_intersection_case: need 2 vehicles with enough targets");
    const int branch_step = static_cast<int>(std::lround(spec.shared_times.at(0) / spec.dt()));
    if (leaves > 1) {
      if (branch_step < 0 || branch_step >= spec.horizon)
        throw std::invalid_argument("build_intersection_case: shared time outside the horizon");
      steps.push_back(std::max(branch_step, 0));
      arities.push_back(leaves);
      weights.assign(kMaxA, 0.0);
      for (int a = 0; a < leaves; ++a) weights[static_cast<size_t>(a)] = 1.0 / leaves;
    }
  } else if (sc.family == BMPC_SCENARIO_LATENCY) {
    spec = sc.spec ? spec_from(*sc.spec) : latency_spec(sc.shared_time[1], sc.horizon, sc.total_time, sc.shared_time[0]);
    if (spec.shared_times.size() != 2 || !(spec.shared_times[0] < spec.shared_times[1]) ||
        !(spec.shared_times[1] < spec.total_time))
      throw std::invalid_argument("build_latency_case: need T_sh0 < T_sh1 < T");
    if (spec.vehicles.size() != 1 || spec.vehicles[0].targets.size() != 2)
      throw std::invalid_argument("build_latency_case: need one vehicle with 2 targets");
    const int k0 = static_cast<int>(std::lround(spec.shared_times[0] / spec.dt()));
    const int k1 = static_cast<int>(std::lround(spec.shared_times[1] / spec.dt()));
    if (k0 < 0 || k0 >= k1 || k1 >= spec.horizon)
      throw std::invalid_argument("build_latency_case: branch steps must satisfy 0 <= k0 < k1 < N");
    steps = {k0, k1};
    arities = {2, 2};
    weights.assign(2 * kMaxA, 0.0);
    weights[0] = weights[1] = weights[kMaxA] = weights[kMaxA + 1] = 0.5;
  } else if (sc.family == BMPC_SCENARIO_MULTISTAGE) {
    spec = sc.spec ? spec_from(*sc.spec) : intersection_spec(sc.horizon, sc.total_time, 0.1);
    if (sc.n_branchings < 0 || sc.n_branchings > 8) throw std::invalid_argument("multistage: 0..8 branchings");
    if (spec.vehicles.size() != 2) throw std::invalid_argument("multistage: need 2 vehicles");
    weights.assign(static_cast<size_t>(std::max(sc.n_branchings, 1)) * kMaxA, 0.0);
    for (int b = 0; b < sc.n_branchings; ++b) {
      const size_t targets = spec.vehicles[static_cast<size_t>(b % 2)].targets.size();
      if (sc.branch_arity[b] < 2 || static_cast<size_t>(sc.branch_arity[b]) > targets)
        throw std::invalid_argument("multistage: arity must be in [2, " + std::to_string(targets) +
                                    "] (the revealing vehicle's speed targets)");
      steps.push_back(sc.branch_step[b]);
      arities.push_back(sc.branch_arity[b]);
      for (int a = 0; a < sc.branch_arity[b]; ++a)
        weights[static_cast<size_t>(b) * kMaxA + a] = 1.0 / sc.branch_arity[b];
    }
  } else {
    throw std::invalid_argument("unknown scenario family");
  }
  pd->tree = make_tree(spec.horizon, static_cast<int>(steps.size()), steps.data(), arities.data(),
                       weights.empty() ? nullptr : weights.data(), kMaxA);
  const bmpc_tree& t = *pd->tree;
  const auto choices = branch_choices(t, steps);
  std::vector<double> veh;
  std::vector<std::array<double, 4>> ref_nodes(static_cast<size_t>(t.node_count));
  if (sc.family == BMPC_SCENARIO_INTERSECTION) {
    const int v2 = sc.v2;
    const auto target_of = [&](size_t vehicle, int node) {
      const auto& c = choices[static_cast<size_t>(node)];
      const int s = c.empty() ? -1 : c[0];
      if (s < 0) return spec.vehicles[vehicle].speed;
      const int option = vehicle == 0 ? s / v2 : s % v2;
      return spec.vehicles[vehicle].targets[static_cast<size_t>(option)];
    };
    veh = predict_vehicles(t, spec, target_of);
    const auto ref = left_turn_reference(spec);
    for (int i = 0; i < t.node_count; ++i) ref_nodes[static_cast<size_t>(i)] = ref[static_cast<size_t>(t.time_step[i])];
  } else if (sc.family == BMPC_SCENARIO_MULTISTAGE) {
    const auto target_of = [&](size_t vehicle, int node) {
      const auto& c = choices[static_cast<size_t>(node)];
      double target = spec.vehicles[vehicle].speed;
      for (size_t j = 0; j < c.size(); ++j)
        if (j % 2 == vehicle && c[j] >= 0) target = spec.vehicles[vehicle].targets.at(static_cast<size_t>(c[j]));
      return target;
    };
    veh = predict_vehicles(t, spec, target_of);
    const auto ref = left_turn_reference(spec);
    for (int i = 0; i < t.node_count; ++i) ref_nodes[static_cast<size_t>(i)] = ref[static_cast<size_t>(t.time_step[i])];
  } else {  // latency (scenarios.hpp:416-441)
    const auto target_of = [&](size_t, int node) {
      const int s = choices[static_cast<size_t>(node)][0];
      return s < 0 ? spec.vehicles[0].speed : spec.vehicles[0].targets[static_cast<size_t>(s)];
    };
    veh = predict_vehicles(t, spec, target_of);
    const double dt = spec.dt();
    ref_nodes[0] = {spec.ego[0], spec.ego[1], spec.ego[2], spec.ego[3]};
    for (int i = 0; i < t.node_count; ++i) {
      for (int c = 0; c < t.child_count[i]; ++c) {
        const int ch = t.first_child[i] + c;
        std::array<double, 4> r = ref_nodes[static_cast<size_t>(i)];
        const bool lead_brakes = choices[static_cast<size_t>(ch)][0] == 1;
        const int decision = choices[static_cast<size_t>(ch)][1];
        double decel = 0.0;
        if (lead_brakes && decision == 0) decel = spec.continue_deceleration;
        if (lead_brakes && decision == 1) decel = spec.backup_deceleration;
        const double v_ref = std::max(0.0, r[3] - decel * dt);
        r[0] += dt * 0.5 * (r[3] + v_ref);
        r[3] = v_ref;
        ref_nodes[static_cast<size_t>(ch)] = r;
      }
    }
  }
  fill_unicycle(*pd, spec);
  if (sc.perturb) perturb(pd->x0, sc.perturb_seed);
  pd->reference.resize(static_cast<size_t>(t.node_count) * 4);
  for (int i = 0; i < t.node_count; ++i)
    for (int j = 0; j < 4; ++j) pd->reference[static_cast<size_t>(i) * 4 + j] = ref_nodes[static_cast<size_t>(i)][j];
  pd->vehicles = std::move(veh);
  pd->pub.tree = pd->tree.get();
  pd->pub.model.initial_state = pd->x0.data();
  pd->pub.model.reference = pd->reference.data();
  pd->pub.model.vehicle_position = pd->vehicles.data();
  return pd.release();
}

// ------------------------------------------------------------ device mem
struct DevBuf {
  void* p{nullptr};
  size_t bytes{0};
  DevBuf() = default;
  explicit DevBuf(size_t n) : bytes(n) {
    if (n) ck(cudaMalloc(&p, n), "cudaMalloc");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Segment plan (see solver.cuh): host copy + device arrays + device Topo.
struct Plan {
  int n{0}, ndepth{0}, nseg{0}, scratch{0}, max_con{0};
  bool has_constraints{false};
  std::vector<int> depth_begin, depth_len, seg_off, seg_nodes, seg_scratch, seg_stride, node_seg, node_pos, seg_depth;
  DevBuf d_ints, d_weight, d_topo;
  Topo topo{};
};

std::unique_ptr<Plan> make_plan(const bmpc_tree& t, int max_con, bool has_constraints, cudaStream_t s) {
  auto pl = std::make_unique<Plan>();
  const int n = t.node_count;
  pl->n = n;
  pl->max_con = max_con;
  pl->has_constraints = has_constraints;
  // Validate the contiguous-children (BFS) layout the device relies on.
  for (int i = 1; i < n; ++i) {
    const int p = t.parent[i];
    if (p < 0 || p >= i || i < t.first_child[p] || i >= t.first_child[p] + t.child_count[p])
      throw std::invalid_argument("tree: children must be contiguous and indexed after their parent");
  }
  // Segments: heads are the root and every child of a branch node.
  struct Seg {
    int depth, head;
    std::vector<int> nodes;
  };
  std::vector<Seg> segs;
  std::vector<std::pair<int, int>> stack{{0, 0}};  // (head, depth)
  while (!stack.empty()) {
    auto [h, d] = stack.back();
    stack.pop_back();
    Seg sg{d, h, {}};
    int i = h;
    while (true) {
      sg.nodes.push_back(i);
      if (t.child_count[i] == 1) {
        i = t.first_child[i];
        continue;
      }
      for (int c = t.child_count[i] - 1; c >= 0; --c) stack.push_back({t.first_child[i] + c, d + 1});
      break;
    }
    segs.push_back(std::move(sg));
  }
  std::stable_sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) {
    return a.depth != b.depth ? a.depth < b.depth : a.head < b.head;
  });
  pl->nseg = static_cast<int>(segs.size());
  pl->ndepth = segs.back().depth + 1;
  pl->depth_begin.assign(static_cast<size_t>(pl->ndepth) + 1, 0);
  pl->depth_len.assign(static_cast<size_t>(pl->ndepth), 0);
  pl->node_seg.assign(static_cast<size_t>(n), -1);
  pl->node_pos.assign(static_cast<size_t>(n), -1);
  pl->seg_off.push_back(0);
  int scratch = 0;
  for (int s = 0; s < pl->nseg; ++s) {
    const Seg& sg = segs[static_cast<size_t>(s)];
    const int L = static_cast<int>(sg.nodes.size());
    if (pl->depth_len[static_cast<size_t>(sg.depth)] == 0) pl->depth_len[static_cast<size_t>(sg.depth)] = L;
    if (pl->depth_len[static_cast<size_t>(sg.depth)] != L)
      throw std::invalid_argument("tree: segments at one branching depth must have equal length (balanced tree)");
    pl->depth_begin[static_cast<size_t>(sg.depth) + 1] = s + 1;
    for (int k = 0; k < L; ++k) {
      pl->node_seg[static_cast<size_t>(sg.nodes[static_cast<size_t>(k)])] = s;
      pl->node_pos[static_cast<size_t>(sg.nodes[static_cast<size_t>(k)])] = k;
      pl->seg_nodes.push_back(sg.nodes[static_cast<size_t>(k)]);
    }
    pl->seg_off.push_back(static_cast<int>(pl->seg_nodes.size()));
    pl->seg_scratch.push_back(scratch);
    // BFS order keeps a chain at a fixed offset within equal-size levels, so
    // consecutive nodes differ by a constant stride (build_tree, tree.hpp:96-115).
    int stride = L >= 2 ? sg.nodes[1] - sg.nodes[0] : 1;
    for (int k = 1; k < L && stride; ++k)
      if (sg.nodes[static_cast<size_t>(k)] - sg.nodes[static_cast<size_t>(k) - 1] != stride) stride = 0;
    pl->seg_stride.push_back(stride);
    pl->seg_depth.push_back(sg.depth);
    // Scan levels n_0 = L, n_{l+1} = ceil(n_l/2): total <= 2L + (#levels).
    scratch += 2 * L + 32;
  }
  for (int d = 1; d <= pl->ndepth; ++d)
    pl->depth_begin[static_cast<size_t>(d)] = std::max(pl->depth_begin[static_cast<size_t>(d)],
                                                       pl->depth_begin[static_cast<size_t>(d) - 1]);
  pl->scratch = scratch;

  // One int buffer for all index arrays.
  std::vector<int> ints;
  auto put = [&ints](const int* p, size_t k) {
    const size_t off = ints.size();
    ints.insert(ints.end(), p, p + k);
    return off;
  };
  const size_t o_parent = put(t.parent, n), o_fc = put(t.first_child, n), o_nc = put(t.child_count, n);
  const size_t o_db = put(pl->depth_begin.data(), pl->depth_begin.size());
  const size_t o_dl = put(pl->depth_len.data(), pl->depth_len.size());
  const size_t o_so = put(pl->seg_off.data(), pl->seg_off.size());
  const size_t o_sn = put(pl->seg_nodes.data(), pl->seg_nodes.size());
  const size_t o_ss = put(pl->seg_scratch.data(), pl->seg_scratch.size());
  const size_t o_st = put(pl->seg_stride.data(), pl->seg_stride.size());
  const size_t o_ns = put(pl->node_seg.data(), pl->node_seg.size());
  const size_t o_np = put(pl->node_pos.data(), pl->node_pos.size());
  const size_t o_sd = put(pl->seg_depth.data(), pl->seg_depth.size());
  pl->d_ints = DevBuf(ints.size() * sizeof(int));
  ck(cudaMemcpyAsync(pl->d_ints.p, ints.data(), ints.size() * sizeof(int), cudaMemcpyHostToDevice, s), "plan");
  pl->d_weight = DevBuf(static_cast<size_t>(n) * sizeof(double));
  ck(cudaMemcpyAsync(pl->d_weight.p, t.weight, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s),
     "plan");
  const int* base = pl->d_ints.as<int>();
  Topo& tp = pl->topo;
  tp.n = n;
  tp.parent = base + o_parent;
  tp.weight = pl->d_weight.as<double>();
  tp.first_child = base + o_fc;
  tp.nchild = base + o_nc;
  tp.ndepth = pl->ndepth;
  tp.depth_begin = base + o_db;
  tp.depth_len = base + o_dl;
  tp.seg_off = base + o_so;
  tp.seg_nodes = base + o_sn;
  tp.seg_scratch = base + o_ss;
  tp.seg_stride = base + o_st;
  tp.node_seg = base + o_ns;
  tp.node_pos = base + o_np;
  tp.seg_depth = base + o_sd;
  tp.has_constraints = has_constraints ? 1 : 0;
  tp.max_con = std::max(max_con, 1);
  // Shared segment (steps <= N_b) and boundary (the heads of the deepest
  // segments, step N_b + 1) for the condensed strategy: BFS numbering makes
  // them the index ranges [0, m) and [m, m + nb).
  tp.n_shared = 0;
  tp.n_bound = 0;
  if (pl->ndepth >= 2) {
    int m = 0;
    for (int s2 = 0; s2 < pl->depth_begin[static_cast<size_t>(pl->ndepth) - 1]; ++s2)
      m += pl->seg_off[static_cast<size_t>(s2) + 1] - pl->seg_off[static_cast<size_t>(s2)];
    const int nb = pl->nseg - pl->depth_begin[static_cast<size_t>(pl->ndepth) - 1];
    bool ok = true;
    for (int s2 = 0; s2 < pl->nseg && ok; ++s2) {
      const bool shared = pl->seg_depth[static_cast<size_t>(s2)] < pl->ndepth - 1;
      for (int k = pl->seg_off[static_cast<size_t>(s2)]; k < pl->seg_off[static_cast<size_t>(s2) + 1]; ++k) {
        const int i = pl->seg_nodes[static_cast<size_t>(k)];
        const bool head = k == pl->seg_off[static_cast<size_t>(s2)];
        if (shared ? i >= m : (head ? (i < m || i >= m + nb) : i < m + nb)) ok = false;
      }
    }
    if (ok) {
      tp.n_shared = m;
      tp.n_bound = nb;
    }
  }
  pl->d_topo = DevBuf(sizeof(Topo));
  ck(cudaMemcpyAsync(pl->d_topo.p, &tp, sizeof(Topo), cudaMemcpyHostToDevice, s), "plan");
  ck(cudaStreamSynchronize(s), "plan sync");
  return pl;
}

DevOptions to_dev(const bmpc_options& o) {
  DevOptions d{};
  d.max_inner_iterations = o.max_inner_iterations;
  d.max_outer_iterations = o.max_outer_iterations;
  d.alpha_levels = o.alpha_levels;
  d.armijo_beta = o.armijo_beta;
  d.merit_gamma = o.merit_gamma;
  d.merit_mu0 = o.merit_mu0;
  d.merit_mu_init = o.merit_mu_init;
  d.defect_epsilon = o.defect_epsilon;
  d.tol_defect = o.tol_defect;
  d.tol_cost = o.tol_cost;
  d.tol_feedforward = o.tol_feedforward;
  d.tol_constraint = o.tol_constraint;
  d.penalty_init = o.penalty_init;
  d.penalty_growth = o.penalty_growth;
  d.penalty_max = o.penalty_max;
  d.reg_init = o.reg_init;
  d.reg_min = o.reg_min;
  d.reg_growth = o.reg_growth;
  d.reg_decay = o.reg_decay;
  d.reg_max = o.reg_max;
  return d;
}

// Column-major n x n with exact zeros off the diagonal.
bool is_diag(const double* w, int n) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (i != j && w[i + n * j] != 0.0) return false;
  return true;
}

void fill_report(const DevResult& r, bmpc_report* out) {
  out->status = r.status;
  out->error_code = r.error_code;
  out->error_node = r.error_node;
  out->inner_iterations = r.inner_iterations;
  out->outer_iterations = r.outer_iterations;
  out->n_records = r.n_records;
  out->final_cost = r.final_cost;
  out->final_violation = r.final_violation;
  out->final_defect_l1 = r.final_defect_l1;
  for (int k = 0; k < 6; ++k) out->times[k] = r.times[k];
  out->final_penalty = r.final_penalty;
  out->final_mu = r.final_mu;
  out->final_reg = r.final_reg;
  out->alpha_evals = r.alpha_evals;
  const char* msg = "";
  char buf[160];
  switch (r.error_code) {
    case kErrRegCap: msg = "regularization exceeded its cap"; break;
    case kErrFactorization: msg = "combine_bwd: singular (I + C P) at regularization cap"; break;
    case kErrLineSearch: msg = "line search failed at maximum regularization"; break;
    case kErrLinearizeNonfinite:  // the reference's three linearize messages (solver.hpp:102-145)
      std::snprintf(buf, sizeof buf, "linearize: non-finite expansion at node %d", r.error_node);
      msg = buf;
      break;
    case kErrLinearizeTerminal:
      std::snprintf(buf, sizeof buf, "linearize: non-finite terminal expansion at node %d", r.error_node);
      msg = buf;
      break;
    case kErrDefectNonfinite:
      std::snprintf(buf, sizeof buf, "linearize: non-finite defect at node %d", r.error_node);
      msg = buf;
      break;
    case kErrRolloutNonfinite:
      std::snprintf(buf, sizeof buf, "nonlinear_rollout: non-finite state at node %d", r.error_node);
      msg = buf;
      break;
    case kErrAlphaLevels: msg = "alpha_levels must lie in [1, 16]"; break;
    default: break;
  }
  std::snprintf(out->message, sizeof out->message, "%s", msg);
}

}  // namespace

// ================================================================== C ABI
struct bmpc_ctx {
  int seq_max_len{-1};  // segments <= this length use the team Riccati sweep (-1: default)
  int ls_block{-1};     // step sizes per line-search round (-1: default, 0: all levels at once)
  int probe{-1};        // batch schedule: probe passes before ordering (-1: default, 0: one FIFO launch)
  int device{0};
  cudaStream_t stream{nullptr};
  bool own_stream{false};
  long long launches{0};
  int sms{0};
  // Batches alive on this ctx: bmpc_ctx_destroy with live batches only marks
  // the ctx, the last bmpc_batch_destroy frees it (any destruction order is
  // safe, e.g. garbage-collected language bindings at interpreter exit).
  int live_batches{0};
  bool destroy_pending{false};
  int lqr_backward{0};  // bmpc_lqr_tree strategy: 0 tree scan, 1 condensed shared segment
};

static void ctx_free(bmpc_ctx* c) {
  cudaSetDevice(c->device);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// Crossover between the team Riccati sweep and the scan (segment length).
// Measured on B200: the O(L) sweep wins below a few hundred nodes.
static int seq_max_for(const bmpc_ctx* c) {
  if (c && c->seq_max_len >= 0) return c->seq_max_len;
  if (const char* env = std::getenv("BMPC_SEQ_MAX")) return std::atoi(env);
  return 384;
}

// Step sizes evaluated per line-search round. The accepted alpha is the first
// accepted level either way; 2 covers ~98 % of cfg4's passes in one round
// (alpha = 1 is accepted in ~79 % of them).
static int ls_block_for(const bmpc_ctx* c) {
  if (c && c->ls_block >= 0) return c->ls_block;
  if (const char* env = std::getenv("BMPC_LS_BLOCK")) return std::atoi(env);
  return 2;
}

// Batch schedule. Pass counts of perturbed instances are heavy-tailed (cfg4:
// mean 85, max 856), so a FIFO launch ends with a tail of long solves that
// started late. When the batch exceeds one wave, a probe launch runs every
// instance for `probe` passes and suspends it (bit-identical resume), the
// instances are ordered by their last constraint violation (the best cheap
// predictor of a long AL run measured on cfg4), and the main launch resumes
// them longest-expected first.
static int probe_for(const bmpc_ctx* c) {
  if (c && c->probe >= 0) return c->probe;
  if (const char* env = std::getenv("BMPC_PROBE")) return std::atoi(env);
  return 10;
}

// Device-resident instances sharing one plan.
struct bmpc_batch {
  bmpc_ctx* ctx{nullptr};
  std::unique_ptr<Plan> plan;
  int count{0}, nx{0}, nu{0}, kind{0}, nv{0}, max_records{0};
  size_t node_data_doubles{0};  // per instance: reference+vehicles or lq stage+leaf
  Strides st{};
  DevBuf model_data, x0, state, records, results, mps, works, red, prof, resume, order;
  std::vector<ModelParams> h_mps;
  std::vector<Work> h_works;
  size_t per_state_doubles{0};
  int threads{256};       // grid mode block size
  int cta_threads{256};   // per-instance block shape (bmpc_batch_set_launch)
  double* h_stage{nullptr};  // pinned H2D staging (set_models)
  double* h_pack{nullptr};   // pinned D2H staging (results)
  DevBuf d_pack;             // device [x | u] pack buffer
  ~bmpc_batch() {
    if (h_stage) cudaFreeHost(h_stage);
    if (h_pack) cudaFreeHost(h_pack);
    if (h_specs) cudaFreeHost(h_specs);
  }
  int cta_min_blocks{1};
  // Schedule of batches with more instances than SMs (see probe_for):
  // probe launch shape, main-launch pass budget (0: to completion) and the
  // low-latency shape that finishes the survivors.
  int probe_threads{256}, probe_min_blocks{1}, main_budget{0}, fin_threads{256}, fin_min_blocks{1};
  bool grid_mode{false};
  int grid_blocks{0};
  DevBuf cond;  // condensed-strategy scratch, allocated by the first scan_condensed solve
  // Device-side scenario generation (bmpc_batch_set_scenes): tree arrays,
  // branch choices, per-instance spec upload and vehicle-speed scratch.
  DevBuf scene_ints, scene_specs, scene_speed;
  int scene_nb{-1}, tree_horizon{0};
  std::vector<int> branch_steps, branch_arity;
  bmpc_scenario_spec* h_specs{nullptr};  // pinned
  size_t h_specs_cap{0};
};

namespace {

size_t align2(size_t v) { return (v + 1) & ~size_t{1}; }

// Per-instance block shape: env BMPC_CTA="<threads>x<min_blocks>" overrides
// the tuned default.
void default_launch_shape(bmpc_batch* b) {
  auto env_shape = [&](const char* name, int* t, int* m) {
    const char* env = std::getenv(name);
    int et = 0, em = 0;
    if (env && std::sscanf(env, "%dx%d", &et, &em) == 2 && cta_variant_supported(b->nx, b->nu, et, em)) *t = et, *m = em;
  };
  // One instance per SM or fewer: 256 threads each (lowest latency). More:
  // (4,2) batches take the measured cfg4 schedule (tools/shape_sweep.py):
  // 64x4 probe and main launches with a 150-pass budget, survivors finished
  // by 256-thread blocks that run nearly alone. With the compact stage
  // records 64x4 (255 registers, 4 blocks per SM) beats 64x8 (128 registers,
  // 2 KB spills): 155.0 vs 162.7 ms per cfg4 step (64x6: 156.4).
  int t = 256, m = 1;
  if (b->nx == 4 && b->nu == 2 && b->count > std::max(1, b->ctx->sms)) {
    t = 64;
    m = 4;
    b->main_budget = 150;
  }
  env_shape("BMPC_CTA", &t, &m);
  if (!cta_variant_supported(b->nx, b->nu, t, m)) {
    t = 256;
    m = 1;
  }
  b->cta_threads = t;
  b->cta_min_blocks = m;
  b->probe_threads = t;
  b->probe_min_blocks = m;
  env_shape("BMPC_SHAPE_PROBE", &b->probe_threads, &b->probe_min_blocks);
  if (!cta_variant_supported(b->nx, b->nu, b->fin_threads, b->fin_min_blocks)) b->main_budget = 0;
  env_shape("BMPC_SHAPE_FINISH", &b->fin_threads, &b->fin_min_blocks);
  if (const char* env = std::getenv("BMPC_MAIN_BUDGET")) b->main_budget = std::atoi(env);
}

// Lays out every per-instance array; returns doubles per instance.
size_t state_layout(const Plan& pl, int nx, int nu, const Strides& st, size_t off[12]) {
  const size_t n = static_cast<size_t>(pl.n);
  size_t o = 0;
  const size_t sizes[] = {align2(n * nx),                                   // x
                          align2(n * nu),                                   // u
                          align2(n * static_cast<size_t>(pl.topo.max_con)), // eta
                          n * static_cast<size_t>(st.stage),                // stage
                          align2(n * nx),                                   // defect
                          n * static_cast<size_t>(st.policy),               // policy
                          static_cast<size_t>(pl.scratch) * st.bwd,          // bwd
                          static_cast<size_t>(pl.scratch) * st.fwd,          // fwd
                          align2(n * nx),                                   // dx
                          align2(n * nu),                                   // du
                          n * static_cast<size_t>(st.value)};               // value
  for (int k = 0; k < 11; ++k) {
    off[k] = o;
    o += sizes[k];
  }
  off[11] = o;
  return o;
}

int check_model(const bmpc_tree* tree, const bmpc_model_desc* m) {
  if (!tree || !m) return fail(BMPC_ERR_INVALID, "null tree or model");
  if (!solve_dims_supported(m->state_dim, m->input_dim))
    return fail(BMPC_ERR_UNSUPPORTED, "state/input dims (" + std::to_string(m->state_dim) + "," +
                                          std::to_string(m->input_dim) + ") not compiled in");
  if (m->kind == BMPC_MODEL_UNICYCLE) {
    if (m->state_dim != 4 || m->input_dim != 2) return fail(BMPC_ERR_INVALID, "unicycle needs nx=4, nu=2");
    if (m->num_vehicles < 0 || m->num_vehicles > kMaxVehicles)
      return fail(BMPC_ERR_UNSUPPORTED, "num_vehicles must lie in [0, 4]");
    if (!m->reference || (m->num_vehicles > 0 && !m->vehicle_position))
      return fail(BMPC_ERR_INVALID, "unicycle model needs reference and vehicle arrays");
  } else if (m->kind == BMPC_MODEL_AFFINE_QUADRATIC) {
    if (!m->lq_stage || !m->lq_leaf) return fail(BMPC_ERR_INVALID, "affine-quadratic model needs stage/leaf arrays");
  } else {
    return fail(BMPC_ERR_UNSUPPORTED, "unknown model kind");
  }
  if (!m->initial_state) return fail(BMPC_ERR_INVALID, "initial_state is null");
  return BMPC_OK;
}

size_t lq_stage_size(int nx, int nu) { return static_cast<size_t>(2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu); }

size_t node_data_doubles(const bmpc_tree* t, const bmpc_model_desc* m) {
  const size_t n = static_cast<size_t>(t->node_count);
  if (m->kind == BMPC_MODEL_UNICYCLE) return align2(n * 4) + align2(n * static_cast<size_t>(m->num_vehicles) * 2);
  const int nx = m->state_dim, nu = m->input_dim;
  return align2(n * lq_stage_size(nx, nu)) + align2(n * static_cast<size_t>(nx * nx + nx));
}

}  // namespace

extern "C" {

const char* bmpc_last_error(void) { return g_error.c_str(); }
const char* bmpc_version(void) { return "bmpc_b200 0.1 (sm_100a)"; }

int bmpc_tree_build(int horizon, int n_branchings, const int* steps, const int* arities, const double* weights,
                    int max_arity, bmpc_tree** out) {
  try {
    if (!out || (n_branchings > 0 && (!steps || !arities || !weights))) return fail(BMPC_ERR_INVALID, "null argument");
    *out = make_tree(horizon, n_branchings, steps, arities, weights, max_arity).release();
    return BMPC_OK;
  } catch (const std::invalid_argument& e) {
    return fail(BMPC_ERR_INVALID, e.what());
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_INVALID, e.what());
  }
}

void bmpc_tree_free(bmpc_tree* t) {
  if (!t) return;
  delete[] t->parent;
  delete[] t->time_step;
  delete[] t->weight;
  delete[] t->first_child;
  delete[] t->child_count;
  delete[] t->step_begin;
  delete[] t->leaves;
  delete t;
}

int bmpc_scenario_build(const bmpc_scenario* spec, bmpc_problem_data** out) {
  try {
    if (!spec || !out) return fail(BMPC_ERR_INVALID, "null argument");
    ProblemData* pd = build_scenario(*spec);
    *out = &pd->pub;
    return BMPC_OK;
  } catch (const std::out_of_range& e) {
    return fail(BMPC_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_INVALID, e.what());
  }
}

void bmpc_problem_data_free(bmpc_problem_data* data) {
  if (!data) return;
  // pub is the first member of ProblemData.
  delete reinterpret_cast<ProblemData*>(data);
}

void bmpc_options_default(bmpc_options* o) {  // solver.hpp:35-57
  o->max_inner_iterations = 100;
  o->max_outer_iterations = 10;
  o->alpha_levels = 11;
  o->armijo_beta = 1e-4;
  o->merit_gamma = 0.5;
  o->merit_mu0 = 1.0;
  o->merit_mu_init = 1.0;
  o->defect_epsilon = 1e-8;
  o->tol_defect = 1e-8;
  o->tol_cost = 1e-8;
  o->tol_feedforward = 1e-6;
  o->tol_constraint = 1e-4;
  o->penalty_init = 10.0;
  o->penalty_growth = 10.0;
  o->penalty_max = 1e8;
  o->reg_init = 0.0;
  o->reg_min = 1e-6;
  o->reg_growth = 10.0;
  o->reg_decay = 10.0;
  o->reg_max = 1e10;
  o->backward = BMPC_BACKWARD_SCAN_TREE_RICCATI;
  o->forward = BMPC_FORWARD_LINEAR;
  o->line_search = BMPC_LINE_SEARCH_PARALLEL;
}

int bmpc_ctx_create(int device, bmpc_ctx** out) {
  try {
    if (!out) return fail(BMPC_ERR_INVALID, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(BMPC_ERR_CUDA, "no CUDA device available");
    if (device < 0 || device >= n) return fail(BMPC_ERR_INVALID, "device index out of range");
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new bmpc_ctx{};
    c->device = device;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->own_stream = true;
    ck(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device), "attr");
    *out = c;
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

void bmpc_ctx_destroy(bmpc_ctx* c) {
  if (!c) return;
  if (c->live_batches > 0) {
    c->destroy_pending = true;
    return;
  }
  ctx_free(c);
}

int bmpc_ctx_set_seq_max_len(bmpc_ctx* c, int len) {
  if (!c) return fail(BMPC_ERR_INVALID, "null ctx");
  c->seq_max_len = len;
  return BMPC_OK;
}

int bmpc_ctx_set_schedule(bmpc_ctx* c, int probe_passes) {
  if (!c) return fail(BMPC_ERR_INVALID, "null ctx");
  c->probe = probe_passes;
  return BMPC_OK;
}

int bmpc_ctx_set_line_search_block(bmpc_ctx* c, int alphas) {
  if (!c) return fail(BMPC_ERR_INVALID, "null ctx");
  c->ls_block = alphas;
  return BMPC_OK;
}

int bmpc_ctx_set_stream(bmpc_ctx* c, void* stream) {
  if (!c) return fail(BMPC_ERR_INVALID, "null ctx");
  // The replacement stream must belong to the ctx's device, not the current one.
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(BMPC_ERR_CUDA, "cudaSetDevice");
  if (stream) {
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  } else {
    cudaStream_t s = nullptr;
    const cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(BMPC_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    c->stream = s;
    c->own_stream = true;
  }
  return BMPC_OK;
}

int bmpc_ctx_synchronize(bmpc_ctx* c) {
  if (!c) return fail(BMPC_ERR_INVALID, "null ctx");
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  return e == cudaSuccess ? BMPC_OK : fail(BMPC_ERR_CUDA, cudaGetErrorString(e));
}

long long bmpc_ctx_launch_count(const bmpc_ctx* c) { return c ? c->launches : 0; }

int bmpc_batch_create(bmpc_ctx* ctx, const bmpc_tree* tree, int count, const bmpc_model_desc* tmpl, int max_records,
                      bmpc_batch** out) {
  try {
    if (!ctx || !out || count < 1) return fail(BMPC_ERR_INVALID, "bad batch arguments");
    if (const int rc = check_model(tree, tmpl); rc != BMPC_OK) return rc;
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    auto b = std::make_unique<bmpc_batch>();
    b->ctx = ctx;
    b->count = count;
    b->nx = tmpl->state_dim;
    b->nu = tmpl->input_dim;
    b->kind = tmpl->kind;
    b->nv = tmpl->kind == BMPC_MODEL_UNICYCLE ? tmpl->num_vehicles : 0;
    b->max_records = std::max(max_records, 0);
    const bool has_con = tmpl->kind == BMPC_MODEL_UNICYCLE;  // box rows at every non-leaf
    const int max_con = tmpl->kind == BMPC_MODEL_UNICYCLE ? 4 + b->nv : 0;
    b->plan = make_plan(*tree, max_con, has_con, ctx->stream);
    b->st = strides_for(b->nx, b->nu);
    size_t off[12];
    b->per_state_doubles = state_layout(*b->plan, b->nx, b->nu, b->st, off);
    b->node_data_doubles = node_data_doubles(tree, tmpl);
    const size_t C = static_cast<size_t>(count);
    b->model_data = DevBuf(C * b->node_data_doubles * sizeof(double));
    b->x0 = DevBuf(C * align2(static_cast<size_t>(b->nx)) * sizeof(double));
    b->state = DevBuf(C * b->per_state_doubles * sizeof(double));
    b->records = DevBuf(C * static_cast<size_t>(std::max(b->max_records, 1)) * sizeof(DevRecord));
    b->results = DevBuf(C * sizeof(DevResult));
    b->mps = DevBuf(C * sizeof(ModelParams));
    b->works = DevBuf(C * sizeof(Work));
    b->resume = DevBuf(C * sizeof(DevResume));
    b->order = DevBuf(C * sizeof(int));
    // Grid mode for a single large tree: all SMs on one instance.
    // Crossover: env BMPC_GRID_MIN_NODES (default 1024, tools/grid_crossover.py).
    int grid_min = 1024;
    if (const char* env = std::getenv("BMPC_GRID_MIN_NODES")) grid_min = std::atoi(env);
    b->grid_mode = count == 1 && tree->node_count > grid_min;
    if (b->grid_mode) {
      b->grid_blocks = solve_grid_blocks(b->nx, b->nu, b->threads);
      if (b->grid_blocks < 1) return fail(BMPC_ERR_CUDA, "grid solve kernel cannot be made co-resident");
      b->red = DevBuf(2 * static_cast<size_t>(b->grid_blocks) * kRedSlotsHost * sizeof(double));
    }
    default_launch_shape(b.get());
    b->h_mps.resize(C);
    b->h_works.resize(C);
    const size_t n = static_cast<size_t>(tree->node_count);
    for (size_t i = 0; i < C; ++i) {
      ModelParams& mp = b->h_mps[i];
      std::memset(&mp, 0, sizeof mp);
      mp.kind = tmpl->kind;
      double* md = b->model_data.as<double>() + i * b->node_data_doubles;
      if (tmpl->kind == BMPC_MODEL_UNICYCLE) {
        mp.nv = b->nv;
        mp.reference = md;
        mp.vehicles = md + align2(n * 4);
      } else {
        mp.lq_stage = md;
        mp.lq_leaf = md + align2(n * lq_stage_size(b->nx, b->nu));
      }
      Work& w = b->h_works[i];
      double* s = b->state.as<double>() + i * b->per_state_doubles;
      w.x0 = b->x0.as<double>() + i * align2(static_cast<size_t>(b->nx));
      w.x = s + off[0];
      w.u = s + off[1];
      w.eta = s + off[2];
      w.stage = s + off[3];
      w.defect = s + off[4];
      w.policy = s + off[5];
      w.bwd = s + off[6];
      w.fwd = s + off[7];
      w.dx = s + off[8];
      w.du = s + off[9];
      w.value = s + off[10];
      w.records = b->records.as<DevRecord>() + i * static_cast<size_t>(std::max(b->max_records, 1));
      w.max_records = b->max_records;
      w.resume = b->grid_mode ? nullptr : b->resume.as<DevResume>() + i;
      w.result = b->results.as<DevResult>() + i;
      w.prof = nullptr;
    }
    ck(cudaMemcpyAsync(b->works.p, b->h_works.data(), C * sizeof(Work), cudaMemcpyHostToDevice, ctx->stream), "works");
    ++ctx->live_batches;
    *out = b.release();
    return BMPC_OK;
  } catch (const std::invalid_argument& e) {
    return fail(BMPC_ERR_INVALID, e.what());
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

void bmpc_batch_destroy(bmpc_batch* b) {
  if (!b) return;
  bmpc_ctx* c = b->ctx;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  delete b;
  if (--c->live_batches == 0 && c->destroy_pending) ctx_free(c);
}

int bmpc_batch_set_models(bmpc_batch* b, const bmpc_model_desc* models, size_t* h2d_bytes) {
  try {
    if (!b || !models) return fail(BMPC_ERR_INVALID, "null argument");
    ck(cudaSetDevice(b->ctx->device), "cudaSetDevice");
    const size_t n = static_cast<size_t>(b->plan->n);
    const size_t C = static_cast<size_t>(b->count);
    const size_t x0s = align2(static_cast<size_t>(b->nx));
    cudaStream_t s = b->ctx->stream;
    // Gather every instance's per-node arrays into one pinned staging buffer
    // laid out exactly like the device buffer, then ONE host-to-device copy.
    ck(cudaStreamSynchronize(s), "staging reuse");
    if (!b->h_stage) ck(cudaMallocHost(&b->h_stage, (C * b->node_data_doubles + C * x0s) * sizeof(double)), "pinned");
    double* hs = b->h_stage;
    double* hx0 = hs + C * b->node_data_doubles;
    for (size_t i = 0; i < C; ++i) {
      const bmpc_model_desc& m = models[i];
      if (m.kind != b->kind || m.state_dim != b->nx || m.input_dim != b->nu ||
          (b->kind == BMPC_MODEL_UNICYCLE && m.num_vehicles != b->nv))
        return fail(BMPC_ERR_INVALID, "model " + std::to_string(i) + " does not match the batch template");
    }
    const bool dense_env = std::getenv("BMPC_DENSE_MODEL") != nullptr;
    // Gather split over a few host threads for large batches (cfg4: 67 MB).
    auto gather = [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        const bmpc_model_desc& m = models[i];
        ModelParams& mp = b->h_mps[i];
        double* md = hs + i * b->node_data_doubles;
        if (b->kind == BMPC_MODEL_UNICYCLE) {
          mp.dt = m.dt;
          std::memcpy(mp.Wx, m.state_weights, sizeof mp.Wx);
          std::memcpy(mp.Wu, m.input_weights, sizeof mp.Wu);
          std::memcpy(mp.Wf, m.terminal_weights, sizeof mp.Wf);
          mp.a_max = m.accel_limit;
          mp.w_max = m.yaw_rate_limit;
          mp.radius = m.safety_radius;
          // BMPC_DENSE_MODEL=1 forces the dense expansion (tests compare both bitwise).
          mp.w_diag = is_diag(mp.Wx, 4) && is_diag(mp.Wu, 2) && is_diag(mp.Wf, 4) && !dense_env;
          std::memcpy(md, m.reference, n * 4 * sizeof(double));
          if (b->nv > 0) std::memcpy(md + align2(n * 4), m.vehicle_position, n * static_cast<size_t>(b->nv) * 2 * sizeof(double));
        } else {
          std::memcpy(md, m.lq_stage, n * lq_stage_size(b->nx, b->nu) * sizeof(double));
          std::memcpy(md + align2(n * lq_stage_size(b->nx, b->nu)), m.lq_leaf,
                      n * static_cast<size_t>(b->nx * b->nx + b->nx) * sizeof(double));
        }
        std::memcpy(hx0 + i * x0s, m.initial_state, static_cast<size_t>(b->nx) * sizeof(double));
      }
    };
    const size_t bytes_data = C * b->node_data_doubles * sizeof(double);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = bytes_data < (size_t{4} << 20) ? 1 : std::min<size_t>(std::min<size_t>(hw, 8), C);
    if (nt <= 1) {
      gather(0, C);
    } else {
      std::vector<std::thread> pool;
      for (size_t k = 1; k < nt; ++k) pool.emplace_back(gather, k * C / nt, (k + 1) * C / nt);
      gather(0, C / nt);
      for (auto& th : pool) th.join();
    }
    ck(cudaMemcpyAsync(b->model_data.p, hs, bytes_data, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(b->x0.p, hx0, C * x0s * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(b->mps.p, b->h_mps.data(), b->h_mps.size() * sizeof(ModelParams), cudaMemcpyHostToDevice, s),
       "h2d");
    if (h2d_bytes) *h2d_bytes = bytes_data + C * x0s * sizeof(double) + b->h_mps.size() * sizeof(ModelParams);
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_set_scenes(bmpc_batch* b, int family, const bmpc_scenario_spec* specs, int n_specs, int v1, int v2,
                          size_t* h2d_bytes) {
  try {
    if (!b || !specs || (n_specs != 1 && n_specs != b->count)) return fail(BMPC_ERR_INVALID, "bad arguments");
    if (b->kind != BMPC_MODEL_UNICYCLE) return fail(BMPC_ERR_INVALID, "scenes need a unicycle batch");
    if (family != BMPC_SCENARIO_INTERSECTION && family != BMPC_SCENARIO_LATENCY && family != BMPC_SCENARIO_MULTISTAGE)
      return fail(BMPC_ERR_INVALID, "unknown scenario family");
    ck(cudaSetDevice(b->ctx->device), "cudaSetDevice");
    cudaStream_t s = b->ctx->stream;
    const Plan& pl = *b->plan;
    const int n = pl.n;
    // The tree the batch was created with: its horizon, branch steps and arities.
    if (b->scene_nb < 0) {
      // Rebuild the host tree arrays from the plan (BFS: children contiguous).
      std::vector<int> ts(static_cast<size_t>(n), 0), fc(static_cast<size_t>(n), -1), cc(static_cast<size_t>(n), 0);
      std::vector<int> par(static_cast<size_t>(n), -1);
      ck(cudaMemcpy(par.data(), pl.topo.parent, n * sizeof(int), cudaMemcpyDeviceToHost), "d2h");
      ck(cudaMemcpy(fc.data(), pl.topo.first_child, n * sizeof(int), cudaMemcpyDeviceToHost), "d2h");
      ck(cudaMemcpy(cc.data(), pl.topo.nchild, n * sizeof(int), cudaMemcpyDeviceToHost), "d2h");
      for (int i = 1; i < n; ++i) ts[static_cast<size_t>(i)] = ts[static_cast<size_t>(par[static_cast<size_t>(i)])] + 1;
      const int horizon = n ? ts[static_cast<size_t>(n) - 1] : 0;
      std::vector<int> sb(static_cast<size_t>(horizon) + 2, 0);
      for (int i = 0; i < n; ++i) sb[static_cast<size_t>(ts[static_cast<size_t>(i)]) + 1] = i + 1;
      for (int k = 1; k <= horizon + 1; ++k) sb[static_cast<size_t>(k)] = std::max(sb[static_cast<size_t>(k)], sb[static_cast<size_t>(k) - 1]);
      b->branch_steps.clear();
      b->branch_arity.clear();
      for (int i = 0; i < n; ++i)
        if (cc[static_cast<size_t>(i)] > 1 &&
            (b->branch_steps.empty() || b->branch_steps.back() != ts[static_cast<size_t>(i)])) {
          b->branch_steps.push_back(ts[static_cast<size_t>(i)]);
          b->branch_arity.push_back(cc[static_cast<size_t>(i)]);
        }
      b->tree_horizon = horizon;
      const int nb = static_cast<int>(b->branch_steps.size());
      bmpc_tree t{};
      t.node_count = n;
      t.time_step = ts.data();
      t.first_child = fc.data();
      t.child_count = cc.data();
      const auto ch = branch_choices(t, b->branch_steps);
      std::vector<int> ints;
      ints.insert(ints.end(), sb.begin(), sb.end());
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < nb; ++k) ints.push_back(ch[static_cast<size_t>(i)][static_cast<size_t>(k)]);
      b->scene_ints = DevBuf(std::max<size_t>(ints.size(), 1) * sizeof(int));
      ck(cudaMemcpy(b->scene_ints.p, ints.data(), ints.size() * sizeof(int), cudaMemcpyHostToDevice), "h2d");
      b->scene_nb = nb;
      b->scene_speed = DevBuf(static_cast<size_t>(b->count) * n * kMaxVehicles * sizeof(double));
    }
    const int nb = b->scene_nb;
    // Every spec must give the batch's tree: same horizon and branch steps (the builders' rounding).
    for (int i = 0; i < n_specs; ++i) {
      const bmpc_scenario_spec& sp = specs[i];
      if (sp.horizon != b->tree_horizon || sp.n_vehicles != b->nv)
        return fail(BMPC_ERR_INVALID, "scene " + std::to_string(i) + ": horizon / vehicle count differ from the batch");
      if (sp.n_vehicles < 0 || sp.n_vehicles > kMaxVehicles || sp.n_shared < 1 || sp.n_shared > 2 || !(sp.total_time > 0))
        return fail(BMPC_ERR_INVALID, "scene " + std::to_string(i) + ": invalid spec");
      for (int v = 0; v < sp.n_vehicles; ++v)
        if (sp.vehicles[v].n_targets < 0 || sp.vehicles[v].n_targets > BMPC_MAX_TARGETS)
          return fail(BMPC_ERR_INVALID, "scene " + std::to_string(i) + ": invalid target count");
      const double dt = sp.total_time / sp.horizon;
      std::vector<int> steps;
      if (family == BMPC_SCENARIO_INTERSECTION) {
        if (sp.n_vehicles != 2 || sp.vehicles[0].n_targets < v1 || sp.vehicles[1].n_targets < v2 || v1 < 1 || v2 < 1)
          return fail(BMPC_ERR_INVALID, "build_intersection_case: need 2 vehicles with enough targets");
        if (v1 * v2 > 1) steps.push_back(static_cast<int>(std::lround(sp.shared_times[0] / dt)));
        if ((v1 * v2 > 1) != (nb == 1) || (nb == 1 && b->branch_arity[0] != v1 * v2))
          return fail(BMPC_ERR_INVALID, "scene " + std::to_string(i) + ": v1 * v2 differs from the batch tree's arity");
      } else if (family == BMPC_SCENARIO_LATENCY) {
        if (sp.n_shared != 2 || sp.n_vehicles != 1 || sp.vehicles[0].n_targets != 2)
          return fail(BMPC_ERR_INVALID, "build_latency_case: need one vehicle with 2 targets and T_sh0 < T_sh1 < T");
        steps = {static_cast<int>(std::lround(sp.shared_times[0] / dt)),
                 static_cast<int>(std::lround(sp.shared_times[1] / dt))};
      } else {
        if (sp.n_vehicles != 2) return fail(BMPC_ERR_INVALID, "multistage: need 2 vehicles");
        steps = b->branch_steps;  // the batch tree's stages; stage j reveals vehicle j mod 2's target
        for (int j = 0; j < nb; ++j)
          if (sp.vehicles[j % 2].n_targets < b->branch_arity[static_cast<size_t>(j)])
            return fail(BMPC_ERR_INVALID, "multistage: a revealing vehicle has fewer targets than the arity");
      }
      if (steps != b->branch_steps)
        return fail(BMPC_ERR_INVALID, "scene " + std::to_string(i) + ": its branch steps differ from the batch's tree");
    }
    // Per-instance model scalars (host copies -> one upload), then the specs.
    for (int i = 0; i < b->count; ++i) {
      const bmpc_scenario_spec& sp = specs[n_specs == 1 ? 0 : i];
      ModelParams& mp = b->h_mps[static_cast<size_t>(i)];
      mp.dt = sp.total_time / sp.horizon;
      std::memset(mp.Wx, 0, sizeof mp.Wx);
      std::memset(mp.Wu, 0, sizeof mp.Wu);
      std::memset(mp.Wf, 0, sizeof mp.Wf);
      for (int j = 0; j < 4; ++j) mp.Wx[5 * j] = sp.state_weights[j], mp.Wf[5 * j] = sp.terminal_weights[j];
      for (int j = 0; j < 2; ++j) mp.Wu[3 * j] = sp.input_weights[j];
      mp.a_max = sp.accel_limit;
      mp.w_max = sp.yaw_rate_limit;
      mp.radius = sp.safety_radius;
      mp.w_diag = std::getenv("BMPC_DENSE_MODEL") ? 0 : 1;
    }
    ck(cudaStreamSynchronize(s), "staging reuse");
    if (b->h_specs_cap < static_cast<size_t>(n_specs)) {
      if (b->h_specs) cudaFreeHost(b->h_specs);
      ck(cudaMallocHost(&b->h_specs, static_cast<size_t>(n_specs) * sizeof(bmpc_scenario_spec)), "pinned");
      b->h_specs_cap = static_cast<size_t>(n_specs);
      b->scene_specs = DevBuf(static_cast<size_t>(n_specs) * sizeof(bmpc_scenario_spec));
    }
    std::memcpy(b->h_specs, specs, static_cast<size_t>(n_specs) * sizeof(bmpc_scenario_spec));
    const size_t spec_bytes = static_cast<size_t>(n_specs) * sizeof(bmpc_scenario_spec);
    ck(cudaMemcpyAsync(b->scene_specs.p, b->h_specs, spec_bytes, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(b->mps.p, b->h_mps.data(), b->h_mps.size() * sizeof(ModelParams), cudaMemcpyHostToDevice, s),
       "h2d");
    SceneTree tr{};
    tr.n = n;
    tr.nb = nb;
    tr.first_child = pl.topo.first_child;
    tr.child_count = pl.topo.nchild;
    tr.step_begin = b->scene_ints.as<int>();
    tr.choices = b->scene_ints.as<int>() + (b->tree_horizon + 2);
    ck(launch_scene(family, b->count, b->scene_specs.as<bmpc_scenario_spec>(), n_specs == 1 ? 1 : 0, tr,
                    std::max(v2, 1), b->model_data.as<double>(), b->node_data_doubles, align2(static_cast<size_t>(n) * 4),
                    b->scene_speed.as<double>(), b->x0.as<double>(), align2(static_cast<size_t>(b->nx)), s),
       "scene");
    ++b->ctx->launches;
    if (h2d_bytes) *h2d_bytes = spec_bytes + b->h_mps.size() * sizeof(ModelParams);
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_scene(bmpc_batch* b, int instance, double* reference, double* vehicles, double* x0) {
  try {
    if (!b || instance < 0 || instance >= b->count || b->kind != BMPC_MODEL_UNICYCLE)
      return fail(BMPC_ERR_INVALID, "bad instance");
    ck(cudaSetDevice(b->ctx->device), "cudaSetDevice");
    ck(cudaStreamSynchronize(b->ctx->stream), "sync");
    const size_t n = static_cast<size_t>(b->plan->n);
    const double* md = b->model_data.as<double>() + static_cast<size_t>(instance) * b->node_data_doubles;
    if (reference) ck(cudaMemcpy(reference, md, n * 4 * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
    if (vehicles && b->nv)
      ck(cudaMemcpy(vehicles, md + align2(n * 4), n * b->nv * 2 * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
    if (x0)
      ck(cudaMemcpy(x0, b->x0.as<double>() + static_cast<size_t>(instance) * align2(static_cast<size_t>(b->nx)),
                    b->nx * sizeof(double), cudaMemcpyDeviceToHost),
         "d2h");
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_set_initial_states(bmpc_batch* b, const double* x0, size_t* h2d_bytes) {
  try {
    if (!b || !x0) return fail(BMPC_ERR_INVALID, "null argument");
    ck(cudaSetDevice(b->ctx->device), "cudaSetDevice");
    const size_t C = static_cast<size_t>(b->count);
    const size_t nx = static_cast<size_t>(b->nx), x0s = align2(nx);
    cudaStream_t s = b->ctx->stream;
    ck(cudaStreamSynchronize(s), "staging reuse");
    if (!b->h_stage) ck(cudaMallocHost(&b->h_stage, (C * b->node_data_doubles + C * x0s) * sizeof(double)), "pinned");
    double* hx0 = b->h_stage + C * b->node_data_doubles;
    for (size_t i = 0; i < C; ++i) std::memcpy(hx0 + i * x0s, x0 + i * nx, nx * sizeof(double));
    ck(cudaMemcpyAsync(b->x0.p, hx0, C * x0s * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
    if (h2d_bytes) *h2d_bytes = C * x0s * sizeof(double);
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_replicate(bmpc_batch* b) {
  try {
    if (!b) return fail(BMPC_ERR_INVALID, "null argument");
    cudaStream_t s = b->ctx->stream;
    for (int i = 1; i < b->count; ++i) {
      b->h_mps[static_cast<size_t>(i)].dt = b->h_mps[0].dt;
      std::memcpy(b->h_mps[static_cast<size_t>(i)].Wx, b->h_mps[0].Wx, sizeof b->h_mps[0].Wx);
      std::memcpy(b->h_mps[static_cast<size_t>(i)].Wu, b->h_mps[0].Wu, sizeof b->h_mps[0].Wu);
      std::memcpy(b->h_mps[static_cast<size_t>(i)].Wf, b->h_mps[0].Wf, sizeof b->h_mps[0].Wf);
      b->h_mps[static_cast<size_t>(i)].a_max = b->h_mps[0].a_max;
      b->h_mps[static_cast<size_t>(i)].w_max = b->h_mps[0].w_max;
      b->h_mps[static_cast<size_t>(i)].radius = b->h_mps[0].radius;
      b->h_mps[static_cast<size_t>(i)].w_diag = b->h_mps[0].w_diag;
      ck(cudaMemcpyAsync(b->model_data.as<double>() + static_cast<size_t>(i) * b->node_data_doubles,
                         b->model_data.as<double>(), b->node_data_doubles * sizeof(double), cudaMemcpyDeviceToDevice,
                         s),
         "d2d");
      ck(cudaMemcpyAsync(b->x0.as<double>() + static_cast<size_t>(i) * align2(static_cast<size_t>(b->nx)),
                         b->x0.as<double>(), static_cast<size_t>(b->nx) * sizeof(double), cudaMemcpyDeviceToDevice, s),
         "d2d");
    }
    ck(cudaMemcpyAsync(b->mps.p, b->h_mps.data(), b->h_mps.size() * sizeof(ModelParams), cudaMemcpyHostToDevice, s),
       "h2d");
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_set_launch(bmpc_batch* b, int threads, int min_blocks) {
  if (!b) return fail(BMPC_ERR_INVALID, "null argument");
  if (!cta_variant_supported(b->nx, b->nu, threads, min_blocks))
    return fail(BMPC_ERR_UNSUPPORTED, "launch shape " + std::to_string(threads) + "x" + std::to_string(min_blocks) +
                                          " not compiled for these dims");
  b->cta_threads = threads;
  b->cta_min_blocks = min_blocks;
  if (!std::getenv("BMPC_SHAPE_PROBE")) {
    b->probe_threads = threads;
    b->probe_min_blocks = min_blocks;
  }
  return BMPC_OK;
}

// Initial inputs: zeros unless given (solver.hpp:604-609).
static int batch_set_inputs(bmpc_batch* b, const double* initial_inputs) {
  const size_t n = static_cast<size_t>(b->plan->n);
  for (int i = 0; i < b->count; ++i) {
    const Work& w = b->h_works[static_cast<size_t>(i)];
    const size_t bytes = n * static_cast<size_t>(b->nu) * sizeof(double);
    if (initial_inputs) {
      ck(cudaMemcpyAsync(w.u, initial_inputs + static_cast<size_t>(i) * n * b->nu, bytes, cudaMemcpyHostToDevice,
                         b->ctx->stream),
         "inputs");
    } else {
      ck(cudaMemsetAsync(w.u, 0, bytes, b->ctx->stream), "inputs");
    }
  }
  return BMPC_OK;
}

// Every segment short enough for the team sweep: launch the sweep-only kernel.
// Sweep or scan per depth level (Solver::seq_depth): short segments, or many
// long ones at one depth (the scan's work grows with them; tools/exp_seq.py).
constexpr int kSeqWideSegs = 64, kSeqWideMax = 1024;
// scan_condensed: largest dense QP (stacked shared inputs) the one-block solve takes.
constexpr size_t kCondMaxInputs = 4096;
static bool seq_depth_host(const Plan& pl, int d, int seq_max) {
  const int L = pl.depth_len[static_cast<size_t>(d)];
  const int ns = pl.depth_begin[static_cast<size_t>(d) + 1] - pl.depth_begin[static_cast<size_t>(d)];
  return seq_max > 0 && (L <= seq_max || (ns >= kSeqWideSegs && L <= kSeqWideMax));
}

// Every depth takes the team sweep: launch the sweep-only kernel.
static bool seq_only(const bmpc_batch* b, int seq_max) {
  for (int d = 0; d < b->plan->ndepth; ++d)
    if (!seq_depth_host(*b->plan, d, seq_max)) return false;
  return true;
}

static int batch_launch(bmpc_batch* b, const bmpc_options* opts, bool zero_inputs) {
  bmpc_options o;
  if (opts)
    o = *opts;
  else
    bmpc_options_default(&o);
  DevOptions d = to_dev(o);
  d.zero_inputs = zero_inputs ? 1 : 0;
  d.seq_max_len = seq_max_for(b->ctx);
  d.seq_wide_segs = kSeqWideSegs;
  d.seq_wide_max = kSeqWideMax;
  d.ls_block = ls_block_for(b->ctx);
  d.fwd_scan_min = std::getenv("BMPC_FWD_SCAN_MIN") ? std::atoi(std::getenv("BMPC_FWD_SCAN_MIN")) : 0;
  // The chunked (time-parallel) backward sweep is compiled only into the
  // kernel-level LQR entry (bmpc_lqr_tree): measured slower than the team
  // sweep in the solve kernels (cfg0 alone, 256 threads: 129 vs 80 us per
  // pass; cfg3-spread on the whole GPU: 147 vs 82 ms).
  d.chunk_bwd = 0;
  // Scanned depths whose elements fit ~2 rounds of the group's teams take the
  // Hillis-Steele scan (one barrier per level); BMPC_BWD_HS=<rounds> (0: off).
  d.bwd_hs = std::getenv("BMPC_BWD_HS") ? std::atoi(std::getenv("BMPC_BWD_HS")) : 2;
  // Segments of >= 64 transitions in the wide non-lean kernels: the parallel
  // forward scan (cfg3's 99/199-step segments gain ~1 %, cfg1's 990-step ones
  // halve; shorter segments walk); BMPC_FWD_BLOCK_SCAN=<min transitions> (0: walk).
  d.fwd_block_scan = std::getenv("BMPC_FWD_BLOCK_SCAN") ? std::atoi(std::getenv("BMPC_FWD_BLOCK_SCAN")) : 64;
  // Strategy enums (solver.hpp:23-26; presets bench.cpp:60-83).
  if (o.backward < 0 || o.backward > 2 || o.forward < 0 || o.forward > 1 || o.line_search < 0 || o.line_search > 1)
    return fail(BMPC_ERR_INVALID, "unknown backward / forward / line_search strategy");
  if (o.backward == BMPC_BACKWARD_SEQUENTIAL_RICCATI) d.seq_max_len = 1 << 30;  // sweep every segment
  if (o.backward == BMPC_BACKWARD_SCAN_CONDENSED && b->plan->topo.n_shared > 0) {
    // Dense QP over the stacked shared inputs (condense_tree): H, a copy for
    // the LU fallback / residual check, h, u, pivots, plus per-node records.
    const Topo& tp = b->plan->topo;
    const size_t n = static_cast<size_t>(tp.n_shared) * b->nu;
    if (n > kCondMaxInputs)
      return fail(BMPC_ERR_UNSUPPORTED, "scan_condensed: shared segment of " + std::to_string(n) +
                                            " inputs exceeds the dense-solve limit " + std::to_string(kCondMaxInputs));
    const size_t rec = (static_cast<size_t>(b->nx) * b->nx + b->nx) * 2 + b->nx + static_cast<size_t>(b->nx) * b->nu;
    const size_t per = static_cast<size_t>(tp.n_shared + tp.n_bound) * ((rec + 1) & ~size_t{1}) + 2 * n * n + 4 * n + 2;
    const size_t need = per * static_cast<size_t>(b->count) * sizeof(double);
    if (b->cond.bytes < need) {
      b->cond = DevBuf(need);
      for (int i = 0; i < b->count; ++i) b->h_works[static_cast<size_t>(i)].cond = b->cond.as<double>() + per * i;
      ck(cudaMemcpyAsync(b->works.p, b->h_works.data(), b->h_works.size() * sizeof(Work), cudaMemcpyHostToDevice,
                         b->ctx->stream),
         "works");
    }
    d.condensed = 1;
  }
  if (o.line_search == BMPC_LINE_SEARCH_SEQUENTIAL) d.ls_block = 1;
  d.nonlinear_ls = o.forward == BMPC_FORWARD_NONLINEAR ? 1 : 0;
  cudaError_t e;
  if (b->grid_mode) {
    e = launch_solve_grid(b->nx, b->nu, b->plan->d_topo.as<Topo>(), b->mps.as<ModelParams>(), b->works.as<Work>(), d,
                          b->red.as<double>(), b->grid_blocks, b->threads, b->ctx->stream);
  } else {
    cudaStream_t s = b->ctx->stream;
    const bool so = seq_only(b, d.seq_max_len);
    auto launch = [&](int threads, int min_blocks, int count, cudaStream_t st) {
      ++b->ctx->launches;
      return launch_solve_cta(b->nx, b->nu, b->plan->d_topo.as<Topo>(), b->mps.as<ModelParams>(),
                              b->works.as<Work>(), d, count, threads, min_blocks, so, st);
    };
    const int pt = b->probe_threads, pm = b->probe_min_blocks, mt = b->cta_threads, mm = b->cta_min_blocks;
    const int ft = b->fin_threads, fm = b->fin_min_blocks, main_budget = b->main_budget;
    e = cudaMemsetAsync(b->resume.p, 0, static_cast<size_t>(b->count) * sizeof(DevResume), s);
    const int probe = probe_for(b->ctx);
    if (e == cudaSuccess && probe > 0 && b->count > std::max(1, b->ctx->sms)) {
      d.pass_budget = probe;
      e = launch(pt, pm, b->count, s);
      if (e == cudaSuccess) {
        ++b->ctx->launches;
        e = launch_order_by_key(b->resume.as<DevResume>(), b->count, b->order.as<int>(), s);
      }
      d.pass_budget = main_budget;
      d.order = b->order.as<int>();
      if (e == cudaSuccess) e = launch(mt, mm, b->count, s);
      if (e == cudaSuccess && main_budget > 0) {
        d.pass_budget = 0;
        e = launch(ft, fm, b->count, s);
      }
    } else if (e == cudaSuccess) {
      e = launch(mt, mm, b->count, s);
    }
  }
  if (e != cudaSuccess) return fail(BMPC_ERR_CUDA, std::string("solve launch: ") + cudaGetErrorString(e));
  if (b->grid_mode) ++b->ctx->launches;
  return BMPC_OK;
}

int bmpc_batch_solve(bmpc_batch* b, const bmpc_options* opts) {
  try {
    if (!b) return fail(BMPC_ERR_INVALID, "null argument");
    ck(cudaSetDevice(b->ctx->device), "cudaSetDevice");
    return batch_launch(b, opts, true);  // zero initial inputs, set on device
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_results(bmpc_batch* b, double* x_out, double* u_out, bmpc_report* reports, size_t* d2h_bytes) {
  try {
    if (!b) return fail(BMPC_ERR_INVALID, "null argument");
    ck(cudaSetDevice(b->ctx->device), "cudaSetDevice");
    cudaStream_t s = b->ctx->stream;
    const size_t n = static_cast<size_t>(b->plan->n);
    const size_t C = static_cast<size_t>(b->count);
    const size_t per = n * static_cast<size_t>(b->nx + b->nu);
    size_t bytes = 0;
    std::vector<DevResult> res(C);
    ck(cudaMemcpyAsync(res.data(), b->results.p, C * sizeof(DevResult), cudaMemcpyDeviceToHost, s), "d2h");
    bytes += C * sizeof(DevResult);
    if (x_out || u_out) {
      // Pack [x | u] of every instance on device, ONE device-to-host copy.
      if (!b->d_pack.p) b->d_pack = DevBuf(C * per * sizeof(double));
      if (!b->h_pack) ck(cudaMallocHost(&b->h_pack, C * per * sizeof(double)), "pinned");
      ck(launch_pack_results(b->works.as<Work>(), b->count, b->plan->n, b->nx, b->nu, b->d_pack.as<double>(), s),
         "pack");
      ++b->ctx->launches;
      ck(cudaMemcpyAsync(b->h_pack, b->d_pack.p, C * per * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
      bytes += C * per * sizeof(double);
    }
    ck(cudaStreamSynchronize(s), "sync");
    if (x_out || u_out) {
      // Unpack [x | u] per instance into the caller's arrays; large batches
      // split over a few host threads (a single core copies ~50 MB, the cfg4
      // step's trajectories, at a fraction of the link rate).
      auto unpack = [&](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; ++i) {
          const double* src = b->h_pack + i * per;
          if (x_out) std::memcpy(x_out + i * n * b->nx, src, n * b->nx * sizeof(double));
          if (u_out) std::memcpy(u_out + i * n * b->nu, src + n * b->nx, n * b->nu * sizeof(double));
        }
      };
      const size_t total_bytes = C * per * sizeof(double);
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      const size_t nt = total_bytes < (size_t{4} << 20) ? 1 : std::min<size_t>(std::min<size_t>(hw, 8), C);
      if (nt <= 1) {
        unpack(0, C);
      } else {
        std::vector<std::thread> pool;
        for (size_t k = 1; k < nt; ++k) pool.emplace_back(unpack, k * C / nt, (k + 1) * C / nt);
        unpack(0, C / nt);
        for (auto& th : pool) th.join();
      }
    }
    if (reports)
      for (size_t i = 0; i < C; ++i) fill_report(res[i], &reports[i]);
    if (d2h_bytes) *d2h_bytes = bytes;
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_device_results(bmpc_batch* b, double** d_x, double** d_u, size_t* bytes_x, size_t* bytes_u) {
  if (!b) return fail(BMPC_ERR_INVALID, "null argument");
  // Per-instance state blocks are strided; expose instance 0 base + stride.
  if (d_x) *d_x = b->h_works[0].x;
  if (d_u) *d_u = b->h_works[0].u;
  if (bytes_x) *bytes_x = b->per_state_doubles * sizeof(double);
  if (bytes_u) *bytes_u = b->per_state_doubles * sizeof(double);
  return BMPC_OK;
}

int bmpc_batch_pack_results(bmpc_batch* b, double* d_dst, size_t* bytes) {
  if (!b || !d_dst) return fail(BMPC_ERR_INVALID, "null argument");
  cudaSetDevice(b->ctx->device);
  const cudaError_t e = launch_pack_results(b->works.as<Work>(), b->count, b->plan->n, b->nx, b->nu, d_dst,
                                            b->ctx->stream);
  if (e != cudaSuccess) return fail(BMPC_ERR_CUDA, cudaGetErrorString(e));
  ++b->ctx->launches;
  if (bytes) *bytes = static_cast<size_t>(b->count) * b->plan->n * (b->nx + b->nu) * sizeof(double);
  return BMPC_OK;
}

// ------------------------------------------------ multi-device batches
struct bmpc_multi {
  std::vector<bmpc_ctx*> ctxs;
  std::vector<bmpc_batch*> shards;  // nullptr for an empty shard
  std::vector<int> begin, cnt;
  int count{0}, n{0}, nx{0}, nu{0};
  ~bmpc_multi() {
    for (bmpc_batch* b : shards)
      if (b) bmpc_batch_destroy(b);
  }
};

int bmpc_shard_range(int count, int n_shards, int g, int* begin, int* n) {
  if (count < 0 || n_shards < 1 || g < 0 || g >= n_shards || !begin || !n) return fail(BMPC_ERR_INVALID, "bad shard");
  const long long b0 = static_cast<long long>(g) * count / n_shards;
  const long long b1 = static_cast<long long>(g + 1) * count / n_shards;
  *begin = static_cast<int>(b0);
  *n = static_cast<int>(b1 - b0);
  return BMPC_OK;
}

int bmpc_multi_create(bmpc_ctx* const* ctxs, int n_ctx, const bmpc_tree* tree, int count,
                      const bmpc_model_desc* tmpl, int max_records, bmpc_multi** out) {
  if (!ctxs || n_ctx < 1 || !tree || !tmpl || !out || count < 1) return fail(BMPC_ERR_INVALID, "bad multi arguments");
  auto m = std::make_unique<bmpc_multi>();
  m->count = count;
  m->n = tree->node_count;
  m->nx = tmpl->state_dim;
  m->nu = tmpl->input_dim;
  for (int g = 0; g < n_ctx; ++g) {
    if (!ctxs[g]) return fail(BMPC_ERR_INVALID, "null ctx");
    int b0 = 0, c = 0;
    bmpc_shard_range(count, n_ctx, g, &b0, &c);
    bmpc_batch* b = nullptr;
    if (c > 0) {
      const int rc = bmpc_batch_create(ctxs[g], tree, c, tmpl, max_records, &b);
      if (rc != BMPC_OK) return rc;
    }
    m->ctxs.push_back(ctxs[g]);
    m->shards.push_back(b);
    m->begin.push_back(b0);
    m->cnt.push_back(c);
  }
  *out = m.release();
  return BMPC_OK;
}

void bmpc_multi_destroy(bmpc_multi* m) { delete m; }

int bmpc_multi_set_models(bmpc_multi* m, const bmpc_model_desc* models, size_t* h2d_bytes) {
  if (!m || !models) return fail(BMPC_ERR_INVALID, "null argument");
  size_t tot = 0;
  for (size_t g = 0; g < m->shards.size(); ++g) {
    if (!m->shards[g]) continue;
    size_t b = 0;
    const int rc = bmpc_batch_set_models(m->shards[g], models + m->begin[g], &b);
    if (rc != BMPC_OK) return rc;
    tot += b;
  }
  if (h2d_bytes) *h2d_bytes = tot;
  return BMPC_OK;
}

int bmpc_multi_set_initial_states(bmpc_multi* m, const double* x0, size_t* h2d_bytes) {
  if (!m || !x0) return fail(BMPC_ERR_INVALID, "null argument");
  size_t tot = 0;
  for (size_t g = 0; g < m->shards.size(); ++g) {
    if (!m->shards[g]) continue;
    size_t b = 0;
    const int rc =
        bmpc_batch_set_initial_states(m->shards[g], x0 + static_cast<size_t>(m->begin[g]) * m->nx, &b);
    if (rc != BMPC_OK) return rc;
    tot += b;
  }
  if (h2d_bytes) *h2d_bytes = tot;
  return BMPC_OK;
}

int bmpc_multi_solve(bmpc_multi* m, const bmpc_options* opts) {
  if (!m) return fail(BMPC_ERR_INVALID, "null argument");
  for (bmpc_batch* b : m->shards) {  // asynchronous: every device runs its shard concurrently
    if (!b) continue;
    const int rc = bmpc_batch_solve(b, opts);
    if (rc != BMPC_OK) return rc;
  }
  return BMPC_OK;
}

int bmpc_multi_gather(bmpc_multi* m, double* d_dst, size_t* bytes) {
  try {
    if (!m || !d_dst) return fail(BMPC_ERR_INVALID, "null argument");
    const int dev0 = m->ctxs[0]->device;
    const size_t per = static_cast<size_t>(m->n) * (m->nx + m->nu);
    for (size_t g = 0; g < m->shards.size(); ++g) {
      bmpc_batch* b = m->shards[g];
      if (!b) continue;
      const int dev = m->ctxs[g]->device;
      double* dst = d_dst + static_cast<size_t>(m->begin[g]) * per;
      ck(cudaSetDevice(dev), "cudaSetDevice");
      int can = dev == dev0 ? 1 : 0;
      if (dev != dev0) {
        ck(cudaDeviceCanAccessPeer(&can, dev, dev0), "peer query");
        if (can) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(dev0, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else if (e != cudaSuccess) can = 0, cudaGetLastError();
        }
      }
      if (can) {  // the pack kernel's stores land in device 0's buffer (NVLink P2P)
        ck(launch_pack_results(b->works.as<Work>(), b->count, b->plan->n, b->nx, b->nu, dst, b->ctx->stream), "pack");
      } else {
        if (!b->d_pack.p) b->d_pack = DevBuf(static_cast<size_t>(b->count) * per * sizeof(double));
        ck(launch_pack_results(b->works.as<Work>(), b->count, b->plan->n, b->nx, b->nu, b->d_pack.as<double>(),
                               b->ctx->stream),
           "pack");
        ck(cudaMemcpyPeerAsync(dst, dev0, b->d_pack.p, dev, static_cast<size_t>(b->count) * per * sizeof(double),
                               b->ctx->stream),
           "peer copy");
      }
      ++b->ctx->launches;
    }
    for (size_t g = 0; g < m->shards.size(); ++g)
      if (m->shards[g]) ck(cudaStreamSynchronize(m->ctxs[g]->stream), "sync");
    if (bytes) *bytes = static_cast<size_t>(m->count) * per * sizeof(double);
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_multi_results(bmpc_multi* m, double* x_out, double* u_out, bmpc_report* reports, size_t* d2h_bytes) {
  if (!m) return fail(BMPC_ERR_INVALID, "null argument");
  size_t tot = 0;
  for (size_t g = 0; g < m->shards.size(); ++g) {
    if (!m->shards[g]) continue;
    const size_t b0 = static_cast<size_t>(m->begin[g]);
    size_t b = 0;
    const int rc = bmpc_batch_results(m->shards[g], x_out ? x_out + b0 * m->n * m->nx : nullptr,
                                      u_out ? u_out + b0 * m->n * m->nu : nullptr, reports ? reports + b0 : nullptr,
                                      &b);
    if (rc != BMPC_OK) return rc;
    tot += b;
  }
  if (d2h_bytes) *d2h_bytes = tot;
  return BMPC_OK;
}

int bmpc_multi_shard(bmpc_multi* m, int g, bmpc_batch** batch, int* begin, int* n) {
  if (!m || g < 0 || g >= static_cast<int>(m->shards.size())) return fail(BMPC_ERR_INVALID, "bad shard");
  if (batch) *batch = m->shards[static_cast<size_t>(g)];
  if (begin) *begin = m->begin[static_cast<size_t>(g)];
  if (n) *n = m->cnt[static_cast<size_t>(g)];
  return BMPC_OK;
}

int bmpc_solve_batch(bmpc_ctx* const* ctxs, int n_ctx, const bmpc_tree* tree, int count,
                     const bmpc_model_desc* models, const bmpc_options* opts, double* x_out, double* u_out,
                     bmpc_report* reports) {
  if (!models) return fail(BMPC_ERR_INVALID, "null models");
  bmpc_multi* m = nullptr;
  int rc = bmpc_multi_create(ctxs, n_ctx, tree, count, &models[0], 0, &m);
  if (rc != BMPC_OK) return rc;
  std::unique_ptr<bmpc_multi> guard(m);
  if ((rc = bmpc_multi_set_models(m, models, nullptr)) != BMPC_OK) return rc;
  if ((rc = bmpc_multi_solve(m, opts)) != BMPC_OK) return rc;
  return bmpc_multi_results(m, x_out, u_out, reports, nullptr);
}

int bmpc_debug_grid_sync_us(bmpc_ctx* ctx, int blocks, int threads, int iters, double* us) {
  if (!ctx || !us) return fail(BMPC_ERR_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  *us = grid_sync_us(blocks, threads, iters, ctx->stream);
  return cudaGetLastError() == cudaSuccess ? BMPC_OK : fail(BMPC_ERR_CUDA, "grid sync benchmark failed");
}

int bmpc_batch_set_profiling(bmpc_batch* b, int on) {
  try {
    if (!b) return fail(BMPC_ERR_INVALID, "null argument");
    cudaSetDevice(b->ctx->device);
    const size_t C = static_cast<size_t>(b->count);
    if (on && !b->prof.p) b->prof = DevBuf(C * kProfSlots * sizeof(double));
    if (on) ck(cudaMemsetAsync(b->prof.p, 0, C * kProfSlots * sizeof(double), b->ctx->stream), "memset");
    for (size_t i = 0; i < C; ++i) b->h_works[i].prof = on ? b->prof.as<double>() + i * kProfSlots : nullptr;
    ck(cudaMemcpyAsync(b->works.p, b->h_works.data(), C * sizeof(Work), cudaMemcpyHostToDevice, b->ctx->stream),
       "works");
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_phase_profile(bmpc_batch* b, int instance, double* out, int n) {
  try {
    if (!b || !out || !b->prof.p || instance < 0 || instance >= b->count) return fail(BMPC_ERR_INVALID, "bad args");
    double tmp[kProfSlots];
    ck(cudaMemcpy(tmp, b->prof.as<double>() + static_cast<size_t>(instance) * kProfSlots, sizeof tmp,
                  cudaMemcpyDeviceToHost),
       "d2h");
    for (int k = 0; k < n && k < kProfSlots; ++k) out[k] = tmp[k];
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_debug_ric_step_cycles(bmpc_ctx* ctx, int steps, int prefetch, double* cycles) {
  if (!ctx || !cycles) return fail(BMPC_ERR_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  *cycles = ric_step_cycles(steps, prefetch, ctx->stream, prefetch >= 2 ? cycles + 1 : nullptr);
  return cudaGetLastError() == cudaSuccess ? BMPC_OK : fail(BMPC_ERR_CUDA, "ric benchmark failed");
}

int bmpc_debug_latency_probe(bmpc_ctx* ctx, double* cycles3) {
  if (!ctx || !cycles3) return fail(BMPC_ERR_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  latency_probe(cycles3, ctx->stream);
  return cudaGetLastError() == cudaSuccess ? BMPC_OK : fail(BMPC_ERR_CUDA, "latency probe failed");
}

int bmpc_fp64_peak_tflops(bmpc_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return fail(BMPC_ERR_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  *tflops = measure_fp64_peak_tflops(ctx->stream);
  return cudaGetLastError() == cudaSuccess ? BMPC_OK : fail(BMPC_ERR_CUDA, "fp64 microbenchmark failed");
}

int bmpc_batch_records(bmpc_batch* b, int instance, bmpc_record* records, int max_records, int* n_records) {
  try {
    if (!b || instance < 0 || instance >= b->count) return fail(BMPC_ERR_INVALID, "bad instance");
    DevResult r;
    ck(cudaMemcpy(&r, b->results.as<DevResult>() + instance, sizeof r, cudaMemcpyDeviceToHost), "d2h");
    const int k = std::min({r.n_records, max_records, b->max_records});
    if (k > 0 && records) {
      static_assert(sizeof(bmpc_record) == sizeof(DevRecord), "record layout");
      ck(cudaMemcpy(records, b->h_works[static_cast<size_t>(instance)].records, static_cast<size_t>(k) * sizeof(DevRecord),
                    cudaMemcpyDeviceToHost),
         "d2h");
    }
    if (n_records) *n_records = r.n_records;
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_batch_info(const bmpc_batch* b, int* threads, int* blocks, int* regs) {
  if (!b) return fail(BMPC_ERR_INVALID, "null argument");
  if (threads) *threads = b->grid_mode ? b->threads : b->cta_threads;
  if (blocks) *blocks = b->grid_mode ? b->grid_blocks : b->count;
  if (regs)
    *regs = b->grid_mode ? 0
                         : solve_cta_regs(b->nx, b->nu, b->cta_threads, b->cta_min_blocks,
                                          seq_only(b, seq_max_for(b->ctx)));
  return BMPC_OK;
}

int bmpc_solve(bmpc_ctx* ctx, const bmpc_tree* tree, const bmpc_model_desc* model, const bmpc_options* opts,
               const double* initial_inputs, double* x_out, double* u_out, bmpc_report* report, bmpc_record* records,
               int max_records) {
  bmpc_batch* b = nullptr;
  int rc = bmpc_batch_create(ctx, tree, 1, model, std::max(max_records, 0), &b);
  if (rc != BMPC_OK) return rc;
  std::unique_ptr<bmpc_batch, void (*)(bmpc_batch*)> guard(b, bmpc_batch_destroy);
  rc = bmpc_batch_set_models(b, model, nullptr);
  if (rc != BMPC_OK) return rc;
  try {
    if (initial_inputs) batch_set_inputs(b, initial_inputs);
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
  rc = batch_launch(b, opts, initial_inputs == nullptr);
  if (rc != BMPC_OK) return rc;
  bmpc_report rep{};
  rc = bmpc_batch_results(b, x_out, u_out, &rep, nullptr);
  if (rc != BMPC_OK) return rc;
  if (report) *report = rep;
  if (records && max_records > 0) {
    int nrec = 0;
    rc = bmpc_batch_records(b, 0, records, max_records, &nrec);
    if (rc != BMPC_OK) return rc;
  }
  if (rep.error_code == kErrRolloutNonfinite) return fail(BMPC_ERR_ROLLOUT, rep.message);
  return BMPC_OK;
}

int bmpc_ctx_set_lqr_strategy(bmpc_ctx* c, int backward) {
  if (!c || (backward != BMPC_BACKWARD_SCAN_TREE_RICCATI && backward != BMPC_BACKWARD_SCAN_CONDENSED))
    return fail(BMPC_ERR_INVALID, "lqr strategy must be scan_tree_riccati or scan_condensed");
  c->lqr_backward = backward;
  return BMPC_OK;
}

int bmpc_lqr_elements(bmpc_ctx* ctx, int op, int nx, int nu, int count, const double* a, const double* b, double reg,
                      double* out) {
  try {
    if (!ctx || !a || !out || count < 0 || op < 0 || op > 2 || (op > 0 && !b)) return fail(BMPC_ERR_INVALID, "bad arguments");
    if (!lqr_dims_supported(nx, nu)) return fail(BMPC_ERR_UNSUPPORTED, "dims not compiled in");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t lq = lq_stage_size(nx, nu), be = 3 * static_cast<size_t>(nx) * nx + 2 * nx,
                 fe = static_cast<size_t>(nx) * nx + nx;
    const size_t in_a = op == 0 ? lq : (op == 1 ? be : fe), in_b = op == 0 ? 0 : in_a, out_e = op == 2 ? fe : be;
    const size_t C = static_cast<size_t>(count);
    DevBuf da(std::max<size_t>(C * in_a, 1) * sizeof(double)), db(std::max<size_t>(C * in_b, 1) * sizeof(double)),
        dout(std::max<size_t>(C * out_e, 1) * sizeof(double));
    cudaStream_t s = ctx->stream;
    ck(cudaMemcpyAsync(da.p, a, C * in_a * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
    if (in_b) ck(cudaMemcpyAsync(db.p, b, C * in_b * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
    ck(launch_lqr_elements(nx, nu, op, count, da.as<double>(), db.as<double>(), reg, dout.as<double>(), s), "launch");
    ++ctx->launches;
    ck(cudaMemcpyAsync(out, dout.p, C * out_e * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    return BMPC_OK;
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

int bmpc_lqr_tree(bmpc_ctx* ctx, const bmpc_tree* tree, int nx, int nu, const double* stage, const double* defect,
                  const double* leaf, double reg, const double* dx0, int grid, double* K, double* k, double* P,
                  double* p, double* dx, double* du, double* scalars) {
  try {
    if (!ctx || !tree || !stage || !defect || !leaf || !dx0 || !scalars) return fail(BMPC_ERR_INVALID, "null argument");
    if (!lqr_dims_supported(nx, nu)) return fail(BMPC_ERR_UNSUPPORTED, "dims not compiled in");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    auto plan = make_plan(*tree, 0, false, s);
    const Strides st = strides_for(nx, nu);
    size_t off[12];
    const size_t per = state_layout(*plan, nx, nu, st, off);
    const size_t n = static_cast<size_t>(tree->node_count);
    // Host-side repack of the TreeStageModels into the device stage records.
    std::vector<double> h(per, 0.0);
    const size_t ss = lq_stage_size(nx, nu), ls = static_cast<size_t>(nx * nx + nx);
    for (size_t i = 0; i < n; ++i) {
      double* rec = h.data() + off[3] + i * st.stage;
      if (tree->child_count[i] == 0) {
        std::memcpy(rec + st.stage_Q, leaf + i * ls, sizeof(double) * nx * nx);
        std::memcpy(rec + st.stage_q, leaf + i * ls + nx * nx, sizeof(double) * nx);
      } else {
        const double* src = stage + i * ss;
        const int oA = 0, oB = nx * nx, oc = oB + nx * nu, oQ = oc + nx, oR = oQ + nx * nx, oM = oR + nu * nu,
                  oq = oM + nu * nx, orr = oq + nx;
        std::memcpy(rec + st.stage_A, src + oA, sizeof(double) * nx * nx);
        std::memcpy(rec + st.stage_B, src + oB, sizeof(double) * nx * nu);
        std::memcpy(rec + st.stage_Q, src + oQ, sizeof(double) * nx * nx);
        std::memcpy(rec + st.stage_R, src + oR, sizeof(double) * nu * nu);
        std::memcpy(rec + st.stage_M, src + oM, sizeof(double) * nu * nx);
        std::memcpy(rec + st.stage_q, src + oq, sizeof(double) * nx);
        std::memcpy(rec + st.stage_r, src + orr, sizeof(double) * nu);
      }
      if (i > 0) std::memcpy(h.data() + off[4] + i * nx, defect + i * nx, sizeof(double) * nx);
    }
    DevBuf d_state(per * sizeof(double)), d_x0(align2(static_cast<size_t>(nx)) * sizeof(double)),
        d_sc(4 * sizeof(double)), d_work(sizeof(Work));
    ck(cudaMemcpyAsync(d_state.p, h.data(), per * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(d_x0.p, dx0, static_cast<size_t>(nx) * sizeof(double), cudaMemcpyHostToDevice, s), "h2d");
    Work w{};
    double* base = d_state.as<double>();
    w.x0 = d_x0.as<double>();
    w.x = base + off[0];  // zeros: the root head perturbation is x0 - x[0] = dx0
    w.u = base + off[1];
    w.eta = base + off[2];
    w.stage = base + off[3];
    w.defect = base + off[4];
    w.policy = base + off[5];
    w.bwd = base + off[6];
    w.fwd = base + off[7];
    w.dx = base + off[8];
    w.du = base + off[9];
    w.value = base + off[10];
    DevBuf red, cond;
    int blocks = 0;
    if (grid) {
      blocks = lqr_grid_blocks(nx, nu, 256);
      red = DevBuf(2 * static_cast<size_t>(std::max(blocks, 1)) * kRedSlotsHost * sizeof(double));
    }
    const int condensed = ctx->lqr_backward == BMPC_BACKWARD_SCAN_CONDENSED && plan->topo.n_shared > 0;
    if (condensed) {  // per-node records + H, H copy, h, u, pivots (see batch_launch)
      const size_t m = static_cast<size_t>(plan->topo.n_shared), nb = static_cast<size_t>(plan->topo.n_bound);
      const size_t ni = m * nu;
      if (ni > kCondMaxInputs) return fail(BMPC_ERR_UNSUPPORTED, "scan_condensed: shared segment too large");
      const size_t rec = (static_cast<size_t>(nx) * nx + nx) * 2 + nx + static_cast<size_t>(nx) * nu;
      cond = DevBuf(((m + nb) * ((rec + 1) & ~size_t{1}) + 2 * ni * ni + 4 * ni + 2) * sizeof(double));
      w.cond = cond.as<double>();
    }
    ck(cudaMemcpyAsync(d_work.p, &w, sizeof w, cudaMemcpyHostToDevice, s), "h2d");
    ck(launch_lqr_tree(nx, nu, grid != 0, plan->d_topo.as<Topo>(), d_work.as<Work>(), reg, d_sc.as<double>(),
                       red.as<double>(), blocks, 256, s, seq_max_for(ctx), condensed),
       "lqr launch");
    ++ctx->launches;
    ck(cudaMemcpyAsync(h.data(), d_state.p, per * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaMemcpyAsync(scalars, d_sc.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    for (size_t i = 0; i < n; ++i) {
      const double* pol = h.data() + off[5] + i * st.policy;
      const double* val = h.data() + off[10] + i * st.value;
      if (K && tree->child_count[i] > 0) std::memcpy(K + i * nu * nx, pol + st.policy_K, sizeof(double) * nu * nx);
      if (k && tree->child_count[i] > 0) std::memcpy(k + i * nu, pol + st.policy_k, sizeof(double) * nu);
      if (P) std::memcpy(P + i * nx * nx, val + st.value_P, sizeof(double) * nx * nx);
      if (p) std::memcpy(p + i * nx, val + st.value_p, sizeof(double) * nx);
      if (dx) std::memcpy(dx + i * nx, h.data() + off[8] + i * nx, sizeof(double) * nx);
      if (du && tree->child_count[i] > 0) std::memcpy(du + i * nu, h.data() + off[9] + i * nu, sizeof(double) * nu);
    }
    return BMPC_OK;
  } catch (const std::invalid_argument& e) {
    return fail(BMPC_ERR_INVALID, e.what());
  } catch (const std::exception& e) {
    return fail(BMPC_ERR_CUDA, e.what());
  }
}

}  // extern "C"
