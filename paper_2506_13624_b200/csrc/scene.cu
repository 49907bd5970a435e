// Device-side scenario generation: the per-node data a scene spec implies
// (scenarios.hpp:61-113 branch choices + vehicle predictions, :201-214 the
// left-turn reference, :416-441 the latency references), written straight
// into a batch's model buffers, so a receding-horizon caller that gets a new
// scene every control step (ego state, surrounding vehicles) uploads the
// ~0.6 KB specs instead of every node's reference and predictions.
//
// One thread per instance walks the tree in BFS order (every child after its
// parent); the arithmetic is the builders' (host.cpp build_scenario), with the
// device's sin / cos / sincos (last-ulp differences to glibc are possible).
#include <cuda_runtime.h>

#include "kernels.h"
#include "model.cuh"

namespace bmpc_b200 {

__global__ void scene_kernel(int family, int count, const SceneSpec* __restrict__ specs, int shared_spec,
                             SceneTree tr, int v2_count, double* __restrict__ model_data, size_t node_data_doubles,
                             size_t veh_offset, double* __restrict__ speed_scratch, double* __restrict__ x0_out,
                             size_t x0_stride) {
  const int inst = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst >= count) return;
  const SceneSpec& s = specs[shared_spec ? 0 : inst];
  const int n = tr.n, nv = s.n_vehicles, nb = tr.nb;
  double* ref = model_data + static_cast<size_t>(inst) * node_data_doubles;
  double* veh = ref + veh_offset;
  double* spd = speed_scratch + static_cast<size_t>(inst) * n * kMaxVehicles;
  const double dt = s.total_time / s.horizon;
  for (int j = 0; j < 4; ++j) x0_out[static_cast<size_t>(inst) * x0_stride + j] = s.ego_start[j];
  // ---- vehicle predictions (predict_vehicles, scenarios.hpp:87-113)
  for (int v = 0; v < nv; ++v) {
    veh[v * 2 + 0] = s.vehicles[v].position[0];
    veh[v * 2 + 1] = s.vehicles[v].position[1];
    spd[v] = s.vehicles[v].speed;
  }
  auto choice = [&](int node, int b) { return tr.choices[static_cast<size_t>(node) * nb + b]; };
  auto target_of = [&](int v, int node) -> double {
    const SceneVehicle& sv = s.vehicles[v];
    if (family == kSceneIntersection) {
      const int c = nb > 0 ? choice(node, 0) : -1;
      if (c < 0) return sv.speed;
      const int option = v == 0 ? c / v2_count : c % v2_count;
      return sv.target_speeds[option];
    }
    if (family == kSceneLatency) {
      const int c = choice(node, 0);
      return c < 0 ? sv.speed : sv.target_speeds[c];
    }
    double target = sv.speed;  // multistage: stage j reveals vehicle j mod 2's target
    for (int j = 0; j < nb; ++j) {
      const int c = choice(node, j);
      if (j % 2 == v && c >= 0) target = sv.target_speeds[c];
    }
    return target;
  };
  for (int i = 0; i < n; ++i) {
    const int c0 = tr.first_child[i], nc = tr.child_count[i];
    for (int ch = c0; ch < c0 + nc; ++ch) {
      for (int v = 0; v < nv; ++v) {
        const SceneVehicle& sv = s.vehicles[v];
        const size_t cur = static_cast<size_t>(i) * nv + v, nxt = static_cast<size_t>(ch) * nv + v;
        const double target = target_of(v, ch);
        const double step = dt * spd[cur];
        veh[nxt * 2 + 0] = veh[cur * 2 + 0] + step * cos(sv.heading);
        veh[nxt * 2 + 1] = veh[cur * 2 + 1] + step * sin(sv.heading);
        spd[nxt] = spd[cur] + dt * (target - spd[cur]) / s.prediction_tau;
      }
    }
  }
  // ---- tracking references
  if (family == kSceneLatency) {  // build_latency_case (scenarios.hpp:416-441)
    for (int j = 0; j < 4; ++j) ref[j] = s.ego_start[j];
    for (int i = 0; i < n; ++i) {
      const int c0 = tr.first_child[i], nc = tr.child_count[i];
      for (int ch = c0; ch < c0 + nc; ++ch) {
        double r[4] = {ref[i * 4 + 0], ref[i * 4 + 1], ref[i * 4 + 2], ref[i * 4 + 3]};
        const bool lead_brakes = choice(ch, 0) == 1;
        const int decision = choice(ch, 1);
        double decel = 0.0;
        if (lead_brakes && decision == 0) decel = s.continue_deceleration;
        if (lead_brakes && decision == 1) decel = s.backup_deceleration;
        const double v_ref = fmax(0.0, r[3] - decel * dt);
        r[0] += dt * 0.5 * (r[3] + v_ref);
        r[3] = v_ref;
        for (int j = 0; j < 4; ++j) ref[ch * 4 + j] = r[j];
      }
    }
  } else {  // left_turn_reference (scenarios.hpp:201-214), shared by every node of a step
    double x[4] = {s.ego_start[0], s.ego_start[1], s.ego_start[2], s.ego_start[3]};
    const double psi_end = s.ego_start[2] + M_PI / 2.0;
    const double turn_radius = s.ego_start[3] / s.reference_turn_rate;
    const double turn_start_y = -turn_radius;
    for (int k = 0; k <= s.horizon; ++k) {
      for (int i = tr.step_begin[k]; i < tr.step_begin[k + 1]; ++i)
        for (int j = 0; j < 4; ++j) ref[i * 4 + j] = x[j];
      double omega = 0.0;
      if (x[1] >= turn_start_y && x[2] < psi_end) omega = s.reference_turn_rate;
      const double u[2] = {0.0, omega};
      double xn[4];
      unicycle_step(x, u, dt, xn);
      for (int j = 0; j < 4; ++j) x[j] = xn[j];
    }
  }
}

cudaError_t launch_scene(int family, int count, const SceneSpec* d_specs, int shared_spec, const SceneTree& tree,
                         int v2_count, double* model_data, size_t node_data_doubles, size_t veh_offset,
                         double* speed_scratch, double* x0_out, size_t x0_stride, cudaStream_t stream) {
  const int threads = 128;
  scene_kernel<<<(count + threads - 1) / threads, threads, 0, stream>>>(family, count, d_specs, shared_spec, tree,
                                                                       v2_count, model_data, node_data_doubles,
                                                                       veh_offset, speed_scratch, x0_out, x0_stride);
  return cudaGetLastError();
}

}  // namespace bmpc_b200
