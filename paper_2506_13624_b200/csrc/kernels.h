// Host-visible launch interface of the device code. Plain C++ types only, so
// host.cpp compiles with the host compiler. Definitions live in
// kernels_impl.cuh and are explicitly instantiated per (nx, nu) in inst_*.cu.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

#include "bmpc_b200.h"

namespace bmpc_b200 {

struct Topo;
struct ModelParams;
struct Work;
struct DevOptions;
struct DevResume;

// Per-node / per-slot strides (doubles) of the device layouts for (nx, nu).
struct Strides {
  int stage;   // StageLayout::stride
  int bwd;     // BwdLayout::stride
  int fwd;     // FwdLayout::stride
  int policy;  // PolicyLayout::stride
  int value;   // ValueLayout::stride
  int stage_A, stage_B, stage_Q, stage_R, stage_M, stage_q, stage_r;
  int policy_K, policy_k, value_P, value_p;
};

template <int NX, int NU>
struct LqrLaunch {
  static Strides strides();
  static cudaError_t lqr_tree(bool grid, const Topo* d_topo, const Work* d_work, double reg, double* d_scalars,
                              double* red, int blocks, int threads, cudaStream_t stream, int seq_max, int condensed);
  // Batched scan-element primitives (one thread per element): op 0
  // init_bwd_element of packed [A B c Q R M q r] records, op 1 combine_bwd,
  // op 2 combine_fwd; elements unpadded (BwdLayout / FwdLayout ::size).
  static cudaError_t elements(int op, int count, const double* a, const double* b, double reg, double* out,
                              cudaStream_t stream);
  static int grid_blocks(int threads);
};

// One thread block of T threads per instance, >= MB blocks resident per SM
// (registers/thread <= 65536 / (T * MB)).
template <int NX, int NU, int T, int MB>
struct CtaVariant {
  static cudaError_t launch(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work, const DevOptions& opts,
                            int count, bool seq_only, cudaStream_t stream);
  static int regs(bool seq_only);
};

template <int NX, int NU>
struct SolveLaunch {
  // All blocks on one instance (cooperative launch); `red` holds
  // 2 * blocks * kRedSlotsHost doubles.
  static cudaError_t solve_grid(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                const DevOptions& opts, double* red, int blocks, int threads, cudaStream_t stream);
  static int grid_blocks(int threads);
  // Kernels with an optional path compiled in (DevOptions::nonlinear_ls: the
  // single-shooting line search; DevOptions::condensed: the condensed shared
  // segment), so the default kernels keep their register allocation.
  static cudaError_t solve_cta_special(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                       const DevOptions& opts, int count, bool seq_only, cudaStream_t stream);
  static cudaError_t solve_grid_special(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                        const DevOptions& opts, double* red, int blocks, int threads,
                                        cudaStream_t stream);
};

// Dispatch over the compiled dimension sets (dispatch.cu).
bool solve_dims_supported(int nx, int nu);
bool lqr_dims_supported(int nx, int nu);
Strides strides_for(int nx, int nu);
// Launch-shape variants of the per-instance kernel compiled for (nx, nu).
bool cta_variant_supported(int nx, int nu, int threads, int min_blocks);
cudaError_t launch_solve_cta(int nx, int nu, const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                             const DevOptions& opts, int count, int threads, int min_blocks, bool seq_only,
                             cudaStream_t stream);
cudaError_t launch_solve_grid(int nx, int nu, const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                              const DevOptions& opts, double* red, int blocks, int threads, cudaStream_t stream);
int solve_grid_blocks(int nx, int nu, int threads);
int solve_cta_regs(int nx, int nu, int threads, int min_blocks, bool seq_only);
cudaError_t launch_lqr_tree(int nx, int nu, bool grid, const Topo* d_topo, const Work* d_work, double reg,
                            double* d_scalars, double* red, int blocks, int threads, cudaStream_t stream, int seq_max,
                            int condensed);
cudaError_t launch_lqr_elements(int nx, int nu, int op, int count, const double* a, const double* b, double reg,
                                double* out, cudaStream_t stream);
int lqr_grid_blocks(int nx, int nu, int threads);

size_t sizeof_topo();
size_t sizeof_model_params();
size_t sizeof_work();
size_t sizeof_dev_result();
size_t sizeof_dev_record();

constexpr int kRedSlotsHost = 64;

// scene.cu: device-side scenario generation (bmpc_batch_set_scenes).
using SceneSpec = bmpc_scenario_spec;
using SceneVehicle = bmpc_vehicle;
constexpr int kSceneIntersection = BMPC_SCENARIO_INTERSECTION, kSceneLatency = BMPC_SCENARIO_LATENCY,
              kSceneMultistage = BMPC_SCENARIO_MULTISTAGE;
struct SceneTree {
  int n, nb;               // nodes, branchings
  const int* first_child;  // [n]
  const int* child_count;  // [n]
  const int* step_begin;   // [horizon + 2]
  const int* choices;      // [n][nb] child index taken at each branching on the node's path, -1 before it
};
cudaError_t launch_scene(int family, int count, const SceneSpec* d_specs, int shared_spec, const SceneTree& tree,
                         int v2_count, double* model_data, size_t node_data_doubles, size_t veh_offset,
                         double* speed_scratch, double* x0_out, size_t x0_stride, cudaStream_t stream);

// util.cu
cudaError_t launch_order_by_key(const DevResume* d_resume, int count, int* d_order, cudaStream_t stream);
cudaError_t launch_pack_results(const Work* d_works, int count, int n, int nx, int nu, double* dst,
                                cudaStream_t stream);
double measure_fp64_peak_tflops(cudaStream_t stream);
double grid_sync_us(int blocks, int threads, int iters, cudaStream_t stream);
double ric_step_cycles(int steps, int prefetch, cudaStream_t stream, double* stages = nullptr);
void latency_probe(double* cyc3, cudaStream_t stream);

}  // namespace bmpc_b200
