// Host-visible launch interface of the device code. Plain C++ types only, so
// host.cpp compiles with the host compiler. Definitions live in
// kernels_impl.cuh and are explicitly instantiated per (nx, nu) in inst_*.cu.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

namespace bmpc_b200 {

struct Topo;
struct ModelParams;
struct Work;
struct DevOptions;

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
                              double* red, int blocks, int threads, cudaStream_t stream);
  static int grid_blocks(int threads);
};

template <int NX, int NU>
struct SolveLaunch {
  // One thread block per instance.
  static cudaError_t solve_cta(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                               const DevOptions& opts, int count, int threads, cudaStream_t stream);
  // All blocks on one instance (cooperative launch); `red` holds
  // 2 * blocks * kRedSlotsHost doubles.
  static cudaError_t solve_grid(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                const DevOptions& opts, double* red, int blocks, int threads, cudaStream_t stream);
  static int grid_blocks(int threads);
  static int cta_regs();
};

// Dispatch over the compiled dimension sets (dispatch.cu).
bool solve_dims_supported(int nx, int nu);
bool lqr_dims_supported(int nx, int nu);
Strides strides_for(int nx, int nu);
cudaError_t launch_solve_cta(int nx, int nu, const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                             const DevOptions& opts, int count, int threads, cudaStream_t stream);
cudaError_t launch_solve_grid(int nx, int nu, const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                              const DevOptions& opts, double* red, int blocks, int threads, cudaStream_t stream);
int solve_grid_blocks(int nx, int nu, int threads);
int solve_cta_regs(int nx, int nu);
cudaError_t launch_lqr_tree(int nx, int nu, bool grid, const Topo* d_topo, const Work* d_work, double reg,
                            double* d_scalars, double* red, int blocks, int threads, cudaStream_t stream);
int lqr_grid_blocks(int nx, int nu, int threads);

size_t sizeof_topo();
size_t sizeof_model_params();
size_t sizeof_work();
size_t sizeof_dev_result();
size_t sizeof_dev_record();

constexpr int kRedSlotsHost = 64;

}  // namespace bmpc_b200
