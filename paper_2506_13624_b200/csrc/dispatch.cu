// Runtime (nx, nu) dispatch onto the explicit instantiations in inst_*.cu.
#include "kernels.h"
#include "solver.cuh"

namespace bmpc_b200 {

// Full solve: unicycle (4,2) and the LQ dims the reference tests use.
#define BMPC_SOLVE_DIMS(X) X(4, 2) X(3, 2) X(2, 1)
// Kernel-level LQR tree: the reference verification grid nx {2,4,8} x
// nu {1,2,4} (verification.hpp:47-48) plus (3,2).
#define BMPC_LQR_DIMS(X) \
  X(2, 1) X(2, 2) X(2, 4) X(3, 2) X(4, 1) X(4, 2) X(4, 4) X(8, 1) X(8, 2) X(8, 4)

extern template struct SolveLaunch<4, 2>;
extern template struct SolveLaunch<3, 2>;
extern template struct SolveLaunch<2, 1>;
#define X(a, b) extern template struct LqrLaunch<a, b>;
BMPC_LQR_DIMS(X)
#undef X

static_assert(kRedSlotsHost == kRedSlots, "reduction slot count mismatch");

bool solve_dims_supported(int nx, int nu) {
#define X(a, b) \
  if (nx == a && nu == b) return true;
  BMPC_SOLVE_DIMS(X)
#undef X
  return false;
}

bool lqr_dims_supported(int nx, int nu) {
#define X(a, b) \
  if (nx == a && nu == b) return true;
  BMPC_LQR_DIMS(X)
#undef X
  return false;
}

Strides strides_for(int nx, int nu) {
#define X(a, b) \
  if (nx == a && nu == b) return LqrLaunch<a, b>::strides();
  BMPC_LQR_DIMS(X)
#undef X
  return Strides{};
}

// Launch-shape variants (threads, min blocks/SM) of the per-instance kernel.
#define BMPC_CTA_VARIANTS(X)                                                                   \
  X(4, 2, 256, 1) X(4, 2, 128, 2) X(4, 2, 64, 4) X(4, 2, 128, 3) X(4, 2, 64, 6) X(4, 2, 128, 4) \
  X(4, 2, 64, 8) X(4, 2, 256, 2) X(4, 2, 512, 1) X(4, 2, 1024, 1) X(4, 2, 256, 3) \
  X(4, 2, 256, 4) X(4, 2, 128, 6) X(4, 2, 128, 8) X(4, 2, 512, 2) X(3, 2, 256, 1) X(3, 2, 64, 4) \
  X(2, 1, 256, 1) X(2, 1, 64, 4)

#define X(a, b, t, m) extern template struct CtaVariant<a, b, t, m>;
BMPC_CTA_VARIANTS(X)
#undef X

bool cta_variant_supported(int nx, int nu, int threads, int min_blocks) {
#define X(a, b, t, m) \
  if (nx == a && nu == b && threads == t && min_blocks == m) return true;
  BMPC_CTA_VARIANTS(X)
#undef X
  return false;
}

cudaError_t launch_solve_cta(int nx, int nu, const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                             const DevOptions& opts, int count, int threads, int min_blocks, bool seq_only,
                             cudaStream_t stream) {
  if (opts.nonlinear_ls || opts.condensed) {  // kernels with an optional path: one shape per (nx, nu)
#define X(a, b)           \
  if (nx == a && nu == b) \
    return SolveLaunch<a, b>::solve_cta_special(d_topo, d_mp, d_work, opts, count, seq_only, stream);
    BMPC_SOLVE_DIMS(X)
#undef X
    return cudaErrorInvalidValue;
  }
#define X(a, b, t, m)                                                 \
  if (nx == a && nu == b && threads == t && min_blocks == m)          \
    return CtaVariant<a, b, t, m>::launch(d_topo, d_mp, d_work, opts, count, seq_only, stream);
  BMPC_CTA_VARIANTS(X)
#undef X
  return cudaErrorInvalidValue;
}

int solve_cta_regs(int nx, int nu, int threads, int min_blocks, bool seq_only) {
#define X(a, b, t, m) \
  if (nx == a && nu == b && threads == t && min_blocks == m) return CtaVariant<a, b, t, m>::regs(seq_only);
  BMPC_CTA_VARIANTS(X)
#undef X
  return 0;
}

cudaError_t launch_solve_grid(int nx, int nu, const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                              const DevOptions& opts, double* red, int blocks, int threads, cudaStream_t stream) {
#define X(a, b)                                                                                              \
  if (nx == a && nu == b)                                                                                    \
    return (opts.nonlinear_ls || opts.condensed)                                                            \
               ? SolveLaunch<a, b>::solve_grid_special(d_topo, d_mp, d_work, opts, red, blocks, threads, stream) \
               : SolveLaunch<a, b>::solve_grid(d_topo, d_mp, d_work, opts, red, blocks, threads, stream);
  BMPC_SOLVE_DIMS(X)
#undef X
  return cudaErrorInvalidValue;
}

int solve_grid_blocks(int nx, int nu, int threads) {
#define X(a, b) \
  if (nx == a && nu == b) return SolveLaunch<a, b>::grid_blocks(threads);
  BMPC_SOLVE_DIMS(X)
#undef X
  return 0;
}

cudaError_t launch_lqr_tree(int nx, int nu, bool grid, const Topo* d_topo, const Work* d_work, double reg,
                            double* d_scalars, double* red, int blocks, int threads, cudaStream_t stream, int seq_max,
                            int condensed) {
#define X(a, b)                                                                                           \
  if (nx == a && nu == b)                                                                                 \
    return LqrLaunch<a, b>::lqr_tree(grid, d_topo, d_work, reg, d_scalars, red, blocks, threads, stream, seq_max, \
                                     condensed);
  BMPC_LQR_DIMS(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_lqr_elements(int nx, int nu, int op, int count, const double* a, const double* b, double reg,
                                double* out, cudaStream_t stream) {
#define X(c, d) \
  if (nx == c && nu == d) return LqrLaunch<c, d>::elements(op, count, a, b, reg, out, stream);
  BMPC_LQR_DIMS(X)
#undef X
  return cudaErrorInvalidValue;
}

int lqr_grid_blocks(int nx, int nu, int threads) {
#define X(a, b) \
  if (nx == a && nu == b) return LqrLaunch<a, b>::grid_blocks(threads);
  BMPC_LQR_DIMS(X)
#undef X
  return 0;
}

size_t sizeof_topo() { return sizeof(Topo); }
size_t sizeof_model_params() { return sizeof(ModelParams); }
size_t sizeof_work() { return sizeof(Work); }
size_t sizeof_dev_result() { return sizeof(DevResult); }
size_t sizeof_dev_record() { return sizeof(DevRecord); }

}  // namespace bmpc_b200
