// Kernel templates and their launchers (sm_100a). One kernel launch per
// solve: the whole iLQR/AL loop is device-resident. Instantiated per (nx, nu)
// in inst_*.cu so the heavy unrolled code compiles in parallel.
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"
#include "solver.cuh"

namespace bmpc_b200 {

static_assert(kRedSlotsHost == kRedSlots, "reduction slot count mismatch");

// Stage the per-instance structs in shared memory (read on every node op).
struct BlockCtx {
  Topo topo;
  ModelParams mp;
  Work work;
};

// THREADS x MINB trade registers for resident instances per SM:
// registers/thread <= 65536 / (THREADS * MINB).
template <int NX, int NU, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) solve_cta_kernel(const Topo* __restrict__ topo,
                                                        const ModelParams* __restrict__ mps,
                                                        const Work* __restrict__ works, DevOptions opts,
                                                        int count) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  const int b = blockIdx.x;
  if (b >= count) return;
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.mp = mps[b];
    ctx.work = works[b];
    red.flag = 0;
  }
  __syncthreads();
  __shared__ TeamSmem<NX> tsm[THREADS / (team_size<NX>() > 0 ? team_size<NX>() : THREADS)];
  Solver<NX, NU, CtaGroup> s(CtaGroup{&red}, ctx.topo, ctx.mp, ctx.work, opts);
  s.tsm = tsm;
  s.solve();
}

template <int NX, int NU>
__global__ void __launch_bounds__(256) solve_grid_kernel(const Topo* __restrict__ topo,
                                                         const ModelParams* __restrict__ mps,
                                                         const Work* __restrict__ works, DevOptions opts,
                                                         double* red_scratch) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.mp = mps[0];
    ctx.work = works[0];
    red.flag = 0;
  }
  __syncthreads();
  __shared__ TeamSmem<NX> tsm[256 / (team_size<NX>() > 0 ? team_size<NX>() : 256)];
  Solver<NX, NU, GridGroup> s(GridGroup{&red, red_scratch, nullptr}, ctx.topo, ctx.mp, ctx.work, opts);
  s.tsm = tsm;
  s.solve();
}

template <int NX, int NU, class G>
__device__ void lqr_tree_body(G g, BlockCtx& ctx, double reg, double* scalars) {
  ModelParams dummy{};
  DevOptions o{};
  __shared__ TeamSmem<NX> tsm[256 / (team_size<NX>() > 0 ? team_size<NX>() : 256)];
  Solver<NX, NU, G> s(g, ctx.topo, dummy, ctx.work, o);
  s.tsm = tsm;
  s.lqr_tree(reg, scalars);
}

template <int NX, int NU>
__global__ void __launch_bounds__(256) lqr_tree_cta_kernel(const Topo* topo, const Work* works, double reg,
                                                           double* scalars) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.work = works[0];
    red.flag = 0;
  }
  __syncthreads();
  lqr_tree_body<NX, NU>(CtaGroup{&red}, ctx, reg, scalars);
}

template <int NX, int NU>
__global__ void __launch_bounds__(256) lqr_tree_grid_kernel(const Topo* topo, const Work* works, double reg,
                                                            double* scalars, double* red_scratch) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.work = works[0];
    red.flag = 0;
  }
  __syncthreads();
  lqr_tree_body<NX, NU>(GridGroup{&red, red_scratch, nullptr}, ctx, reg, scalars);
}


template <class K>
static int max_coresident(K kernel, int threads) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  return sms * per_sm;
}

template <int NX, int NU>
Strides LqrLaunch<NX, NU>::strides() {
  using SL = StageLayout<NX, NU>;
  using PL = PolicyLayout<NX, NU>;
  using VL = ValueLayout<NX>;
  Strides s;
  s.stage = SL::stride;
  s.bwd = BwdLayout<NX>::stride;
  s.fwd = FwdLayout<NX>::stride;
  s.policy = PL::stride;
  s.value = VL::stride;
  s.stage_A = SL::A;
  s.stage_B = SL::B;
  s.stage_Q = SL::Q;
  s.stage_R = SL::R;
  s.stage_M = SL::M;
  s.stage_q = SL::q;
  s.stage_r = SL::r;
  s.policy_K = PL::K;
  s.policy_k = PL::k;
  s.value_P = VL::P;
  s.value_p = VL::p;
  return s;
}

template <int NX, int NU>
cudaError_t LqrLaunch<NX, NU>::lqr_tree(bool grid, const Topo* d_topo, const Work* d_work, double reg,
                                        double* d_scalars, double* red, int blocks, int threads,
                                        cudaStream_t stream) {
  if (!grid) {
    lqr_tree_cta_kernel<NX, NU><<<1, threads, 0, stream>>>(d_topo, d_work, reg, d_scalars);
    return cudaGetLastError();
  }
  void* args[] = {&d_topo, &d_work, &reg, &d_scalars, &red};
  const int nb = blocks > 0 ? blocks : max_coresident(lqr_tree_grid_kernel<NX, NU>, threads);
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lqr_tree_grid_kernel<NX, NU>), dim3(nb),
                                     dim3(threads), args, 0, stream);
}

template <int NX, int NU>
int LqrLaunch<NX, NU>::grid_blocks(int threads) {
  return max_coresident(lqr_tree_grid_kernel<NX, NU>, threads);
}

template <int NX, int NU, int T, int MB>
cudaError_t CtaVariant<NX, NU, T, MB>::launch(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                              const DevOptions& opts, int count, cudaStream_t stream) {
  solve_cta_kernel<NX, NU, T, MB><<<count, T, 0, stream>>>(d_topo, d_mp, d_work, opts, count);
  return cudaGetLastError();
}

template <int NX, int NU, int T, int MB>
int CtaVariant<NX, NU, T, MB>::regs() {
  cudaFuncAttributes attr{};
  cudaFuncGetAttributes(&attr, solve_cta_kernel<NX, NU, T, MB>);
  return attr.numRegs;
}

template <int NX, int NU>
cudaError_t SolveLaunch<NX, NU>::solve_grid(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                            const DevOptions& opts, double* red, int blocks, int threads,
                                            cudaStream_t stream) {
  DevOptions o = opts;
  void* args[] = {&d_topo, &d_mp, &d_work, &o, &red};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(solve_grid_kernel<NX, NU>), dim3(blocks),
                                     dim3(threads), args, 0, stream);
}

template <int NX, int NU>
int SolveLaunch<NX, NU>::grid_blocks(int threads) {
  return max_coresident(solve_grid_kernel<NX, NU>, threads);
}


}  // namespace bmpc_b200
