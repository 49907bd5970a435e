// Kernel templates and their launchers (sm_100a). One kernel launch per
// solve: the whole iLQR/AL loop is device-resident. Instantiated per (nx, nu)
// in inst_*.cu so the heavy unrolled code compiles in parallel.
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"
#include "solver.cuh"

namespace bmpc_b200 {

static_assert(kRedSlotsHost == kRedSlots, "reduction slot count mismatch");

__host__ __device__ constexpr size_t red_smem_bytes(int threads) {
  return ((static_cast<size_t>(kRedSlots) * (threads / 32) * sizeof(double)) + 15) / 16 * 16;
}

// Stage the per-instance structs in shared memory (read on every node op).
struct BlockCtx {
  Topo topo;
  ModelParams mp;
  Work work;
};

// THREADS x MINB trade registers for resident instances per SM:
// registers/thread <= 65536 / (THREADS * MINB).
template <int NX, int NU, int THREADS, int MINB, bool SEQ, int FEAT = 0>
__global__ void __launch_bounds__(THREADS, MINB) solve_cta_kernel(const Topo* __restrict__ topo,
                                                        const ModelParams* __restrict__ mps,
                                                        const Work* __restrict__ works, DevOptions opts,
                                                        int count) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  if (static_cast<int>(blockIdx.x) >= count) return;
  const int b = opts.order ? opts.order[blockIdx.x] : static_cast<int>(blockIdx.x);
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.mp = mps[b];
    ctx.work = works[b];
    red.flag = 0;
  }
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  red.part = reinterpret_cast<double*>(dyn_smem);
  __syncthreads();
  // One warp per segment team when the block is wide enough (>= 4 teams).
  constexpr int kTeam = (THREADS >= 128 && team_size<NX, NU>() == 16) ? 32 : 0;
  Solver<NX, NU, CtaGroupT<THREADS>, SEQ, kTeam, FEAT> s(CtaGroupT<THREADS>{&red}, ctx.topo, ctx.mp, ctx.work, opts);
  s.tsm = dyn_smem + red_smem_bytes(THREADS);
  s.wbuf = reinterpret_cast<double*>(s.tsm);
  s.wcap = THREADS;
  s.solve();
}

template <int NX, int NU, int FEAT = 0>
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
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  red.part = reinterpret_cast<double*>(dyn_smem);
  __syncthreads();
  // One warp per team, as in the 256-thread per-instance kernels.
  constexpr int kTeam = team_size<NX, NU>() == 16 ? 32 : 0;
  Solver<NX, NU, GridGroup, false, kTeam, FEAT> s(GridGroup{&red, red_scratch, nullptr}, ctx.topo, ctx.mp, ctx.work,
                                                  opts);
  s.tsm = dyn_smem + red_smem_bytes(blockDim.x);
  s.wbuf = reinterpret_cast<double*>(s.tsm);
  s.wcap = blockDim.x;
  s.solve();
}

template <int NX, int NU, class G>
__device__ void lqr_tree_body(G g, BlockCtx& ctx, double reg, double* scalars, int seq_max, int condensed) {
  ModelParams dummy{};
  DevOptions o{};
  o.seq_max_len = seq_max;
  o.condensed = condensed;
  o.fwd_scan_min = seq_max > 0 ? seq_max + 1 : 1;  // kernel-level API: forward mirrors the backward strategy
  o.keep_values = 1;
  o.chunk_bwd = 1;  // long segments in 256-thread blocks: the chunked sweep (tested against the oracle here)
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  Solver<NX, NU, G, false, 0, kFeatCond | kFeatChunk> s(g, ctx.topo, dummy, ctx.work, o);
  s.tsm = dyn_smem + red_smem_bytes(blockDim.x);
  s.wbuf = reinterpret_cast<double*>(s.tsm);
  s.wcap = blockDim.x;
  s.lqr_tree(reg, scalars);
}

template <int NX, int NU>
__global__ void __launch_bounds__(256) lqr_tree_cta_kernel(const Topo* topo, const Work* works, double reg,
                                                           double* scalars, int seq_max, int condensed) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.work = works[0];
    red.flag = 0;
  }
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  red.part = reinterpret_cast<double*>(dyn_smem);
  __syncthreads();
  lqr_tree_body<NX, NU>(CtaGroup{&red}, ctx, reg, scalars, seq_max, condensed);
}

template <int NX, int NU>
__global__ void __launch_bounds__(256) lqr_tree_grid_kernel(const Topo* topo, const Work* works, double reg,
                                                            double* scalars, double* red_scratch, int seq_max,
                                                            int condensed) {
  __shared__ RedSmem red;
  __shared__ BlockCtx ctx;
  if (threadIdx.x == 0) {
    ctx.topo = *topo;
    ctx.work = works[0];
    red.flag = 0;
  }
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  red.part = reinterpret_cast<double*>(dyn_smem);
  __syncthreads();
  lqr_tree_body<NX, NU>(GridGroup{&red, red_scratch, nullptr}, ctx, reg, scalars, seq_max, condensed);
}

// Batched scan-element primitives of lqr_scan.hpp (the `associativity`
// suite's entry point, verification.hpp:110-137).
template <int NX, int NU>
__global__ void lqr_elements_kernel(int op, int count, const double* __restrict__ a, const double* __restrict__ b,
                                    double reg, double* __restrict__ out) {
  using E = BwdLayout<NX>;
  using F = FwdLayout<NX>;
  using S = LqStage<NX, NU>;
  using SL = StageLayout<NX, NU>;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    if (op == 0) {  // init_bwd_element (lqr_scan.hpp:28-49)
      const double* r = a + static_cast<size_t>(i) * S::size;
      double st[SL::size];
      copy<NX * NX>(r + S::A, st + SL::A);
      copy<NX * NU>(r + S::B, st + SL::B);
      copy<NX * NX>(r + S::Q, st + SL::Q);
      copy<NU * NU>(r + S::R, st + SL::R);
      copy<NU * NX>(r + S::M, st + SL::M);
      copy<NX>(r + S::q, st + SL::q);
      copy<NU>(r + S::r, st + SL::r);
      double* e = out + static_cast<size_t>(i) * E::size;
      if (init_bwd_element<NX, NU>(st, reg, r + S::c, e) != kBwdOk)
        for (int k = 0; k < E::size; ++k) e[k] = NAN;  // the reference's LDLT(R) failure
    } else if (op == 1) {  // combine_bwd (lqr_scan.hpp:80-111), first (+) second
      combine_bwd<NX>(a + static_cast<size_t>(i) * E::size, b + static_cast<size_t>(i) * E::size,
                      out + static_cast<size_t>(i) * E::size);
    } else {  // combine_fwd (lqr_scan.hpp:171-173)
      combine_fwd<NX>(a + static_cast<size_t>(i) * F::size, b + static_cast<size_t>(i) * F::size,
                      out + static_cast<size_t>(i) * F::size);
    }
  }
}

template <int NX, int NU>
cudaError_t LqrLaunch<NX, NU>::elements(int op, int count, const double* a, const double* b, double reg, double* out,
                                        cudaStream_t stream) {
  const int blocks = count > 0 ? (count + 127) / 128 : 1;
  lqr_elements_kernel<NX, NU><<<blocks < 1184 ? blocks : 1184, 128, 0, stream>>>(op, count, a, b, reg, out);
  return cudaGetLastError();
}


// Dynamic shared memory of one block: reduction warp partials, then the
// cooperative-combine team scratch.
template <int NX, int NU>
static size_t team_smem_bytes(int threads) {
  constexpr int ts = team_size<NX, NU>();
  const size_t team = ts > 0 ? static_cast<size_t>(threads / ts) * Solver<NX, NU, CtaGroup>::slot_bytes() : 16;
  const size_t walk = static_cast<size_t>(threads) * Solver<NX, NU, CtaGroup>::kWE * sizeof(double);
  return red_smem_bytes(threads) + (team > walk ? team : walk);
}

// The dynamic shared-memory opt-in is a per-device-context attribute, so it is
// set before every launch (a host-side call of ~1 us) rather than once per
// process: a process that solves on several devices gets it on each.
template <class K>
static void allow_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(bytes));
}

template <class K>
static int max_coresident(K kernel, int threads, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  allow_smem(kernel, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
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
                                        cudaStream_t stream, int seq_max, int condensed) {
  const size_t smem = team_smem_bytes<NX, NU>(threads);
  if (!grid) {
    allow_smem(lqr_tree_cta_kernel<NX, NU>, smem);
    lqr_tree_cta_kernel<NX, NU><<<1, threads, smem, stream>>>(d_topo, d_work, reg, d_scalars, seq_max, condensed);
    return cudaGetLastError();
  }
  void* args[] = {&d_topo, &d_work, &reg, &d_scalars, &red, &seq_max, &condensed};
  const int nb = blocks > 0 ? blocks : max_coresident(lqr_tree_grid_kernel<NX, NU>, threads, smem);
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lqr_tree_grid_kernel<NX, NU>), dim3(nb),
                                     dim3(threads), args, smem, stream);
}

template <int NX, int NU>
int LqrLaunch<NX, NU>::grid_blocks(int threads) {
  return max_coresident(lqr_tree_grid_kernel<NX, NU>, threads, team_smem_bytes<NX, NU>(threads));
}

template <int NX, int NU, int T, int MB>
cudaError_t CtaVariant<NX, NU, T, MB>::launch(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                              const DevOptions& opts, int count, bool seq_only, cudaStream_t stream) {
  const size_t smem = team_smem_bytes<NX, NU>(T);
  if (seq_only && team_size<NX, NU>() > 0) {
    allow_smem(solve_cta_kernel<NX, NU, T, MB, true>, smem);
    solve_cta_kernel<NX, NU, T, MB, true><<<count, T, smem, stream>>>(d_topo, d_mp, d_work, opts, count);
  } else {
    allow_smem(solve_cta_kernel<NX, NU, T, MB, false>, smem);
    solve_cta_kernel<NX, NU, T, MB, false><<<count, T, smem, stream>>>(d_topo, d_mp, d_work, opts, count);
  }
  return cudaGetLastError();
}

template <int NX, int NU, int T, int MB>
int CtaVariant<NX, NU, T, MB>::regs(bool seq_only) {
  cudaFuncAttributes attr{};
  if (seq_only)
    cudaFuncGetAttributes(&attr, solve_cta_kernel<NX, NU, T, MB, true>);
  else
    cudaFuncGetAttributes(&attr, solve_cta_kernel<NX, NU, T, MB, false>);
  return attr.numRegs;
}

template <int NX, int NU>
cudaError_t SolveLaunch<NX, NU>::solve_grid(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                            const DevOptions& opts, double* red, int blocks, int threads,
                                            cudaStream_t stream) {
  DevOptions o = opts;
  void* args[] = {&d_topo, &d_mp, &d_work, &o, &red};
  const size_t smem = team_smem_bytes<NX, NU>(threads);
  allow_smem(solve_grid_kernel<NX, NU>, smem);
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(solve_grid_kernel<NX, NU>), dim3(blocks),
                                     dim3(threads), args, smem, stream);
}

// Solves with an optional path (single-shooting line search, condensed shared
// segment): one 256-thread shape per (nx, nu), FIFO over the batch, and the
// whole-GPU kernel; FEAT selects the compiled-in paths.
template <int NX, int NU, int FEAT>
static cudaError_t launch_cta_feat(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                   const DevOptions& opts, int count, bool seq_only, cudaStream_t stream) {
  constexpr int T = 256;
  const size_t smem = team_smem_bytes<NX, NU>(T);
  if (seq_only && team_size<NX, NU>() > 0) {
    allow_smem(solve_cta_kernel<NX, NU, T, 1, true, FEAT>, smem);
    solve_cta_kernel<NX, NU, T, 1, true, FEAT><<<count, T, smem, stream>>>(d_topo, d_mp, d_work, opts, count);
  } else {
    allow_smem(solve_cta_kernel<NX, NU, T, 1, false, FEAT>, smem);
    solve_cta_kernel<NX, NU, T, 1, false, FEAT><<<count, T, smem, stream>>>(d_topo, d_mp, d_work, opts, count);
  }
  return cudaGetLastError();
}

template <int NX, int NU, int FEAT>
static cudaError_t launch_grid_feat(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                    const DevOptions& opts, double* red, int blocks, int threads,
                                    cudaStream_t stream) {
  DevOptions o = opts;
  void* args[] = {&d_topo, &d_mp, &d_work, &o, &red};
  const size_t smem = team_smem_bytes<NX, NU>(threads);
  const int fit = max_coresident(solve_grid_kernel<NX, NU, FEAT>, threads, smem);
  if (blocks > fit) blocks = fit;  // co-residency of this variant (red holds >= blocks rows)
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(solve_grid_kernel<NX, NU, FEAT>), dim3(blocks),
                                     dim3(threads), args, smem, stream);
}

template <int NX, int NU>
cudaError_t SolveLaunch<NX, NU>::solve_cta_special(const Topo* d_topo, const ModelParams* d_mp, const Work* d_work,
                                                   const DevOptions& opts, int count, bool seq_only,
                                                   cudaStream_t stream) {
  if (opts.nonlinear_ls && opts.condensed)
    return launch_cta_feat<NX, NU, kFeatNL | kFeatCond>(d_topo, d_mp, d_work, opts, count, seq_only, stream);
  if (opts.condensed) return launch_cta_feat<NX, NU, kFeatCond>(d_topo, d_mp, d_work, opts, count, seq_only, stream);
  return launch_cta_feat<NX, NU, kFeatNL>(d_topo, d_mp, d_work, opts, count, seq_only, stream);
}

template <int NX, int NU>
cudaError_t SolveLaunch<NX, NU>::solve_grid_special(const Topo* d_topo, const ModelParams* d_mp,
                                                    const Work* d_work, const DevOptions& opts, double* red,
                                                    int blocks, int threads, cudaStream_t stream) {
  if (opts.nonlinear_ls && opts.condensed)
    return launch_grid_feat<NX, NU, kFeatNL | kFeatCond>(d_topo, d_mp, d_work, opts, red, blocks, threads, stream);
  if (opts.condensed)
    return launch_grid_feat<NX, NU, kFeatCond>(d_topo, d_mp, d_work, opts, red, blocks, threads, stream);
  return launch_grid_feat<NX, NU, kFeatNL>(d_topo, d_mp, d_work, opts, red, blocks, threads, stream);
}

template <int NX, int NU>
int SolveLaunch<NX, NU>::grid_blocks(int threads) {
  return max_coresident(solve_grid_kernel<NX, NU>, threads, team_smem_bytes<NX, NU>(threads));
}


}  // namespace bmpc_b200
