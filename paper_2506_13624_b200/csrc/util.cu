// Utility kernels: result packing for the multi-GPU gather, and the FP64
// FMA microbenchmark that measures the roofline denominator (MEASURED_PEAKS
// has no FP64 figure; SURVEY.md §8d asks for a DFMA measurement).
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <vector>

#include "types.h"

namespace bmpc_b200 {

// dst[i] = [x_i (n*nx) | u_i (n*nu)] for every instance i, contiguous.
__global__ void pack_results_kernel(const Work* __restrict__ works, int count, int n, int nx, int nu,
                                    double* __restrict__ dst) {
  const long long per = static_cast<long long>(n) * (nx + nu);
  const long long total = per * count;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int inst = static_cast<int>(q / per);
    const long long r = q % per;
    const Work& w = works[inst];
    dst[q] = r < static_cast<long long>(n) * nx ? w.x[r] : w.u[r - static_cast<long long>(n) * nx];
  }
}

// Batch scheduling: order instances by their suspended-solve key (descending:
// the largest constraint violation after the probe launch first; finished
// instances last), ties by index. One block, bitonic sort in shared memory;
// beyond kMaxSortCount the identity order is used.
constexpr int kMaxSortCount = 8192;

__global__ void order_by_key_kernel(const DevResume* __restrict__ rs, int count, int npow2, int* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* key = reinterpret_cast<double*>(sm);
  int* idx = reinterpret_cast<int*>(key + npow2);
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    double k = -INFINITY;
    if (i < count && rs[i].state == 1 && !isnan(rs[i].key)) k = rs[i].key;
    key[i] = k;
    idx[i] = i < count ? i : 0x7fffffff;
  }
  __syncthreads();
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool before = key[i] > key[l] || (key[i] == key[l] && idx[i] < idx[l]);
          if (((i & k) == 0) != before) {
            const double tk = key[i];
            key[i] = key[l];
            key[l] = tk;
            const int ti = idx[i];
            idx[i] = idx[l];
            idx[l] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < count; i += blockDim.x) order[i] = idx[i];
}

__global__ void identity_order_kernel(int count, int* __restrict__ order) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) order[i] = i;
}

cudaError_t launch_order_by_key(const DevResume* d_resume, int count, int* d_order, cudaStream_t stream) {
  if (count > kMaxSortCount) {
    identity_order_kernel<<<64, 256, 0, stream>>>(count, d_order);
    return cudaGetLastError();
  }
  int npow2 = 1;
  while (npow2 < count) npow2 <<= 1;
  const size_t smem = static_cast<size_t>(npow2) * (sizeof(double) + sizeof(int));
  // Per-device-context attribute: set before every launch (see allow_smem).
  cudaFuncSetAttribute(reinterpret_cast<const void*>(order_by_key_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kMaxSortCount * (sizeof(double) + sizeof(int))));
  order_by_key_kernel<<<1, 1024, smem, stream>>>(d_resume, count, npow2, d_order);
  return cudaGetLastError();
}

cudaError_t launch_pack_results(const Work* d_works, int count, int n, int nx, int nu, double* dst,
                                cudaStream_t stream) {
  pack_results_kernel<<<1184, 256, 0, stream>>>(d_works, count, n, nx, nu, dst);
  return cudaGetLastError();
}

// 8 independent DFMA chains per thread, `iters` rounds: 16 flops per round.
__global__ void dfma_peak_kernel(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 42.0) out[0] = s;  // keep the chains alive
}

double measure_fp64_peak_tflops(cudaStream_t stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  dfma_peak_kernel<<<blocks, threads, 0, stream>>>(d, iters);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, stream);
    dfma_peak_kernel<<<blocks, threads, 0, stream>>>(d, iters);
    cudaEventRecord(e1, stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flops = 2.0 * 8.0 * static_cast<double>(iters) * blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace bmpc_b200

namespace bmpc_b200 {

// Cost of one cooperative-groups grid barrier (diagnostic for grid mode).
__global__ void grid_sync_bench_kernel(int iters, unsigned long long* out) {
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = t1 - t0;
  }
}

double grid_sync_us(int blocks, int threads, int iters, cudaStream_t stream) {
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sizeof(unsigned long long));
  void* args[] = {&iters, &d};
  cudaLaunchCooperativeKernel(reinterpret_cast<void*>(grid_sync_bench_kernel), dim3(blocks), dim3(threads), args, 0,
                              stream);
  cudaLaunchCooperativeKernel(reinterpret_cast<void*>(grid_sync_bench_kernel), dim3(blocks), dim3(threads), args, 0,
                              stream);
  unsigned long long ns = 0;
  cudaMemcpyAsync(&ns, d, sizeof ns, cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  cudaFree(d);
  return ns * 1e-3 / iters;
}

}  // namespace bmpc_b200

// ---------------------------------------------------------------------------
// Microbenchmark of the team Riccati step (diagnostic): one 16-lane team walks
// a synthetic chain of `steps` stage records resident in global memory.
#include "lqr.cuh"

namespace bmpc_b200 {

template <bool kStamp, int TS>
__global__ void ric_bench_kernel(const double* stages, const double* defects, double* vals, double* pols, int steps,
                                 int prefetch, unsigned long long* cycles) {
  constexpr int NX = 4, NU = 2;
  using SL = StageLayout<NX, NU>;
  using F = RicFlat<NX, NU>;
  __shared__ __align__(16) double Fm[F::size];
  const int lane = threadIdx.x;
  const unsigned mask = TS == 32 ? 0xffffffffu : ((1u << TS) - 1u);
  for (int k = lane; k < F::size; k += TS) Fm[k] = 0.0;
  __syncwarp(mask);
  for (int k = lane; k < NX * NX; k += TS) ric_put_P<NX, NU>(Fm, k, (k % 5 == 0) ? 1.0 : 0.0);
  if (lane < NX) Fm[F::p + lane] = 0.1;
  for (int k = lane; k < SL::size; k += TS) Fm[F::S + k] = stages[k];
  if (lane < NX) Fm[F::c + lane] = defects[lane];
  __syncwarp(mask);
  unsigned long long st[5] = {0, 0, 0, 0, 0};


  unsigned long long t0 = clock64();
  int err = 0;
  for (int k = 0; k < steps; ++k) {
    constexpr int PRE = (SL::size + TS - 1) / TS;
    double pre[PRE];
    double prec = 0.0;
    const double* sp = stages + static_cast<size_t>((k + 1) % steps) * SL::stride;
#pragma unroll
    for (int j = 0; j < PRE; ++j) {
      const int idx = lane + j * TS;
      pre[j] = idx < SL::size ? sp[idx] : 0.0;
    }
    if (lane < NX) prec = defects[((k + 1) % steps) * NX + lane];
    err |= team_riccati_step_u<NX, NU, TS, kStamp>(0.0, mask, Fm, lane, vals + static_cast<size_t>(k) * 20,
                                                   pols + static_cast<size_t>(k) * 10, st);
    __syncwarp(mask);
#pragma unroll
    for (int j = 0; j < PRE; ++j) {
      const int idx = lane + j * TS;
      if (idx < SL::size) Fm[F::S + idx] = pre[j];
    }
    if (lane < NX) Fm[F::c + lane] = prec;
  }
  unsigned long long t1 = clock64();
  if (lane == 0) {
    cycles[0] = t1 - t0;
    cycles[1] = err;
    for (int q = 0; q < 5; ++q) cycles[2 + q] = st[q];
  }
  (void)prefetch;
}

// Cycles per isolated team Riccati step; prefetch == 2: stage-stamped run,
// out[1..5] = cycles per step of each stage (diagnostic).
double ric_step_cycles(int steps, int prefetch, cudaStream_t stream, double* stages) {
  using SL = StageLayout<4, 2>;
  std::vector<double> hs(static_cast<size_t>(steps) * SL::stride, 0.0), hd(static_cast<size_t>(steps) * 4, 0.01);
  for (int k = 0; k < steps; ++k) {
    double* s = hs.data() + static_cast<size_t>(k) * SL::stride;
    for (int i = 0; i < 4; ++i) s[SL::A + i * 5] = 1.0, s[SL::Q + i * 5] = 1.0, s[SL::q + i] = 0.1;
    s[SL::B + 3] = 0.1, s[SL::B + 6] = 0.1, s[SL::R] = 0.5, s[SL::R + 3] = 0.5, s[SL::r] = 0.01;
  }
  double *ds, *dd, *dv, *dp;
  unsigned long long* dc;
  cudaMalloc(&ds, hs.size() * 8);
  cudaMalloc(&dd, hd.size() * 8);
  cudaMalloc(&dv, static_cast<size_t>(steps) * 20 * 8);
  cudaMalloc(&dp, static_cast<size_t>(steps) * 10 * 8);
  cudaMalloc(&dc, 7 * sizeof(unsigned long long));
  cudaMemcpy(ds, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) {
    if (prefetch == 2)
      ric_bench_kernel<true, 16><<<1, 16, 0, stream>>>(ds, dd, dv, dp, steps, prefetch, dc);
    else if (prefetch == 3)  // 32-lane team (diagnostic)
      ric_bench_kernel<true, 32><<<1, 32, 0, stream>>>(ds, dd, dv, dp, steps, prefetch, dc);
    else
      ric_bench_kernel<false, 16><<<1, 16, 0, stream>>>(ds, dd, dv, dp, steps, prefetch, dc);
  }
  unsigned long long hc[7];
  cudaMemcpyAsync(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  cudaFree(ds), cudaFree(dd), cudaFree(dv), cudaFree(dp), cudaFree(dc);
  if (stages && prefetch >= 2)
    for (int q = 0; q < 5; ++q) stages[q] = static_cast<double>(hc[2 + q]) / steps;
  return static_cast<double>(hc[0]) / steps;
}

}  // namespace bmpc_b200

namespace bmpc_b200 {

// Dependent-latency probes (diagnostic): one thread, `n` dependent ops.
__global__ void lat_probe_kernel(double* io, int n, unsigned long long* out) {
  __shared__ double sm[64];
  double a = io[0], b = io[1];
  if (threadIdx.x < 64) sm[threadIdx.x] = io[threadIdx.x % 4];
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
  unsigned long long t1 = clock64();
  int idx = static_cast<int>(a) & 3;
  for (int i = 0; i < n; ++i) idx = static_cast<int>(sm[idx]) & 3;  // dependent LDS chain
  unsigned long long t2 = clock64();
  double c = a;
  for (int i = 0; i < n; ++i) c = 1.0 / (c + 1.5);  // dependent FP64 division chain
  unsigned long long t3 = clock64();
  io[2] = a + idx + c;
  out[0] = t1 - t0;
  out[1] = t2 - t1;
  out[2] = t3 - t2;
}

void latency_probe(double* cyc3, cudaStream_t stream) {
  double h[4] = {1.0000001, 0.9999999, 0, 0};
  double* d;
  unsigned long long* o;
  cudaMalloc(&d, sizeof h);
  cudaMalloc(&o, 3 * sizeof(unsigned long long));
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 4096;
  lat_probe_kernel<<<1, 64, 0, stream>>>(d, n, o);
  lat_probe_kernel<<<1, 64, 0, stream>>>(d, n, o);
  unsigned long long ho[3];
  cudaMemcpyAsync(ho, o, sizeof ho, cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  for (int k = 0; k < 3; ++k) cyc3[k] = static_cast<double>(ho[k]) / n;
  cudaFree(d);
  cudaFree(o);
}

}  // namespace bmpc_b200
