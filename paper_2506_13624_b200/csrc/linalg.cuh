// Fixed-size FP64 block algebra for the branch-MPC hot path (sm_100a).
//
// All blocks are tiny (nx <= 8, nu <= 4) and column-major (X[i + j*rows]),
// matching the reference's Eigen layout so records can be exchanged bit for
// bit. Everything is register/local-array code, fully unrolled by template
// dimension; no dynamic allocation. The two factorizations restate the
// algorithms the reference relies on through Eigen:
//   * Ldlt<N>  — Eigen::LDLT as used by init_bwd_element (lqr_scan.hpp:29),
//                feedback_from_values (lqr_scan.hpp:149) and riccati_step
//                (riccati.hpp:31): pivot on the largest remaining |diagonal|,
//                left-looking LDL^T; `positive()` is the reference's
//                `info() == Success && !(vectorD() <= 0).any()` test.
//   * Lu<N>    — Eigen::PartialPivLU as used by combine_bwd
//                (lqr_scan.hpp:84-90), including the transposed solve that lets
//                one factorization of (I + C P) serve (I + P C)^-1.
#pragma once

#include <cmath>

#ifndef BMPC_HD
#define BMPC_HD __host__ __device__ __forceinline__
#endif

namespace bmpc_b200 {

// out(MxN) = a(MxK) * b(KxN); accumulation order l = 0..K-1 like the
// reference shim's coefficient loop.
template <int M, int K, int N>
BMPC_HD void mm(const double* a, const double* b, double* out) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) s = fma(a[i + l * M], b[l + j * K], s);
      out[i + j * M] = s;
    }
  }
}

// out(MxN) = a^T * b with a (KxM), b (KxN).
template <int M, int K, int N>
BMPC_HD void mtm(const double* a, const double* b, double* out) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) s = fma(a[l + i * K], b[l + j * K], s);
      out[i + j * M] = s;
    }
  }
}

// out(MxN) = a * b^T with a (MxK), b (NxK).
template <int M, int K, int N>
BMPC_HD void mmt(const double* a, const double* b, double* out) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) s = fma(a[i + l * M], b[j + l * N], s);
      out[i + j * M] = s;
    }
  }
}

// y(M) = a(MxK) x(K)
template <int M, int K>
BMPC_HD void mv(const double* a, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < K; ++l) s = fma(a[i + l * M], x[l], s);
    y[i] = s;
  }
}

// y(M) = a^T x with a (KxM)
template <int M, int K>
BMPC_HD void mtv(const double* a, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < K; ++l) s = fma(a[l + i * K], x[l], s);
    y[i] = s;
  }
}

template <int N>
BMPC_HD void symmetrize(double* m) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      const double v = 0.5 * (m[i + j * N] + m[j + i * N]);
      m[i + j * N] = v;
      m[j + i * N] = v;
    }
  }
}

template <int S>
BMPC_HD void copy(const double* a, double* b) {
#pragma unroll
  for (int i = 0; i < S; ++i) b[i] = a[i];
}

template <int S>
BMPC_HD bool all_finite(const double* a) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < S; ++i) ok = ok && isfinite(a[i]);
  return ok;
}

template <int S>
BMPC_HD double dot(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < S; ++i) s = fma(a[i], b[i], s);
  return s;
}

// ---------------------------------------------------------------------------
// Pivoted LDL^T of a symmetric N x N matrix (lower triangle read).
template <int N>
struct Ldlt {
  double m[N * N];
  double dinv[N];  // 1 / D_ii (0 when |D_ii| <= DBL_MIN, Eigen's pseudo-inverse)
  int t[N];
  bool info_ok;

  BMPC_HD void compute(const double* a) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
#pragma unroll
      for (int i = 0; i < N; ++i) m[i + j * N] = i >= j ? a[i + j * N] : a[j + i * N];
    }
    info_ok = true;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      int big = k;
      double bigv = fabs(m[k + k * N]);
#pragma unroll
      for (int i = k + 1; i < N; ++i) {
        const double v = fabs(m[i + i * N]);
        if (v > bigv) {
          bigv = v;
          big = i;
        }
      }
      t[k] = big;
      // Symmetric swap of k <-> big, written with static indices only so the
      // factor stays in registers (a runtime index would force local memory).
#pragma unroll
      for (int b = k + 1; b < N; ++b) {
        if (big == b) {
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double tmp = m[k + j * N];
            m[k + j * N] = m[b + j * N];
            m[b + j * N] = tmp;
          }
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const double tmp = m[i + k * N];
            m[i + k * N] = m[i + b * N];
            m[i + b * N] = tmp;
          }
        }
      }
      if (k > 0) {
        double temp[N];
#pragma unroll
        for (int j = 0; j < k; ++j) temp[j] = m[j + j * N] * m[k + j * N];
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < k; ++j) s = fma(m[k + j * N], temp[j], s);
        m[k + k * N] -= s;
#pragma unroll
        for (int i = k + 1; i < N; ++i) {
          double u = 0.0;
#pragma unroll
          for (int j = 0; j < k; ++j) u = fma(m[i + j * N], temp[j], u);
          m[i + k * N] -= u;
        }
      }
      const double akk = m[k + k * N];
      const double inv = 1.0 / akk;
      dinv[k] = fabs(akk) > 2.2250738585072014e-308 ? inv : 0.0;
      if (k + 1 < N) {
        if (fabs(akk) > 0.0) {
#pragma unroll
          for (int i = k + 1; i < N; ++i) m[i + k * N] *= inv;
        } else {
#pragma unroll
          for (int i = k + 1; i < N; ++i) info_ok = info_ok && (m[i + k * N] == 0.0);
        }
      }
    }
  }

  // info() == Success and every D_ii > 0.
  BMPC_HD bool positive() const {
    bool ok = info_ok;
#pragma unroll
    for (int i = 0; i < N; ++i) ok = ok && (m[i + i * N] > 0.0);
    return ok;
  }

  // swap(x[k], x[tk]) for tk >= k, with static indices.
  BMPC_HD static void swap_static(double* x, int k, int tk) {
#pragma unroll
    for (int b = 0; b < N; ++b) {
      if (b > k && tk == b) {
        const double tmp = x[k];
        x[k] = x[b];
        x[b] = tmp;
      }
    }
  }

  // In-place solve of A X = B for C right-hand-side columns (B is N x C).
  template <int C>
  BMPC_HD void solve(double* b) const {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double* x = b + c * N;
#pragma unroll
      for (int k = 0; k < N; ++k) swap_static(x, k, t[k]);
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int k = 0; k < i; ++k) x[i] = fma(-m[i + k * N], x[k], x[i]);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] *= dinv[i];
#pragma unroll
      for (int i = N - 1; i >= 0; --i) {
#pragma unroll
        for (int k = i + 1; k < N; ++k) x[i] = fma(-m[k + i * N], x[k], x[i]);
      }
#pragma unroll
      for (int k = N - 1; k >= 0; --k) swap_static(x, k, t[k]);
    }
  }
};

// ---------------------------------------------------------------------------
// Row-pivoted LU of a general N x N matrix. Zero pivots are skipped (no
// division), so a singular matrix propagates inf/nan into the solves exactly
// like Eigen::PartialPivLU; combine_bwd then reports FactorizationError.
template <int N>
struct Lu {
  double lu[N * N];
  double uinv[N];  // 1 / U_ii (inf / nan propagate like a division would)
  int perm[N];  // row i of P*A is row perm[i] of A

  BMPC_HD void compute(const double* a) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) lu[i] = a[i];
#pragma unroll
    for (int i = 0; i < N; ++i) perm[i] = i;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      int p = k;
      double best = fabs(lu[k + k * N]);
#pragma unroll
      for (int i = k + 1; i < N; ++i) {
        const double v = fabs(lu[i + k * N]);
        if (v > best) {
          best = v;
          p = i;
        }
      }
      if (best != 0.0) {
#pragma unroll
        for (int b = k + 1; b < N; ++b) {
          if (p == b) {
#pragma unroll
            for (int j = 0; j < N; ++j) {
              const double tmp = lu[k + j * N];
              lu[k + j * N] = lu[b + j * N];
              lu[b + j * N] = tmp;
            }
            const int tp = perm[k];
            perm[k] = perm[b];
            perm[b] = tp;
          }
        }
        const double inv = 1.0 / lu[k + k * N];
#pragma unroll
        for (int i = k + 1; i < N; ++i) lu[i + k * N] *= inv;
      }
      uinv[k] = 1.0 / lu[k + k * N];
#pragma unroll
      for (int j = k + 1; j < N; ++j) {
        const double ukj = lu[k + j * N];
#pragma unroll
        for (int i = k + 1; i < N; ++i) lu[i + j * N] = fma(-lu[i + k * N], ukj, lu[i + j * N]);
      }
    }
  }

  // x = A^-1 b for C columns; b (N x C) in, x out (distinct buffers).
  template <int C>
  BMPC_HD void solve(const double* b, double* x) const {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double* bc = b + c * N;
      double* xc = x + c * N;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double v = bc[0];
#pragma unroll
        for (int j = 1; j < N; ++j) v = perm[i] == j ? bc[j] : v;
        xc[i] = v;
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int k = 0; k < i; ++k) xc[i] = fma(-lu[i + k * N], xc[k], xc[i]);
      }
#pragma unroll
      for (int i = N - 1; i >= 0; --i) {
#pragma unroll
        for (int k = i + 1; k < N; ++k) xc[i] = fma(-lu[i + k * N], xc[k], xc[i]);
        xc[i] = xc[i] * uinv[i];
      }
    }
  }

  // x = A^-T b for C columns: A^T = U^T L^T P, x = P^T L^-T U^-T b.
  template <int C>
  BMPC_HD void solve_transposed(const double* b, double* x) const {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double* bc = b + c * N;
      double y[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = bc[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s = fma(-lu[k + i * N], y[k], s);
        y[i] = s * uinv[i];
      }
#pragma unroll
      for (int i = N - 1; i >= 0; --i) {
        double s = y[i];
#pragma unroll
        for (int k = i + 1; k < N; ++k) s = fma(-lu[k + i * N], y[k], s);
        y[i] = s;
      }
      double* xc = x + c * N;
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j)
          if (perm[i] == j) xc[j] = y[i];
      }
    }
  }
};

}  // namespace bmpc_b200

namespace bmpc_b200 {

// Asynchronous global -> shared copies (LDGSTS), 16 bytes each; both
// addresses 16-byte aligned.
__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace bmpc_b200
