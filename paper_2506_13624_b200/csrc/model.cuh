// Device node models: the reference's per-node callbacks (problem.hpp:15-40)
// restated as device functions selected at compile time, since std::function
// callbacks cannot run on the GPU. Two families cover every problem the
// reference builds:
//   * UnicycleTracking — kinematic unicycle with RK4 (unicycle.hpp:19-74),
//     quadratic tracking costs (problem.hpp:194-222) and the ego constraints
//     (scenarios.hpp:206-248): intersection, latency and multi-stage scenes.
//   * AffineQuadratic  — affine dynamics + convex quadratic costs without
//     constraints: testing::random_lq_problem (oracles.hpp:316-365).
#pragma once

#include "linalg.cuh"
#include "lqr.cuh"
#include "types.h"

namespace bmpc_b200 {

template <int NX, int NU>
struct LqStage {  // packing of ModelParams::lq_stage records
  static constexpr int A = 0, B = NX * NX, c = B + NX * NU, Q = c + NX, R = Q + NX * NX, M = R + NU * NU,
                       q = M + NU * NX, r = q + NX, size = r + NU;
};

// Constraint rows at a node: non-leaf 4 box rows + nv distance rows, leaf nv.
template <int NX, int NU>
__device__ __forceinline__ int num_constraints(const ModelParams& mp, bool leaf) {
  if (mp.kind != kModelUnicycle) return 0;
  return (leaf ? 0 : 4) + mp.nv;
}

// --------------------------------------------------------------- unicycle
__device__ __forceinline__ void unicycle_derivative(const double* x, const double* u, double* dx) {
  double s, c;
  sincos(x[2], &s, &c);
  dx[0] = x[3] * c;
  dx[1] = x[3] * s;
  dx[2] = u[1];
  dx[3] = u[0];
}

// unicycle::step (unicycle.hpp:36-42). The heading at stages 2 and 3 is the
// same expression psi + dt/2 * u1 (psi' = u1), so its sincos is shared.
__device__ __forceinline__ void unicycle_step(const double* x, const double* u, double dt, double* xn) {
  double k1[4], k2[4], k3[4], k4[4], t[4];
  unicycle_derivative(x, u, k1);
  const double hdt = 0.5 * dt;
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = x[i] + hdt * k1[i];
  double s2, c2;
  sincos(t[2], &s2, &c2);
  k2[0] = t[3] * c2;
  k2[1] = t[3] * s2;
  k2[2] = u[1];
  k2[3] = u[0];
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = x[i] + hdt * k2[i];
  k3[0] = t[3] * c2;  // t[2] == x[2] + hdt * u[1] again
  k3[1] = t[3] * s2;
  k3[2] = u[1];
  k3[3] = u[0];
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = x[i] + dt * k3[i];
  unicycle_derivative(t, u, k4);
  const double s6 = dt / 6.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) xn[i] = x[i] + s6 * (((k1[i] + 2.0 * k2[i]) + 2.0 * k3[i]) + k4[i]);
}

// d(derivative)/dx at x (unicycle.hpp:25-34); only (0,2),(0,3),(1,2),(1,3) are
// non-zero, d/du is the constant selector Ju(2,1) = Ju(3,0) = 1.
__device__ __forceinline__ void unicycle_jx(const double* x, double* j02, double* j03, double* j12, double* j13) {
  double s, c;
  sincos(x[2], &s, &c);
  *j02 = -x[3] * s;
  *j03 = c;
  *j12 = x[3] * c;
  *j13 = s;
}

// unicycle::step_jacobians (unicycle.hpp:44-74): the analytic chain rule
// through the RK4 stages, evaluated on the sparsity of the stage Jacobians
// (J has four non-zeros, so J*(I + h dk) touches rows 0-1 only).
__device__ __forceinline__ void unicycle_step_jacobians(const double* x, const double* u, double dt, double* A,
                                                        double* B) {
  double k1[4], k2[4], k3[4], x2[4], x3[4], x4[4];
  unicycle_derivative(x, u, k1);
  const double hdt = 0.5 * dt;
#pragma unroll
  for (int i = 0; i < 4; ++i) x2[i] = x[i] + hdt * k1[i];
  unicycle_derivative(x2, u, k2);
#pragma unroll
  for (int i = 0; i < 4; ++i) x3[i] = x[i] + hdt * k2[i];
  unicycle_derivative(x3, u, k3);
#pragma unroll
  for (int i = 0; i < 4; ++i) x4[i] = x[i] + dt * k3[i];

  // Dense 4x4 / 4x2 stage derivatives (column-major), kept dense for clarity;
  // the zero pattern is exact, so rounding matches the dense reference.
  double J[4][16];
  {
    const double* pts[4] = {x, x2, x3, x4};
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int i = 0; i < 16; ++i) J[s][i] = 0.0;
      unicycle_jx(pts[s], &J[s][0 + 2 * 4], &J[s][0 + 3 * 4], &J[s][1 + 2 * 4], &J[s][1 + 3 * 4]);
    }
  }
  // Ju: (2,1) = 1, (3,0) = 1.
  double Ju[8] = {0, 0, 0, 1, 0, 0, 1, 0};
  double I[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) I[i] = (i % 5 == 0) ? 1.0 : 0.0;

  double dk1x[16], dk2x[16], dk3x[16], dk4x[16], T[16];
  copy<16>(J[0], dk1x);
#pragma unroll
  for (int i = 0; i < 16; ++i) T[i] = I[i] + hdt * dk1x[i];
  mm<4, 4, 4>(J[1], T, dk2x);
#pragma unroll
  for (int i = 0; i < 16; ++i) T[i] = I[i] + hdt * dk2x[i];
  mm<4, 4, 4>(J[2], T, dk3x);
#pragma unroll
  for (int i = 0; i < 16; ++i) T[i] = I[i] + dt * dk3x[i];
  mm<4, 4, 4>(J[3], T, dk4x);

  double dk1u[8], dk2u[8], dk3u[8], dk4u[8], Tu[8];
  copy<8>(Ju, dk1u);
#pragma unroll
  for (int i = 0; i < 8; ++i) Tu[i] = hdt * dk1u[i];
  mm<4, 4, 2>(J[1], Tu, dk2u);
#pragma unroll
  for (int i = 0; i < 8; ++i) dk2u[i] += Ju[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) Tu[i] = hdt * dk2u[i];
  mm<4, 4, 2>(J[2], Tu, dk3u);
#pragma unroll
  for (int i = 0; i < 8; ++i) dk3u[i] += Ju[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) Tu[i] = dt * dk3u[i];
  mm<4, 4, 2>(J[3], Tu, dk4u);
#pragma unroll
  for (int i = 0; i < 8; ++i) dk4u[i] += Ju[i];

  const double s6 = dt / 6.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) A[i] = I[i] + s6 * (((dk1x[i] + 2.0 * dk2x[i]) + 2.0 * dk3x[i]) + dk4x[i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) B[i] = s6 * (((dk1u[i] + 2.0 * dk2u[i]) + 2.0 * dk3u[i]) + dk4u[i]);
}

// unicycle_step_jacobians on its sparsity, bit-identical to the dense chain
// rule above for finite inputs: the stage Jacobians J only couple (px, py) to
// (psi, v), whose own dynamics are trivial, so dk_s/dx = J_s exactly, the
// stage-3 point has the stage-2 heading and speed (J_3 = J_2), and every
// dropped term of the dense products is an exact zero. Three sincos instead
// of seven, no 4x4 products.
__device__ __forceinline__ void unicycle_step_jacobians_sparse(const double* x, const double* u, double dt,
                                                               double* A, double* B) {
  const double hdt = 0.5 * dt;
  const double psi2 = x[2] + hdt * u[1], v2 = x[3] + hdt * u[0];  // stages 2 and 3
  const double psi4 = x[2] + dt * u[1], v4 = x[3] + dt * u[0];
  double s1, c1, s2, c2, s4, c4;
  sincos(x[2], &s1, &c1);
  sincos(psi2, &s2, &c2);
  sincos(psi4, &s4, &c4);
  // J(0,2) = -v s, J(0,3) = c, J(1,2) = v c, J(1,3) = s at each stage point.
  const double j1[4] = {-x[3] * s1, c1, x[3] * c1, s1};
  const double j2[4] = {-v2 * s2, c2, v2 * c2, s2};
  const double j4[4] = {-v4 * s4, c4, v4 * c4, s4};
  const double s6 = dt / 6.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) A[i] = (i % 5 == 0) ? 1.0 : 0.0;
  // A(r, c) for r in {0,1}, c in {2,3}: entry e = 2r + (c - 2).
#pragma unroll
  for (int r = 0; r < 2; ++r) {
#pragma unroll
    for (int c = 2; c < 4; ++c) {
      const int e = 2 * r + (c - 2);
      A[r + 4 * c] = 0.0 + s6 * (((j1[e] + 2.0 * j2[e]) + 2.0 * j2[e]) + j4[e]);
    }
  }
  // B rows 0,1: dk_s u(r, 0) = J_s(r,3) h_s, dk_s u(r, 1) = J_s(r,2) h_s (h = dt/2, dt/2, dt);
  // rows 2,3: the selector Ju, B(2,1) = B(3,0) = s6 * 6.
#pragma unroll
  for (int r = 0; r < 2; ++r) {
#pragma unroll
    for (int cu = 0; cu < 2; ++cu) {
      const int e = 2 * r + (cu == 0 ? 1 : 0);
      const double d2 = j2[e] * hdt, d3 = j2[e] * hdt, d4 = j4[e] * dt;
      B[r + 4 * cu] = s6 * (((0.0 + 2.0 * d2) + 2.0 * d3) + d4);
    }
  }
  const double sel = s6 * (((1.0 + 2.0 * 1.0) + 2.0 * 1.0) + 1.0);
  B[2 + 4 * 0] = s6 * (((0.0 + 2.0 * 0.0) + 2.0 * 0.0) + 0.0);
  B[3 + 4 * 0] = sel;
  B[2 + 4 * 1] = sel;
  B[3 + 4 * 1] = B[2 + 4 * 0];
}

// ego_constraints (scenarios.hpp:206-248) values and, optionally, Jacobians.
// Rows: [a-amax, -a-amax, w-wmax, -w-wmax] (non-leaf) then r - sqrt(d^2+eps).
template <bool kJac>
__device__ __forceinline__ int ego_constraints(const ModelParams& mp, int node, bool leaf, const double* x,
                                               const double* u, double* g, double* Jx /*[kMaxCon*4]*/,
                                               double* Ju /*[kMaxCon*2]*/) {
  const int nb = leaf ? 0 : 4;
  const int nc = nb + mp.nv;
  if (kJac) {
#pragma unroll
    for (int i = 0; i < kMaxCon * 4; ++i) Jx[i] = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxCon * 2; ++i) Ju[i] = 0.0;
  }
  if (!leaf) {
    g[0] = u[0] - mp.a_max;
    g[1] = -u[0] - mp.a_max;
    g[2] = u[1] - mp.w_max;
    g[3] = -u[1] - mp.w_max;
    if (kJac) {  // Ju row-major over rows here: Ju[row*2 + col]
      Ju[0 * 2 + 0] = 1.0;
      Ju[1 * 2 + 0] = -1.0;
      Ju[2 * 2 + 1] = 1.0;
      Ju[3 * 2 + 1] = -1.0;
    }
  }
  const double* vp = mp.vehicles + static_cast<long long>(node) * mp.nv * 2;
#pragma unroll
  for (int v = 0; v < kMaxVehicles; ++v) {
    if (v < mp.nv) {
      const double dx = x[0] - vp[2 * v + 0];
      const double dy = x[1] - vp[2 * v + 1];
      const double dist = sqrt(dx * dx + dy * dy + 1e-6);
      g[nb + v] = mp.radius - dist;
      if (kJac) {
        Jx[(nb + v) * 4 + 0] = -dx / dist;
        Jx[(nb + v) * 4 + 1] = -dy / dist;
      }
    }
  }
  return nc;
}

// Active-set AL penalty (problem.hpp:85-93).
__device__ __forceinline__ double al_penalty(const double* g, const double* eta, int nc, double rho) {
  double value = 0.0;
#pragma unroll
  for (int m = 0; m < kMaxCon; ++m) {
    if (m < nc && (g[m] >= 0.0 || eta[m] > 0.0)) value += eta[m] * g[m] + 0.5 * rho * g[m] * g[m];
  }
  return value;
}

// 0.5 e' W e with W dense n x n (column-major).
template <int N>
__device__ __forceinline__ double quad_form(const double* W, const double* e) {
  double We[N];
  mv<N, N>(W, e, We);
  return 0.5 * dot<N>(e, We);
}
// Same value for a diagonal W (the dropped terms of mv are exact zeros).
template <int N>
__device__ __forceinline__ double quad_form_diag(const double* W, const double* e) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) s = fma(e[i], W[(N + 1) * i] * e[i], s);
  return 0.5 * s;
}

// ----------------------------------------------------------- generic node API
// Dynamics f(x, u) of non-leaf `node`.
template <int NX, int NU>
__device__ __forceinline__ void node_dynamics(const ModelParams& mp, int node, const double* x, const double* u,
                                              double* xn) {
  if constexpr (NX == 4 && NU == 2) {
    if (mp.kind == kModelUnicycle) {
      unicycle_step(x, u, mp.dt, xn);
      return;
    }
  }
  using S = LqStage<NX, NU>;
  const double* s = mp.lq_stage + static_cast<long long>(node) * S::size;
  double a[NX], b[NX];
  mv<NX, NX>(s + S::A, x, a);
  mv<NX, NU>(s + S::B, u, b);
#pragma unroll
  for (int i = 0; i < NX; ++i) xn[i] = (a[i] + b[i]) + s[S::c + i];
}

// Node objective value (weight not applied) plus AL penalty and max g.
// Matches evaluate (problem.hpp:115-134) per node.
template <int NX, int NU>
__device__ __forceinline__ void node_cost(const ModelParams& mp, int node, bool leaf, const double* x,
                                          const double* u, const double* eta, double rho, double* cost,
                                          double* penalty, double* gmax) {
  *penalty = 0.0;
  *gmax = -INFINITY;
  if constexpr (NX == 4 && NU == 2) {
    if (mp.kind == kModelUnicycle) {
      const double* ref = mp.reference + static_cast<long long>(node) * 4;
      double e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = x[i] - ref[i];
      if (mp.w_diag) {
        *cost = leaf ? quad_form_diag<4>(mp.Wf, e) : quad_form_diag<4>(mp.Wx, e) + quad_form_diag<2>(mp.Wu, u);
      } else if (leaf) {
        *cost = quad_form<4>(mp.Wf, e);
      } else {
        *cost = quad_form<4>(mp.Wx, e) + quad_form<2>(mp.Wu, u);
      }
      // ego_constraints + al_penalty + max g fused row by row (same rows, same
      // expressions, same order), so no constraint array is materialised: a
      // runtime-indexed g[] lives in local memory on the line-search path.
      double value = 0.0, m = -INFINITY;
      auto row = [&](double gm, double em) {
        if (gm >= 0.0 || em > 0.0) value += em * gm + 0.5 * rho * gm * gm;
        m = fmax(m, gm);
      };
      if (!leaf) {
        row(u[0] - mp.a_max, eta[0]);
        row(-u[0] - mp.a_max, eta[1]);
        row(u[1] - mp.w_max, eta[2]);
        row(-u[1] - mp.w_max, eta[3]);
      }
      const int nb = leaf ? 0 : 4;
      const double* vp = mp.vehicles + static_cast<long long>(node) * mp.nv * 2;
#pragma unroll
      for (int v = 0; v < kMaxVehicles; ++v) {
        if (v < mp.nv) {
          const double dx = x[0] - vp[2 * v + 0];
          const double dy = x[1] - vp[2 * v + 1];
          const double dist = sqrt(dx * dx + dy * dy + 1e-6);
          row(mp.radius - dist, eta[nb + v]);
        }
      }
      *penalty = value;
      *gmax = m;
      return;
    }
  }
  if (leaf) {
    const double* l = mp.lq_leaf + static_cast<long long>(node) * (NX * NX + NX);
    double Px[NX];
    mv<NX, NX>(l, x, Px);
    *cost = 0.5 * dot<NX>(x, Px) + dot<NX>(l + NX * NX, x);
  } else {
    using S = LqStage<NX, NU>;
    const double* s = mp.lq_stage + static_cast<long long>(node) * S::size;
    double Qx[NX], Ru[NU], Mx[NU];
    mv<NX, NX>(s + S::Q, x, Qx);
    mv<NU, NU>(s + S::R, u, Ru);
    mv<NU, NX>(s + S::M, x, Mx);
    *cost = (((0.5 * dot<NX>(x, Qx) + dot<NX>(s + S::q, x)) + 0.5 * dot<NU>(u, Ru)) + dot<NU>(s + S::r, u)) +
            dot<NU>(u, Mx);
  }
}

// Structured form of the unicycle expansion below for diagonal weights: the
// same operations on the non-zero pattern (box rows have Ju = +-1 and Jx = 0,
// distance rows Jx in columns 0-1 only, M = 0), so the stage record is
// bit-identical to the dense path for finite inputs at a fraction of the work
// and registers. Only the kVar variable entries change between passes; the
// constant remainder (identity / zero blocks, the input selector of B) is
// written once per solve by unicycle_stage_constants.
struct UniRec {
  using L = StageLayout<4, 2>;
  static constexpr int kVar = 22;
  // Dense StageLayout offsets of the variable entries: A(0..1, 2..3), B(0..1, :),
  // Q(0..1, 0..1) Q22 Q33, R00 R11, q, r. Leaves use the Q / q ones (8..13, 16..19).
  __host__ __device__ static constexpr int pos(int e) {
    constexpr int t[kVar] = {L::A + 8,  L::A + 12, L::A + 9, L::A + 13, L::B + 0, L::B + 4, L::B + 1, L::B + 5,
                             L::Q + 0,  L::Q + 1,  L::Q + 4, L::Q + 5,  L::Q + 10, L::Q + 15, L::R + 0, L::R + 3,
                             L::q + 0,  L::q + 1,  L::q + 2, L::q + 3,  L::r + 0,  L::r + 1};
    return t[e];
  }
  __host__ __device__ static constexpr bool is_var(int k) {
    for (int e = 0; e < kVar; ++e)
      if (pos(e) == k) return true;
    return false;
  }
};

// Compact structured records (the batch kernels' layout for diagonal-weight
// unicycle problems): only the kVar variable entries, kCompactStride doubles
// per node, in UniRec order; the constant entries are implied.
constexpr int kCompactStride = 24;
// UniRec::pos as a constant-bank table for runtime entry indices, and its
// inverse over the dense StageLayout<4, 2> offsets (-1: a constant entry).
static __constant__ int kUniPosTab[UniRec::kVar] = {
    UniRec::pos(0),  UniRec::pos(1),  UniRec::pos(2),  UniRec::pos(3),  UniRec::pos(4),  UniRec::pos(5),
    UniRec::pos(6),  UniRec::pos(7),  UniRec::pos(8),  UniRec::pos(9),  UniRec::pos(10), UniRec::pos(11),
    UniRec::pos(12), UniRec::pos(13), UniRec::pos(14), UniRec::pos(15), UniRec::pos(16), UniRec::pos(17),
    UniRec::pos(18), UniRec::pos(19), UniRec::pos(20), UniRec::pos(21)};
__host__ __device__ constexpr int uni_var_of(int k) {
  for (int e = 0; e < UniRec::kVar; ++e)
    if (UniRec::pos(e) == k) return e;
  return -1;
}

// Constant value at dense offset k of a non-leaf structured record.
__device__ __forceinline__ double unicycle_stage_constant(double dt, int k) {
  using L = StageLayout<4, 2>;
  const double s6 = dt / 6.0;
  if (k < L::B) return ((k - L::A) % 5 == 0) ? 1.0 : 0.0;
  if (k == L::B + 3 || k == L::B + 6) return s6 * (((1.0 + 2.0 * 1.0) + 2.0 * 1.0) + 1.0);
  if (k == L::B + 2 || k == L::B + 7) return s6 * (((0.0 + 2.0 * 0.0) + 2.0 * 0.0) + 0.0);
  return 0.0;
}

// Dense A (4x4) and B (4x2) of a structured record from its variable entries.
__device__ __forceinline__ void unicycle_load_AB(const double* rec, double dt, double* A, double* B) {
  using L = StageLayout<4, 2>;
#pragma unroll
  for (int k = 0; k < 16; ++k) A[k] = UniRec::is_var(L::A + k) ? rec[L::A + k] : unicycle_stage_constant(dt, L::A + k);
#pragma unroll
  for (int k = 0; k < 8; ++k) B[k] = UniRec::is_var(L::B + k) ? rec[L::B + k] : unicycle_stage_constant(dt, L::B + k);
}

// The constant entries of a structured record (exactly what the dense path writes there).
__device__ __forceinline__ void unicycle_stage_constants(double dt, bool leaf, double* rec) {
  using L = StageLayout<4, 2>;
  const double s6 = dt / 6.0;
  const double sel = s6 * (((1.0 + 2.0 * 1.0) + 2.0 * 1.0) + 1.0);
  const double bz = s6 * (((0.0 + 2.0 * 0.0) + 2.0 * 0.0) + 0.0);
#pragma unroll
  for (int k = 0; k < L::size; ++k) {
    if (UniRec::is_var(k)) continue;
    if (leaf && (k < L::Q || k >= L::R) && !(k >= L::q && k < L::r)) continue;  // leaves: Q, q only
    double v = 0.0;
    if (k < L::B) v = ((k - L::A) % 5 == 0) ? 1.0 : 0.0;
    else if (k == L::B + 3 || k == L::B + 6) v = sel;
    else if (k == L::B + 2 || k == L::B + 7) v = bz;
    rec[k] = v;
  }
}

// Variable entries v[UniRec::kVar] of a node's structured record; returns false
// on a non-finite expansion (the constants are finite).
__device__ __forceinline__ bool unicycle_linearize_structured(const ModelParams& mp, int node, bool leaf, double w,
                                                              const double* x, const double* u, const double* eta,
                                                              double rho, double* v) {
  const double* ref = mp.reference + static_cast<long long>(node) * 4;
  const double* W = leaf ? mp.Wf : mp.Wx;
  double q[4], Q[4];  // diagonal of Q
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    Q[i] = W[5 * i];
    q[i] = W[5 * i] * (x[i] - ref[i]);
  }
  // Distance rows: Jx(m, 0..1) = -(dx, dy) / dist; q += Jx' lam, Q(0..1, 0..1) += Jx' diag(as) Jx.
  const int nb = leaf ? 0 : 4;
  const double* vp = mp.vehicles + static_cast<long long>(node) * mp.nv * 2;
  double sq0 = 0.0, sq1 = 0.0, s00 = 0.0, s10 = 0.0, s01 = 0.0, s11 = 0.0;
#pragma unroll
  for (int vv = 0; vv < kMaxVehicles; ++vv) {
    if (vv < mp.nv) {
      const double dx = x[0] - vp[2 * vv + 0];
      const double dy = x[1] - vp[2 * vv + 1];
      const double dist = sqrt(dx * dx + dy * dy + 1e-6);
      const double g = mp.radius - dist;
      const double e = eta[nb + vv];
      const double as = (g >= 0.0 || e > 0.0) ? rho : 0.0;
      const double lam = e + as * g;
      const double j0 = -dx / dist, j1 = -dy / dist;
      sq0 = fma(j0, lam, sq0);
      sq1 = fma(j1, lam, sq1);
      s00 = fma(j0 * as, j0, s00);
      s10 = fma(j1 * as, j0, s10);
      s01 = fma(j0 * as, j1, s01);
      s11 = fma(j1 * as, j1, s11);
    }
  }
  v[8] = w * (Q[0] + s00);
  v[9] = w * (0.0 + s10);
  v[10] = w * (0.0 + s01);
  v[11] = w * (Q[1] + s11);
  v[12] = w * (Q[2] + 0.0);
  v[13] = w * (Q[3] + 0.0);
  v[16] = w * (q[0] + sq0);
  v[17] = w * (q[1] + sq1);
  v[18] = w * (q[2] + 0.0);
  v[19] = w * (q[3] + 0.0);
  bool ok = true;
#pragma unroll
  for (int e = 8; e < 20; ++e)
    if (e < 14 || e >= 16) ok = ok && isfinite(v[e]);
  if (leaf) return ok;
  // Box rows [a - amax, -a - amax, w - wmax, -w - wmax]: Ju = (+1, -1) on u0, u1.
  double as[4], lam[4];
  {
    const double g[4] = {u[0] - mp.a_max, -u[0] - mp.a_max, u[1] - mp.w_max, -u[1] - mp.w_max};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      as[m] = (g[m] >= 0.0 || eta[m] > 0.0) ? rho : 0.0;
      lam[m] = eta[m] + as[m] * g[m];
    }
  }
  double r0 = mp.Wu[0] * u[0], r1 = mp.Wu[3] * u[1];
  r0 += fma(-1.0, lam[1], fma(1.0, lam[0], 0.0));
  r1 += fma(-1.0, lam[3], fma(1.0, lam[2], 0.0));
  v[14] = w * (mp.Wu[0] + fma(-as[1], -1.0, fma(as[0], 1.0, 0.0)));
  v[15] = w * (mp.Wu[3] + fma(-as[3], -1.0, fma(as[2], 1.0, 0.0)));
  v[20] = w * r0;
  v[21] = w * r1;
  // Jacobians (unicycle_step_jacobians_sparse, variable entries only).
  {
    const double dt = mp.dt, hdt = 0.5 * dt;
    const double psi2 = x[2] + hdt * u[1], v2 = x[3] + hdt * u[0];
    const double psi4 = x[2] + dt * u[1], v4 = x[3] + dt * u[0];
    double s1, c1, s2, c2, s4, c4;
    sincos(x[2], &s1, &c1);
    sincos(psi2, &s2, &c2);
    sincos(psi4, &s4, &c4);
    const double j1[4] = {-x[3] * s1, c1, x[3] * c1, s1};
    const double j2[4] = {-v2 * s2, c2, v2 * c2, s2};
    const double j4[4] = {-v4 * s4, c4, v4 * c4, s4};
    const double s6 = dt / 6.0;
    // v[0..3] = A(0,2) A(0,3) A(1,2) A(1,3); j index e = 2r + (c - 2).
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = 0.0 + s6 * (((j1[e] + 2.0 * j2[e]) + 2.0 * j2[e]) + j4[e]);
    // v[4..7] = B(0,0) B(0,1) B(1,0) B(1,1): column 0 uses J(r,3), column 1 J(r,2).
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int cu = 0; cu < 2; ++cu) {
        const int e = 2 * r + (cu == 0 ? 1 : 0);
        const double d2 = j2[e] * hdt, d3 = j2[e] * hdt, d4 = j4[e] * dt;
        v[4 + 2 * r + cu] = s6 * (((0.0 + 2.0 * d2) + 2.0 * d3) + d4);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) ok = ok && isfinite(v[e]);
#pragma unroll
  for (int e = 14; e < 16; ++e) ok = ok && isfinite(v[e]);
  return ok && isfinite(v[20]) && isfinite(v[21]);
}

// linearize (solver.hpp:76-136) of one node: weighted, AL-augmented
// Gauss-Newton stage record (non-leaf) or terminal (P, p) in the Q/q slots.
// Returns false on a non-finite expansion.
// compact: structured records in the compact layout (kCompactStride, UniRec order).
template <int NX, int NU>
__device__ __forceinline__ bool node_linearize(const ModelParams& mp, int node, bool leaf, double w, const double* x,
                                               const double* u, const double* eta, double rho, double* rec,
                                               bool compact = false) {
  using L = StageLayout<NX, NU>;
  if constexpr (NX == 4 && NU == 2) {
    if (mp.kind == kModelUnicycle && mp.w_diag) {  // constants written once per solve (or implied)
      double v[UniRec::kVar];
      const bool ok = unicycle_linearize_structured(mp, node, leaf, w, x, u, eta, rho, v);
#pragma unroll
      for (int e = 0; e < UniRec::kVar; ++e)
        if (!leaf || (e >= 8 && e < 14) || (e >= 16 && e < 20)) rec[compact ? e : UniRec::pos(e)] = v[e];
      return ok;
    }
    if (mp.kind == kModelUnicycle) {
      const double* ref = mp.reference + static_cast<long long>(node) * 4;
      double e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = x[i] - ref[i];
      double g[kMaxCon], Jx[kMaxCon * 4], Ju[kMaxCon * 2];  // row-major Jacobians
      const int nc = ego_constraints<true>(mp, node, leaf, x, u, g, Jx, Ju);
      double as[kMaxCon], lam[kMaxCon];
#pragma unroll
      for (int m = 0; m < kMaxCon; ++m) {
        as[m] = (m < nc && (g[m] >= 0.0 || eta[m] > 0.0)) ? rho : 0.0;
        lam[m] = m < nc ? eta[m] + as[m] * g[m] : 0.0;
      }
      double Q[16], q[4];
      const double* W = leaf ? mp.Wf : mp.Wx;
      copy<16>(W, Q);
      mv<4, 4>(W, e, q);
      // q += Jx' lam ; Q += (Jx' diag(as)) Jx
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxCon; ++m) s = fma(Jx[m * 4 + i], lam[m], s);
        q[i] += s;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < kMaxCon; ++m) s = fma(Jx[m * 4 + i] * as[m], Jx[m * 4 + j], s);
          Q[i + 4 * j] += s;
        }
      }
      bool ok = true;
      if (leaf) {
#pragma unroll
        for (int i = 0; i < 16; ++i) rec[L::Q + i] = w * Q[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) rec[L::q + i] = w * q[i];
        ok = all_finite<16>(rec + L::Q) && all_finite<4>(rec + L::q);
        return ok;
      }
      double R[4], M[8], r[2];
      copy<4>(mp.Wu, R);
      mv<2, 2>(mp.Wu, u, r);
#pragma unroll
      for (int i = 0; i < 8; ++i) M[i] = 0.0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxCon; ++m) s = fma(Ju[m * 2 + i], lam[m], s);
        r[i] += s;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < kMaxCon; ++m) s = fma(Ju[m * 2 + i] * as[m], Ju[m * 2 + j], s);
          R[i + 2 * j] += s;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < kMaxCon; ++m) s = fma(Ju[m * 2 + i] * as[m], Jx[m * 4 + j], s);
          M[i + 2 * j] += s;
        }
      }
      unicycle_step_jacobians_sparse(x, u, mp.dt, rec + L::A, rec + L::B);
#pragma unroll
      for (int i = 0; i < 16; ++i) rec[L::Q + i] = w * Q[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) rec[L::R + i] = w * R[i];
#pragma unroll
      for (int i = 0; i < 8; ++i) rec[L::M + i] = w * M[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) rec[L::q + i] = w * q[i];
#pragma unroll
      for (int i = 0; i < 2; ++i) rec[L::r + i] = w * r[i];
      ok = all_finite<16>(rec + L::A) && all_finite<8>(rec + L::B) && all_finite<16>(rec + L::Q) &&
           all_finite<4>(rec + L::R) && all_finite<4>(rec + L::q) && all_finite<2>(rec + L::r);
      return ok;
    }
  }
  // Affine-quadratic: expansion is point-independent except the gradients.
  if (leaf) {
    const double* l = mp.lq_leaf + static_cast<long long>(node) * (NX * NX + NX);
    double Px[NX];
    mv<NX, NX>(l, x, Px);
#pragma unroll
    for (int i = 0; i < NX * NX; ++i) rec[L::Q + i] = w * l[i];
#pragma unroll
    for (int i = 0; i < NX; ++i) rec[L::q + i] = w * (Px[i] + l[NX * NX + i]);
    return all_finite<NX * NX>(rec + L::Q) && all_finite<NX>(rec + L::q);
  }
  using S = LqStage<NX, NU>;
  const double* s = mp.lq_stage + static_cast<long long>(node) * S::size;
  double Qx[NX], Mtu[NX], Ru[NU], Mx[NU];
  mv<NX, NX>(s + S::Q, x, Qx);
  mtv<NX, NU>(s + S::M, u, Mtu);
  mv<NU, NU>(s + S::R, u, Ru);
  mv<NU, NX>(s + S::M, x, Mx);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) rec[L::A + i] = s[S::A + i];
#pragma unroll
  for (int i = 0; i < NX * NU; ++i) rec[L::B + i] = s[S::B + i];
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) rec[L::Q + i] = w * s[S::Q + i];
#pragma unroll
  for (int i = 0; i < NU * NU; ++i) rec[L::R + i] = w * s[S::R + i];
#pragma unroll
  for (int i = 0; i < NU * NX; ++i) rec[L::M + i] = w * s[S::M + i];
#pragma unroll
  for (int i = 0; i < NX; ++i) rec[L::q + i] = w * ((Qx[i] + s[S::q + i]) + Mtu[i]);
#pragma unroll
  for (int i = 0; i < NU; ++i) rec[L::r + i] = w * ((Ru[i] + s[S::r + i]) + Mx[i]);
  return all_finite<L::size>(rec);
}

// Constraint values only (multiplier update, solver.hpp:764-769).
template <int NX, int NU>
__device__ __forceinline__ int node_constraints(const ModelParams& mp, int node, bool leaf, const double* x,
                                                const double* u, double* g) {
  if constexpr (NX == 4 && NU == 2) {
    if (mp.kind == kModelUnicycle) return ego_constraints<false>(mp, node, leaf, x, u, g, nullptr, nullptr);
  }
  return 0;
}

}  // namespace bmpc_b200
