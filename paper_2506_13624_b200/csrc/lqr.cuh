// LQR-tree building blocks on device: stage records, the dual conditional
// value-function scan element and its associative combination, the tree
// Bellman step at branch nodes, feedback extraction, and the affine forward
// maps. Each function restates one reference routine (cited) with fixed-size
// register arithmetic; error conditions the reference signals with
// exceptions are returned as codes so the device solve loop can take the same
// branch (Levenberg escalation) the reference's catch sites take.
#pragma once

#include "linalg.cuh"

namespace bmpc_b200 {

enum BwdError : int { kBwdOk = 0, kIndefinite = 1, kFactorization = 2 };

// Per-node stage record (reference StageModel, types.hpp:28-40, minus the
// offset c, which lives per child edge as in TreeStageModels,
// riccati.hpp:77-84). Leaves store their terminal (P, p) in the Q / q slots.
template <int NX, int NU>
struct StageLayout {
  static constexpr int A = 0;
  static constexpr int B = A + NX * NX;
  static constexpr int Q = B + NX * NU;
  static constexpr int R = Q + NX * NX;
  static constexpr int M = R + NU * NU;
  static constexpr int q = M + NU * NX;
  static constexpr int r = q + NX;
  static constexpr int size = r + NU;
  static constexpr int stride = (size + 1) & ~1;  // 16-byte aligned records
};

// ScanElementBwd (lqr_scan.hpp:15-24): P, p, C, A, c.
template <int NX>
struct BwdLayout {
  static constexpr int P = 0;
  static constexpr int p = P + NX * NX;
  static constexpr int C = p + NX;
  static constexpr int A = C + NX * NX;
  static constexpr int c = A + NX * NX;
  static constexpr int size = c + NX;
  static constexpr int stride = (size + 1) & ~1;
};

// ScanElementFwd (lqr_scan.hpp:160-163): A, c.
template <int NX>
struct FwdLayout {
  static constexpr int A = 0;
  static constexpr int c = NX * NX;
  static constexpr int size = NX * NX + NX;
  static constexpr int stride = (size + 1) & ~1;
};

template <int NX>
struct ValueLayout {  // ValueFunction (types.hpp:43-50)
  static constexpr int P = 0;
  static constexpr int p = NX * NX;
  static constexpr int stride = (NX * NX + NX + 1) & ~1;
};

template <int NX, int NU>
struct PolicyLayout {  // FeedbackPolicy (types.hpp:53-56)
  static constexpr int K = 0;
  static constexpr int k = NU * NX;
  static constexpr int stride = (NU * NX + NU + 1) & ~1;
};

// init_bwd_element (lqr_scan.hpp:28-49) for stage `s` (R already carrying the
// Levenberg shift `reg`, solver.hpp:212-222) with offset `c`.
template <int NX, int NU>
__device__ int init_bwd_element(const double* s, double reg, const double* c, double* e) {
  using L = StageLayout<NX, NU>;
  using E = BwdLayout<NX>;
  double R[NU * NU];
  copy<NU * NU>(s + L::R, R);
#pragma unroll
  for (int i = 0; i < NU; ++i) R[i + i * NU] += reg;
  Ldlt<NU> f;
  f.compute(R);
  if (!f.positive()) return kFactorization;
  double RiMt[NU * NX];  // R^-1 M
  copy<NU * NX>(s + L::M, RiMt);
  f.template solve<NX>(RiMt);
  double RiBt[NU * NX];  // R^-1 B'
#pragma unroll
  for (int j = 0; j < NX; ++j) {
#pragma unroll
    for (int i = 0; i < NU; ++i) RiBt[i + j * NU] = s[L::B + j + i * NX];
  }
  f.template solve<NX>(RiBt);
  double Rir[NU];
  copy<NU>(s + L::r, Rir);
  f.template solve<1>(Rir);

  double tmp[NX * NX];
  // P = Q - M' R^-1 M
  mtm<NX, NU, NX>(s + L::M, RiMt, tmp);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) e[E::P + i] = s[L::Q + i] - tmp[i];
  // p = q - M' R^-1 r
  double v[NX];
  mtv<NX, NU>(s + L::M, Rir, v);
#pragma unroll
  for (int i = 0; i < NX; ++i) e[E::p + i] = s[L::q + i] - v[i];
  // C = B R^-1 B'
  mm<NX, NU, NX>(s + L::B, RiBt, tmp);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) e[E::C + i] = tmp[i];
  // A = A - B R^-1 M
  mm<NX, NU, NX>(s + L::B, RiMt, tmp);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) e[E::A + i] = s[L::A + i] - tmp[i];
  // c = c - B R^-1 r
  mv<NX, NU>(s + L::B, Rir, v);
#pragma unroll
  for (int i = 0; i < NX; ++i) e[E::c + i] = c[i] - v[i];
  symmetrize<NX>(e + E::P);
  symmetrize<NX>(e + E::C);
  return kBwdOk;
}

// embed_terminal (lqr_scan.hpp:55-66).
template <int NX>
__device__ void embed_terminal(const double* P, const double* p, double* e) {
  using E = BwdLayout<NX>;
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) {
    e[E::P + i] = P[i];
    e[E::C + i] = 0.0;
    e[E::A + i] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    e[E::p + i] = p[i];
    e[E::c + i] = 0.0;
  }
}

// combine_bwd (lqr_scan.hpp:80-111): out = first (+) second, first = k->j,
// second = j->i. One PartialPivLU of G = I + C1 P2 serves both G^-1 and
// G^-T. Returns kFactorization when any output is non-finite.
template <int NX>
__device__ int combine_bwd(const double* __restrict__ e1, const double* __restrict__ e2, double* __restrict__ out) {
  using E = BwdLayout<NX>;
  double G[NX * NX];
  mm<NX, NX, NX>(e1 + E::C, e2 + E::P, G);
#pragma unroll
  for (int i = 0; i < NX; ++i) G[i + i * NX] += 1.0;
  Lu<NX> lu;
  lu.compute(G);

  double X[NX * NX], Y[NX * NX], v[NX], w[NX];
  bool ok = true;
  // out.A = A2 G^-1 A1
  lu.template solve<NX>(e1 + E::A, X);
  mm<NX, NX, NX>(e2 + E::A, X, Y);
  ok = ok && all_finite<NX * NX>(Y);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) out[E::A + i] = Y[i];
  // out.c = A2 G^-1 (c1 - C1 p2) + c2
  mv<NX, NX>(e1 + E::C, e2 + E::p, v);
#pragma unroll
  for (int i = 0; i < NX; ++i) v[i] = e1[E::c + i] - v[i];
  lu.template solve<1>(v, w);
  mv<NX, NX>(e2 + E::A, w, v);
#pragma unroll
  for (int i = 0; i < NX; ++i) v[i] += e2[E::c + i];
  ok = ok && all_finite<NX>(v);
#pragma unroll
  for (int i = 0; i < NX; ++i) out[E::c + i] = v[i];
  // out.C = (A2 G^-1 C1) A2' + C2
  lu.template solve<NX>(e1 + E::C, X);
  mm<NX, NX, NX>(e2 + E::A, X, Y);
  mmt<NX, NX, NX>(Y, e2 + E::A, X);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) X[i] += e2[E::C + i];
  symmetrize<NX>(X);
  ok = ok && all_finite<NX * NX>(X);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) out[E::C + i] = X[i];
  // out.p = A1' G^-T (p2 + P2 c1) + p1
  mv<NX, NX>(e2 + E::P, e1 + E::c, v);
#pragma unroll
  for (int i = 0; i < NX; ++i) v[i] += e2[E::p + i];
  lu.template solve_transposed<1>(v, w);
  mtv<NX, NX>(e1 + E::A, w, v);
#pragma unroll
  for (int i = 0; i < NX; ++i) v[i] += e1[E::p + i];
  ok = ok && all_finite<NX>(v);
#pragma unroll
  for (int i = 0; i < NX; ++i) out[E::p + i] = v[i];
  // out.P = A1' G^-T (P2 A1) + P1
  mm<NX, NX, NX>(e2 + E::P, e1 + E::A, X);
  lu.template solve_transposed<NX>(X, Y);
  mtm<NX, NX, NX>(e1 + E::A, Y, X);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) X[i] += e1[E::P + i];
  symmetrize<NX>(X);
  ok = ok && all_finite<NX * NX>(X);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) out[E::P + i] = X[i];
  return ok ? kBwdOk : kFactorization;
}

// feedback_from_values (lqr_scan.hpp:146-157): policy at a node from the
// value (P, p) of its single successor and the edge offset c.
template <int NX, int NU>
__device__ int feedback(const double* s, double reg, const double* c, const double* P, const double* p,
                        double* K, double* k) {
  using L = StageLayout<NX, NU>;
  double BtP[NU * NX];
  mtm<NU, NX, NX>(s + L::B, P, BtP);
  double H[NU * NU];
  mm<NU, NX, NU>(BtP, s + L::B, H);
#pragma unroll
  for (int i = 0; i < NU * NU; ++i) H[i] += s[L::R + i];
#pragma unroll
  for (int i = 0; i < NU; ++i) H[i + i * NU] += reg;
  symmetrize<NU>(H);
  Ldlt<NU> f;
  f.compute(H);
  if (!f.positive()) return kIndefinite;
  // K = -H^-1 (M + B'PA)
  double X[NU * NX];
  mm<NU, NX, NX>(BtP, s + L::A, X);
#pragma unroll
  for (int i = 0; i < NU * NX; ++i) X[i] += s[L::M + i];
  f.template solve<NX>(X);
#pragma unroll
  for (int i = 0; i < NU * NX; ++i) K[i] = -X[i];
  // k = -H^-1 (r + B'(p + P c))
  double pc[NX];
  mv<NX, NX>(P, c, pc);
#pragma unroll
  for (int i = 0; i < NX; ++i) pc[i] += p[i];
  double y[NU];
  mtv<NU, NX>(s + L::B, pc, y);
#pragma unroll
  for (int i = 0; i < NU; ++i) y[i] += s[L::r + i];
  f.template solve<1>(y);
#pragma unroll
  for (int i = 0; i < NU; ++i) k[i] = -y[i];
  return kBwdOk;
}

// riccati_step (riccati.hpp:22-43) at a branch node, with the continuation
// already aggregated over the children: Pn = sum P_ch, pn = sum (p_ch + P_ch d_ch).
template <int NX, int NU>
__device__ int riccati_step(const double* s, double reg, const double* Pn, const double* pn, double* Pout,
                            double* pout, double* K, double* k) {
  using L = StageLayout<NX, NU>;
  double AtP[NX * NX];
  mtm<NX, NX, NX>(s + L::A, Pn, AtP);
  double Qxx[NX * NX];
  mm<NX, NX, NX>(AtP, s + L::A, Qxx);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) Qxx[i] += s[L::Q + i];
  double BtP[NU * NX];
  mtm<NU, NX, NX>(s + L::B, Pn, BtP);
  double Quu[NU * NU];
  mm<NU, NX, NU>(BtP, s + L::B, Quu);
#pragma unroll
  for (int i = 0; i < NU * NU; ++i) Quu[i] += s[L::R + i];
#pragma unroll
  for (int i = 0; i < NU; ++i) Quu[i + i * NU] += reg;
  double Qux[NU * NX];
  mm<NU, NX, NX>(BtP, s + L::A, Qux);
#pragma unroll
  for (int i = 0; i < NU * NX; ++i) Qux[i] += s[L::M + i];
  double qx[NX];
  mtv<NX, NX>(s + L::A, pn, qx);
#pragma unroll
  for (int i = 0; i < NX; ++i) qx[i] += s[L::q + i];
  double qu[NU];
  mtv<NU, NX>(s + L::B, pn, qu);
#pragma unroll
  for (int i = 0; i < NU; ++i) qu[i] += s[L::r + i];
  symmetrize<NU>(Quu);
  Ldlt<NU> f;
  f.compute(Quu);
  if (!f.positive()) return kIndefinite;
  double X[NU * NX];
  copy<NU * NX>(Qux, X);
  f.template solve<NX>(X);
#pragma unroll
  for (int i = 0; i < NU * NX; ++i) K[i] = -X[i];
  double y[NU];
  copy<NU>(qu, y);
  f.template solve<1>(y);
#pragma unroll
  for (int i = 0; i < NU; ++i) k[i] = -y[i];
  // P = Qxx + Qux' K ; p = qx + Qux' k
  double T[NX * NX];
  mtm<NX, NU, NX>(Qux, K, T);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) Pout[i] = Qxx[i] + T[i];
  double t[NX];
  mtv<NX, NU>(Qux, k, t);
#pragma unroll
  for (int i = 0; i < NX; ++i) pout[i] = qx[i] + t[i];
  symmetrize<NX>(Pout);
  return kBwdOk;
}

// init_fwd_element (lqr_scan.hpp:166-168): (A + B K, c + B k).
template <int NX, int NU>
__device__ void init_fwd_element(const double* s, const double* c, const double* K, const double* k, double* f) {
  using L = StageLayout<NX, NU>;
  using F = FwdLayout<NX>;
  double BK[NX * NX];
  mm<NX, NU, NX>(s + L::B, K, BK);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) f[F::A + i] = s[L::A + i] + BK[i];
  double Bk[NX];
  mv<NX, NU>(s + L::B, k, Bk);
#pragma unroll
  for (int i = 0; i < NX; ++i) f[F::c + i] = c[i] + Bk[i];
}

// ---------------------------------------------------------------------------
// Team-cooperative combine_bwd: TS lanes (TS >= NX*NX, a power of two <= 32)
// compute one combination, lane l owning entry (l % NX, l / NX) of every NX x
// NX block. Operands are staged in shared memory (conflict-free column-major
// reads), G = I + C1 P2 is inverted once (every lane factors it redundantly
// in registers, then produces its own entry of G^-1), and the five update
// formulas of lqr_scan.hpp:68-97 become small matrix products:
//   A = A2 (G^-1 A1),  C = (A2 (G^-1 C1)) A2' + C2,  c = A2 G^-1 (c1 - C1 p2) + c2,
//   P = A1' (G^-T (P2 A1)) + P1,  p = A1' G^-T (p2 + P2 c1) + p1.
// P and C are formed symmetric directly (each lane evaluates its (i,j) and
// (j,i) entries, the reference's symmetrize). Latency ~7 short stages
// instead of one thread's ~1.5 kflop dependent chain. `out` may alias e1/e2.
template <int NX>
struct TeamSmem {
  double e1[BwdLayout<NX>::size], e2[BwdLayout<NX>::size];
  double G[NX * NX], GI[NX * NX], X[NX * NX], W[NX * NX], Y[NX * NX], Z[NX * NX], T[NX * NX];
  double v[NX], v2[NX], w[NX], w2[NX];
};

template <int NX, int TS>
__device__ int team_combine_bwd(const double* e1g, const double* e2g, double* out, int lane, unsigned mask,
                                TeamSmem<NX>& sm) {
  using E = BwdLayout<NX>;
  constexpr int N2 = NX * NX;
  static_assert(TS >= N2 && TS <= 32, "team too small");
  // Stage the operands.
  for (int k = lane; k < E::size; k += TS) {
    sm.e1[k] = e1g[k];
    sm.e2[k] = e2g[k];
  }
  __syncwarp(mask);
  const int i = lane % NX, j = lane / NX;
  const bool act = lane < N2;
  // G = I + C1 P2 ; vector pre-terms v = c1 - C1 p2, v2 = p2 + P2 c1.
  if (act) {
    double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) s = fma(sm.e1[E::C + i + l * NX], sm.e2[E::P + l + j * NX], s);
    sm.G[lane] = s;
  }
  if (lane < NX) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      a = fma(sm.e1[E::C + lane + l * NX], sm.e2[E::p + l], a);
      b = fma(sm.e2[E::P + lane + l * NX], sm.e1[E::c + l], b);
    }
    sm.v[lane] = sm.e1[E::c + lane] - a;
    sm.v2[lane] = b + sm.e2[E::p + lane];
  }
  __syncwarp(mask);
  // G^-1: redundant register LU per lane, lane (i, j) keeps entry (i, j).
  if (act) {
    Lu<NX> lu;
    lu.compute(sm.G);
    double ej[NX], col[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) ej[r] = (r == j) ? 1.0 : 0.0;
    lu.template solve<1>(ej, col);
    double g = col[0];
#pragma unroll
    for (int r = 1; r < NX; ++r) g = (r == i) ? col[r] : g;
    sm.GI[lane] = g;
  }
  __syncwarp(mask);
  // X = G^-1 A1, W = G^-1 C1, Z = P2 A1 ; w = G^-1 v, w2 = G^-T v2.
  if (act) {
    double x = 0.0, wv = 0.0, z = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      const double gil = sm.GI[i + l * NX];
      x = fma(gil, sm.e1[E::A + l + j * NX], x);
      wv = fma(gil, sm.e1[E::C + l + j * NX], wv);
      z = fma(sm.e2[E::P + i + l * NX], sm.e1[E::A + l + j * NX], z);
    }
    sm.X[lane] = x;
    sm.W[lane] = wv;
    sm.Z[lane] = z;
  }
  if (lane < NX) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      a = fma(sm.GI[lane + l * NX], sm.v[l], a);
      b = fma(sm.GI[l + lane * NX], sm.v2[l], b);
    }
    sm.w[lane] = a;
    sm.w2[lane] = b;
  }
  __syncwarp(mask);
  // A_out = A2 X ; Y = A2 W ; T = G^-T Z ; c_out, p_out.
  bool ok = true;
  double a_out = 0.0, c_out = 0.0, p_out = 0.0;
  if (act) {
    double y = 0.0, tt = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      const double a2il = sm.e2[E::A + i + l * NX];
      a_out = fma(a2il, sm.X[l + j * NX], a_out);
      y = fma(a2il, sm.W[l + j * NX], y);
      tt = fma(sm.GI[l + i * NX], sm.Z[l + j * NX], tt);
    }
    sm.Y[lane] = y;
    sm.T[lane] = tt;
  }
  if (lane < NX) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      a = fma(sm.e2[E::A + lane + l * NX], sm.w[l], a);
      b = fma(sm.e1[E::A + l + lane * NX], sm.w2[l], b);
    }
    c_out = a + sm.e2[E::c + lane];
    p_out = b + sm.e1[E::p + lane];
  }
  __syncwarp(mask);
  // C_out = Y A2' + C2 and P_out = A1' T + P1, symmetrized entrywise.
  double C_out = 0.0, P_out = 0.0;
  if (act) {
    double cij = 0.0, cji = 0.0, pij = 0.0, pji = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      cij = fma(sm.Y[i + l * NX], sm.e2[E::A + j + l * NX], cij);
      cji = fma(sm.Y[j + l * NX], sm.e2[E::A + i + l * NX], cji);
      pij = fma(sm.e1[E::A + l + i * NX], sm.T[l + j * NX], pij);
      pji = fma(sm.e1[E::A + l + j * NX], sm.T[l + i * NX], pji);
    }
    cij += sm.e2[E::C + lane];
    cji += sm.e2[E::C + j + i * NX];
    pij += sm.e1[E::P + lane];
    pji += sm.e1[E::P + j + i * NX];
    C_out = 0.5 * (cij + cji);
    P_out = 0.5 * (pij + pji);
    ok = isfinite(a_out) && isfinite(C_out) && isfinite(P_out);
  }
  if (lane < NX) ok = ok && isfinite(c_out) && isfinite(p_out);
  // `out` may alias e1g / e2g or the staged operands themselves (sm.e2, the
  // chunked scan's accumulator): every lane finishes its reads first.
  __syncwarp(mask);
  if (act) {
    out[E::A + lane] = a_out;
    out[E::C + lane] = C_out;
    out[E::P + lane] = P_out;
  }
  if (lane < NX) {
    out[E::c + lane] = c_out;
    out[E::p + lane] = p_out;
  }
  // Per-lane status: the callers fold error codes with a max over every
  // thread, so the team needs no vote here.
  __syncwarp(mask);
  return ok ? kBwdOk : kFactorization;
}

// combine_fwd (lqr_scan.hpp:171-173): (A2 A1, A2 c1 + c2).
template <int NX>
__device__ void combine_fwd(const double* f1, const double* f2, double* out) {  // out may alias f2
  using F = FwdLayout<NX>;
  double A[NX * NX], c[NX];
  mm<NX, NX, NX>(f2 + F::A, f1 + F::A, A);
  mv<NX, NX>(f2 + F::A, f1 + F::c, c);
#pragma unroll
  for (int i = 0; i < NX; ++i) c[i] += f2[F::c + i];
  copy<NX * NX>(A, out + F::A);
  copy<NX>(c, out + F::c);
}

// ---------------------------------------------------------------------------
// Team-cooperative sequential Riccati sweep along one segment (short
// segments, where the O(L) recursion beats the O(L log L)-work scan). One
// step is riccati_step (riccati.hpp:22-43) with the continuation (P, p + P c)
// of the successor — for single-child nodes exactly feedback_from_values
// (lqr_scan.hpp:146-157) plus the value update; for a branch node the summed
// children (riccati.hpp:112-116). TS lanes, entries distributed as in
// team_combine_bwd; (P, p) stay in shared memory between steps.
template <int NX, int NU>
struct RicSmem {
  double s[StageLayout<NX, NU>::size];
  double P[NX * NX], p[NX], c[NX], psh[NX];
  double BtP[NU * NX], AtP[NX * NX], Qxx[NX * NX], Quu[NU * NU], Qux[NU * NX], qx[NX], qu[NU];
  double K[NU * NX], k[NU];
};

// Loads the stage record of `node` and the edge offset c (nullptr: zero).
template <int NX, int NU, int TS>
__device__ __forceinline__ void ric_load(const double* stage_g, const double* c_g, int lane, RicSmem<NX, NU>& sm) {
  using L = StageLayout<NX, NU>;
  for (int t = lane; t < L::size; t += TS) sm.s[t] = stage_g[t];
  if (lane < NX) sm.c[lane] = c_g ? c_g[lane] : 0.0;
}

// One Bellman step on the staged stage/c/(P, p); overwrites (P, p) with the
// node's value and writes value / policy to global memory. Returns an error
// code (kIndefinite when R + B'PB is not positive definite).
template <int NX, int NU, int TS>
__device__ int team_riccati_step(double reg, int lane, unsigned mask, RicSmem<NX, NU>& sm, double* V_g, double* K_g,
                                 double* k_g) {
  using L = StageLayout<NX, NU>;
  constexpr int N2 = NX * NX;
  const double* s = sm.s;
  __syncwarp(mask);
  // p_shifted = p + P c ; B'P ; A'P
  if (lane < NX) {
    double a = sm.p[lane];
#pragma unroll
    for (int l = 0; l < NX; ++l) a = fma(sm.P[lane + l * NX], sm.c[l], a);
    sm.psh[lane] = a;
  }
  if (lane < NU * NX) {
    const int a = lane % NU, j = lane / NU;
    double v = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(s[L::B + l + a * NX], sm.P[l + j * NX], v);
    sm.BtP[lane] = v;
  }
  if (lane < N2) {
    const int i = lane % NX, j = lane / NX;
    double v = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(s[L::A + l + i * NX], sm.P[l + j * NX], v);
    sm.AtP[lane] = v;
  }
  __syncwarp(mask);
  // Qxx, Quu (+reg), Qux, qx, qu
  if (lane < N2) {
    const int i = lane % NX, j = lane / NX;
    double v = s[L::Q + lane];
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(sm.AtP[i + l * NX], s[L::A + l + j * NX], v);
    sm.Qxx[lane] = v;
  }
  if (lane < NU * NX) {
    const int a = lane % NU, j = lane / NU;
    double v = s[L::M + lane];
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(sm.BtP[a + l * NU], s[L::A + l + j * NX], v);
    sm.Qux[lane] = v;
  }
  if (lane < NU * NU) {
    const int a = lane % NU, b = lane / NU;
    double v = s[L::R + lane] + (a == b ? reg : 0.0);
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(sm.BtP[a + l * NU], s[L::B + l + b * NX], v);
    sm.Quu[lane] = v;
  }
  if (lane < NX) {
    double v = s[L::q + lane];
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(s[L::A + l + lane * NX], sm.psh[l], v);
    sm.qx[lane] = v;
  }
  if (lane < NU) {
    double v = s[L::r + lane];
#pragma unroll
    for (int l = 0; l < NX; ++l) v = fma(s[L::B + l + lane * NX], sm.psh[l], v);
    sm.qu[lane] = v;
  }
  __syncwarp(mask);
  // Huu = sym(Quu); LDLT; K = -Huu^-1 Qux, k = -Huu^-1 qu (every lane factors).
  bool pos;
  {
    double H[NU * NU];
#pragma unroll
    for (int t = 0; t < NU * NU; ++t) H[t] = sm.Quu[t];
    symmetrize<NU>(H);
    Ldlt<NU> f;
    f.compute(H);
    pos = f.positive();
    if (lane < NU * NX) {
      const int a = lane % NU, j = lane / NU;
      double col[NU];
#pragma unroll
      for (int t = 0; t < NU; ++t) col[t] = sm.Qux[t + j * NU];
      f.template solve<1>(col);
      double v = col[0];
#pragma unroll
      for (int t = 1; t < NU; ++t) v = (t == a) ? col[t] : v;
      sm.K[lane] = -v;
      if (K_g) K_g[lane] = -v;
    }
    if (lane >= NU * NX && lane < NU * NX + NU) {
      const int a = lane - NU * NX;
      double col[NU];
#pragma unroll
      for (int t = 0; t < NU; ++t) col[t] = sm.qu[t];
      f.template solve<1>(col);
      double v = col[0];
#pragma unroll
      for (int t = 1; t < NU; ++t) v = (t == a) ? col[t] : v;
      sm.k[a] = -v;
      if (k_g) k_g[a] = -v;
    }
  }
  __syncwarp(mask);
  // P = sym(Qxx + Qux' K), p = qx + Qux' k
  double Pij = 0.0, pi = 0.0;
  if (lane < N2) {
    const int i = lane % NX, j = lane / NX;
    double a = sm.Qxx[lane], b = sm.Qxx[j + i * NX];
#pragma unroll
    for (int t = 0; t < NU; ++t) {
      a = fma(sm.Qux[t + i * NU], sm.K[t + j * NU], a);
      b = fma(sm.Qux[t + j * NU], sm.K[t + i * NU], b);
    }
    Pij = 0.5 * (a + b);
  }
  if (lane < NX) {
    double v = sm.qx[lane];
#pragma unroll
    for (int t = 0; t < NU; ++t) v = fma(sm.Qux[t + lane * NU], sm.k[t], v);
    pi = v;
  }
  __syncwarp(mask);
  if (lane < N2) {
    sm.P[lane] = Pij;
    if (V_g) V_g[ValueLayout<NX>::P + lane] = Pij;
  }
  if (lane < NX) {
    sm.p[lane] = pi;
    if (V_g) V_g[ValueLayout<NX>::p + lane] = pi;
  }
  const unsigned bad = __ballot_sync(mask, !pos);
  return bad ? kIndefinite : kBwdOk;
}

// ---------------------------------------------------------------------------
// Divergence-free team Riccati step. Every small product of riccati_step is a
// "dot slot" out = base (+ reg on a diagonal) + sum_l X[xo + l] Y[yo + l] over
// one flat shared array; each lane owns fixed slots, so all lanes run one
// instruction stream per stage (4 stages + the redundant NU x NU LDLT).
// Every operand is laid out contiguous (P also as its transpose PT, B'P and
// A'P row-major), so both operands stream with unit stride and, for even NX,
// as 16-byte vector loads at even offsets. The products and their order are
// those of the reference's dense riccati_step.
template <int NX, int NU>
struct RicFlat {  // offsets into the team's flat shared array
  using L = StageLayout<NX, NU>;
  static constexpr int ev(int v) { return (v + 1) & ~1; }
  static constexpr int S = 0, A = L::A, B = L::B, Q = L::Q, R = L::R, M = L::M, q = L::q, r = L::r;
  static constexpr int P = ev(L::size), PT = P + NX * NX, p = ev(PT + NX * NX), c = ev(p + NX), psh = ev(c + NX),
                       BtP = ev(psh + NX),         // row-major NU x NX: BtP[a * NX + l] = (B'P)(a, l)
                       AtP = ev(BtP + NU * NX),    // row-major NX x NX: AtP[i * NX + l] = (A'P)(i, l)
                       Qxx = ev(AtP + NX * NX), Qux = ev(Qxx + NX * NX), Quu = ev(Qux + NU * NX),
                       qx = ev(Quu + NU * NU), qu = ev(qx + NX), K = ev(qu + NU), k = ev(K + NU * NX),
                       ZERO = ev(k + NU), DUMMY = ZERO + ev(NX), size = DUMMY + 8;
  static constexpr int n1 = NX + NU * NX + NX * NX;                  // psh, B'P, A'P
  static constexpr int n2 = NX * NX + NU * NX + NX + NU;             // Qxx, Qux, qx, qu (Quu: every lane)
  static constexpr int n3 = NU * NX + NU;                            // K, k
  static constexpr int n4 = NX * NX + NX;                            // P, p
  static constexpr bool kVec = NX % 2 == 0;  // all X / Y operand offsets even
};

// P(i, j) (column-major index k = i + NX j) and its transposed copy.
template <int NX, int NU>
__device__ __forceinline__ void ric_put_P(double* Fm, int k, double v) {
  using F = RicFlat<NX, NU>;
  Fm[F::P + k] = v;
  Fm[F::PT + (k % NX) * NX + k / NX] = v;
}

struct DotSlot {
  short bo, xo, yo, oo;
  bool diag;  // add the Levenberg shift (Quu diagonal)
};

// Slot descriptors computed on the fly from the lane index (integer selects
// only), so no per-lane descriptor state stays live across the sweep.
template <int NX, int NU>
__device__ __forceinline__ DotSlot ric_slot1(int q) {
  using F = RicFlat<NX, NU>;
  if (q < NX) return {short(F::p + q), short(F::PT + q * NX), F::c, short(F::psh + q), false};  // psh = p + P c
  if (q < NX + NU * NX) {  // B'P (a, j) = B(:, a) . P(:, j)
    const int t = q - NX, a = t / NX, j = t % NX;
    return {F::ZERO, short(F::B + a * NX), short(F::P + j * NX), short(F::BtP + t), false};
  }
  if (q < F::n1) {  // A'P (i, j) = A(:, i) . P(:, j)
    const int t = q - NX - NU * NX, i = t / NX, j = t % NX;
    return {F::ZERO, short(F::A + i * NX), short(F::P + j * NX), short(F::AtP + t), false};
  }
  return {F::ZERO, F::ZERO, F::ZERO, F::DUMMY, false};
}

template <int NX, int NU>
__device__ __forceinline__ DotSlot ric_slot2(int q) {
  using F = RicFlat<NX, NU>;
  if (q < NX * NX) {  // Qxx = Q + A'P A
    const int i = q % NX, j = q / NX;
    return {short(F::Q + q), short(F::AtP + i * NX), short(F::A + j * NX), short(F::Qxx + q), false};
  }
  q -= NX * NX;
  if (q < NU * NX) {  // Qux = M + B'P A
    const int a = q % NU, j = q / NU;
    return {short(F::M + q), short(F::BtP + a * NX), short(F::A + j * NX), short(F::Qux + q), false};
  }
  q -= NU * NX;
  if (q < NX) return {short(F::q + q), short(F::A + q * NX), F::psh, short(F::qx + q), false};  // qx
  q -= NX;
  if (q < NU) return {short(F::r + q), short(F::B + q * NX), F::psh, short(F::qu + q), false};  // qu
  return {F::ZERO, F::ZERO, F::ZERO, F::DUMMY, false};
}

template <int LEN, bool kVec>
__device__ __forceinline__ double dot_slot(const double* Fm, const DotSlot& s, double reg) {
  double a = Fm[s.bo] + (s.diag ? reg : 0.0);
  if constexpr (kVec && LEN % 2 == 0) {
    const double2* X = reinterpret_cast<const double2*>(Fm + s.xo);
    const double2* Y = reinterpret_cast<const double2*>(Fm + s.yo);
#pragma unroll
    for (int l = 0; l < LEN / 2; ++l) {
      const double2 x = X[l], y = Y[l];
      a = fma(x.x, y.x, a);
      a = fma(x.y, y.y, a);
    }
  } else {
#pragma unroll
    for (int l = 0; l < LEN; ++l) a = fma(Fm[s.xo + l], Fm[s.yo + l], a);
  }
  return a;
}

// One Bellman step on the team's flat array (stage, c, P, p staged).
// Overwrites P, p; writes value / policy records. Returns kIndefinite when
// R + B'PB is not positive definite (lqr_scan.hpp:150, riccati.hpp:31-35).
// kStamp (diagnostic): lane 0 accumulates clock64 deltas per stage into st[0..4].
template <int NX, int NU, int TS, bool kStamp = false>
__device__ int team_riccati_step_u(double reg, unsigned mask, double* Fm, int lane, double* V_g, double* pol_g,
                                   unsigned long long* st = nullptr) {
  using F = RicFlat<NX, NU>;
  constexpr int R1 = (F::n1 + TS - 1) / TS, R2 = (F::n2 + TS - 1) / TS, R4 = (F::n4 + TS - 1) / TS;
  long long ck = 0;
  auto stamp = [&](int k) {
    if constexpr (kStamp) {
      const long long now = clock64();
      if (lane == 0 && k > 0) st[k - 1] += now - ck;
      ck = now;
    }
  };
  stamp(0);
  __syncwarp(mask);
  {
    double o[R1];
    short oo[R1];
#pragma unroll
    for (int r = 0; r < R1; ++r) {
      const DotSlot sl = ric_slot1<NX, NU>(lane + r * TS);
      o[r] = dot_slot<NX, F::kVec>(Fm, sl, 0.0);
      oo[r] = sl.oo;
    }
#pragma unroll
    for (int r = 0; r < R1; ++r) Fm[oo[r]] = o[r];
  }
  __syncwarp(mask);
  stamp(1);
  // Huu = sym(Quu), Quu = R (+reg) + B'P B formed by every lane (the same
  // dot-slot arithmetic as a shared slot) and factored here, so the LDLT and
  // Huu^-1 overlap this stage's slots instead of following them.
  double inv[NU * NU];
  bool pos;
  {
    double o[R2];
    short oo[R2];
#pragma unroll
    for (int r = 0; r < R2; ++r) {
      const DotSlot sl = ric_slot2<NX, NU>(lane + r * TS);
      o[r] = dot_slot<NX, F::kVec>(Fm, sl, reg);
      oo[r] = sl.oo;
    }
    double H[NU * NU];
#pragma unroll
    for (int q = 0; q < NU * NU; ++q) {
      const int a = q % NU, b = q / NU;
      const DotSlot sl{short(F::R + q), short(F::BtP + a * NX), short(F::B + b * NX), F::DUMMY, a == b};
      H[q] = dot_slot<NX, F::kVec>(Fm, sl, reg);
    }
#pragma unroll
    for (int r = 0; r < R2; ++r) Fm[oo[r]] = o[r];
    symmetrize<NU>(H);
    Ldlt<NU> f;
    f.compute(H);
    pos = f.positive();
#pragma unroll
    for (int t = 0; t < NU * NU; ++t) inv[t] = (t % (NU + 1) == 0) ? 1.0 : 0.0;
    f.template solve<NU>(inv);
  }
  __syncwarp(mask);
  stamp(2);
  // Operands of this lane's P / p outputs.
  double s4i[R4][NU], s4j[R4][NU], s4a[R4], s4b[R4];
#pragma unroll
  for (int r = 0; r < R4; ++r) {
    const int q = lane + r * TS;
    if (q < NX * NX) {
      const int i = q % NX, j = q / NX;
#pragma unroll
      for (int t = 0; t < NU; ++t) {
        s4i[r][t] = Fm[F::Qux + t + i * NU];
        s4j[r][t] = Fm[F::Qux + t + j * NU];
      }
      s4a[r] = Fm[F::Qxx + q];
      s4b[r] = Fm[F::Qxx + j + i * NX];
    } else {
      const int i = q < F::n4 ? q - NX * NX : 0;
#pragma unroll
      for (int t = 0; t < NU; ++t) {
        s4i[r][t] = Fm[F::Qux + t + i * NU];
        s4j[r][t] = Fm[F::qu + t];
      }
      s4a[r] = Fm[F::qx + i];
      s4b[r] = 0.0;
    }
  }
  // Each lane builds the K / k columns its own outputs need (no shared-memory
  // round trip for K): K(a, j) = -Huu^-1(a, :) Qux(:, j), k(a) = -Huu^-1(a, :) qu.
  auto kcol = [&](const double* v, double* out) {  // out = -Huu^-1 v
#pragma unroll
    for (int a = 0; a < NU; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < NU; ++b) s = fma(inv[a + b * NU], v[b], s);
      out[a] = -s;
    }
  };
  stamp(3);
  double o4[R4];
  short oo4[R4], ot4[R4], g4[R4];
#pragma unroll
  for (int r = 0; r < R4; ++r) {
    const int q = lane + r * TS;
    double a = 0.0, b = 0.0;
    ot4[r] = F::DUMMY;
    if (q < NX * NX) {  // P(i,j) = sym(Qxx + Qux' K)
      const int i = q % NX, j = q / NX;
      ot4[r] = short(F::PT + i * NX + j);
      double Ki[NU], Kj[NU];
      const double* qi = s4i[r];
      const double* qj = s4j[r];
      kcol(qi, Ki);
      kcol(qj, Kj);
      if (pol_g && i == 0) {  // lanes of column 0 of P hold K(:, j): the policy write
#pragma unroll
        for (int t = 0; t < NU; ++t) __stcg(pol_g + PolicyLayout<NX, NU>::K + t + j * NU, Kj[t]);
      }
      a = s4a[r];
      b = s4b[r];
#pragma unroll
      for (int t = 0; t < NU; ++t) {
        a = fma(qi[t], Kj[t], a);
        b = fma(qj[t], Ki[t], b);
      }
      oo4[r] = short(F::P + q);
      g4[r] = short(ValueLayout<NX>::P + q);
    } else if (q < F::n4) {  // p = qx + Qux' k
      const int i = q - NX * NX;
      double kk[NU];
      const double* qi = s4i[r];
      kcol(s4j[r], kk);
      if (pol_g && i == 0) {
#pragma unroll
        for (int t = 0; t < NU; ++t) __stcg(pol_g + PolicyLayout<NX, NU>::k + t, kk[t]);
      }
      a = s4a[r];
#pragma unroll
      for (int t = 0; t < NU; ++t) a = fma(qi[t], kk[t], a);
      b = a;
      oo4[r] = short(F::p + i);
      g4[r] = short(ValueLayout<NX>::p + i);
    } else {
      oo4[r] = F::DUMMY;
      g4[r] = -1;
    }
    o4[r] = 0.5 * (a + b);
  }
  stamp(4);
  // P, p are no longer read in this step (S1/S2 finished behind barriers);
  // the next step opens with a __syncwarp.
#pragma unroll
  for (int r = 0; r < R4; ++r) {
    Fm[oo4[r]] = o4[r];
    Fm[ot4[r]] = o4[r];
    // Explicit global-space stores: a generic store would order the next
    // step's shared-memory loads behind it.
    if (V_g && g4[r] >= 0) __stcg(V_g + g4[r], o4[r]);
  }
  // Every lane factored the same Huu with the same instructions, so `pos`
  // is uniform across the team: no vote needed (the next step opens with a
  // __syncwarp).
  stamp(5);
  return pos ? kBwdOk : kIndefinite;
}

}  // namespace bmpc_b200
