/* bmpc_oracle.c — plain-C restatement of the reference solve path.
 * TEST INFRASTRUCTURE ONLY (see bmpc_oracle.h). Compiled with
 * -ffp-contract=off; every expression keeps the evaluation order the
 * reference's Eigen expressions have under oracle/eigen_shim (products
 * accumulate l = 0..k-1 from 0.0), so results agree with oracle/_ref to
 * rounding level — bitwise wherever the shim's order is reproduced exactly.
 * File:line citations are to /root/reference/proj/include/bmpc.
 */
#include "bmpc_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MX BO_MAXN
#define MX2 (BO_MAXN * BO_MAXN)

/* ------------------------------------------------------------ algebra */
/* out(m x n) = a(m x k) b(k x n), column-major. */
static void mm(int m, int k, int n, const double* a, const double* b, double* out) {
  double t[MX2 * 4];
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[i + l * m] * b[l + j * k];
      t[i + j * m] = s;
    }
  memcpy(out, t, sizeof(double) * m * n);
}
/* out(m x n) = a' b, a (k x m), b (k x n). */
static void mtm(int m, int k, int n, const double* a, const double* b, double* out) {
  double t[MX2 * 4];
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[l + i * k] * b[l + j * k];
      t[i + j * m] = s;
    }
  memcpy(out, t, sizeof(double) * m * n);
}
/* out(m x n) = a b', a (m x k), b (n x k). */
static void mmt(int m, int k, int n, const double* a, const double* b, double* out) {
  double t[MX2 * 4];
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[i + l * m] * b[j + l * n];
      t[i + j * m] = s;
    }
  memcpy(out, t, sizeof(double) * m * n);
}
static void mv(int m, int k, const double* a, const double* x, double* y) {
  double t[MX * 4];
  for (int i = 0; i < m; ++i) {
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += a[i + l * m] * x[l];
    t[i] = s;
  }
  memcpy(y, t, sizeof(double) * m);
}
static void mtv(int m, int k, const double* a, const double* x, double* y) { /* y = a' x, a (k x m) */
  double t[MX * 4];
  for (int i = 0; i < m; ++i) {
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += a[l + i * k] * x[l];
    t[i] = s;
  }
  memcpy(y, t, sizeof(double) * m);
}
static double dot(int n, const double* a, const double* b) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static void add(int n, const double* a, const double* b, double* o) {
  for (int i = 0; i < n; ++i) o[i] = a[i] + b[i];
}
static void sub(int n, const double* a, const double* b, double* o) {
  for (int i = 0; i < n; ++i) o[i] = a[i] - b[i];
}
static void symmetrize(int n, double* m) { /* types.hpp:58 */
  double t[MX2];
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) t[i + j * n] = 0.5 * (m[i + j * n] + m[j + i * n]);
  memcpy(m, t, sizeof(double) * n * n);
}
static int finite(int n, const double* a) {
  for (int i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

/* Eigen::LDLT restated (as in oracle/eigen_shim). */
typedef struct {
  int n, ok;
  double m[MX2];
  int t[MX];
} ldlt_t;
static void ldlt(ldlt_t* f, int n, const double* a) {
  f->n = n;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) f->m[i + j * n] = i >= j ? a[i + j * n] : a[j + i * n];
  int ok = 1;
  double temp[MX];
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bv = fabs(f->m[k + k * n]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(f->m[i + i * n]) > bv) {
        bv = fabs(f->m[i + i * n]);
        big = i;
      }
    f->t[k] = big;
    if (big != k) {
      for (int j = 0; j < n; ++j) {
        double x = f->m[k + j * n];
        f->m[k + j * n] = f->m[big + j * n];
        f->m[big + j * n] = x;
      }
      for (int i = 0; i < n; ++i) {
        double x = f->m[i + k * n];
        f->m[i + k * n] = f->m[i + big * n];
        f->m[i + big * n] = x;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = f->m[j + j * n] * f->m[k + j * n];
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += f->m[k + j * n] * temp[j];
      f->m[k + k * n] -= s;
      for (int i = k + 1; i < n; ++i) {
        double u = 0.0;
        for (int j = 0; j < k; ++j) u += f->m[i + j * n] * temp[j];
        f->m[i + k * n] -= u;
      }
    }
    const double akk = f->m[k + k * n];
    if (k + 1 < n) {
      if (fabs(akk) > 0.0) {
        for (int i = k + 1; i < n; ++i) f->m[i + k * n] /= akk;
      } else {
        for (int i = k + 1; i < n; ++i) ok = ok && f->m[i + k * n] == 0.0;
      }
    }
  }
  f->ok = ok;
}
static int ldlt_positive(const ldlt_t* f) { /* info() == Success && !(vectorD() <= 0).any() */
  if (!f->ok) return 0;
  for (int i = 0; i < f->n; ++i)
    if (!(f->m[i + i * f->n] > 0.0)) return 0;
  return 1;
}
static void ldlt_solve(const ldlt_t* f, int cols, const double* b, double* x) {
  const int n = f->n;
  double t[MX2 * 4];
  memcpy(t, b, sizeof(double) * n * cols);
  for (int c = 0; c < cols; ++c) {
    double* y = t + c * n;
    for (int k = 0; k < n; ++k) {
      double s = y[k];
      y[k] = y[f->t[k]];
      y[f->t[k]] = s;
    }
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) y[i] -= f->m[i + k * n] * y[k];
    for (int i = 0; i < n; ++i) {
      const double d = f->m[i + i * n];
      y[i] = fabs(d) > 2.2250738585072014e-308 ? y[i] / d : 0.0;
    }
    for (int i = n - 1; i >= 0; --i)
      for (int k = i + 1; k < n; ++k) y[i] -= f->m[k + i * n] * y[k];
    for (int k = n - 1; k >= 0; --k) {
      double s = y[k];
      y[k] = y[f->t[k]];
      y[f->t[k]] = s;
    }
  }
  memcpy(x, t, sizeof(double) * n * cols);
}

/* Eigen::PartialPivLU restated. */
typedef struct {
  int n;
  double lu[MX2];
  int perm[MX];
} lu_t;
static void lu_compute(lu_t* f, int n, const double* a) {
  f->n = n;
  memcpy(f->lu, a, sizeof(double) * n * n);
  for (int i = 0; i < n; ++i) f->perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(f->lu[k + k * n]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(f->lu[i + k * n]) > best) {
        best = fabs(f->lu[i + k * n]);
        p = i;
      }
    if (best != 0.0) {
      if (p != k) {
        for (int j = 0; j < n; ++j) {
          double x = f->lu[k + j * n];
          f->lu[k + j * n] = f->lu[p + j * n];
          f->lu[p + j * n] = x;
        }
        int tp = f->perm[k];
        f->perm[k] = f->perm[p];
        f->perm[p] = tp;
      }
      const double piv = f->lu[k + k * n];
      for (int i = k + 1; i < n; ++i) f->lu[i + k * n] /= piv;
    }
    for (int j = k + 1; j < n; ++j) {
      const double ukj = f->lu[k + j * n];
      for (int i = k + 1; i < n; ++i) f->lu[i + j * n] -= f->lu[i + k * n] * ukj;
    }
  }
}
static void lu_solve(const lu_t* f, int cols, const double* b, double* x) {
  const int n = f->n;
  double t[MX2 * 4];
  for (int c = 0; c < cols; ++c) {
    double* y = t + c * n;
    for (int i = 0; i < n; ++i) y[i] = b[f->perm[i] + c * n];
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) y[i] -= f->lu[i + k * n] * y[k];
    for (int i = n - 1; i >= 0; --i) {
      for (int k = i + 1; k < n; ++k) y[i] -= f->lu[i + k * n] * y[k];
      y[i] /= f->lu[i + i * n];
    }
  }
  memcpy(x, t, sizeof(double) * n * cols);
}
static void lu_solve_t(const lu_t* f, int cols, const double* b, double* x) { /* A' x = b */
  const int n = f->n;
  double t[MX2 * 4];
  for (int c = 0; c < cols; ++c) {
    double y[MX];
    for (int i = 0; i < n; ++i) {
      double s = b[i + c * n];
      for (int k = 0; k < i; ++k) s -= f->lu[k + i * n] * y[k];
      y[i] = s / f->lu[i + i * n];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= f->lu[k + i * n] * y[k];
      y[i] = s;
    }
    for (int i = 0; i < n; ++i) t[f->perm[i] + c * n] = y[i];
  }
  memcpy(x, t, sizeof(double) * n * cols);
}

/* ------------------------------------------------------------ LQR types */
typedef struct {
  double A[MX2], B[MX * 4], c[MX], Q[MX2], R[16], M[MX * 4], q[MX], r[4];
} stage_t; /* StageModel (types.hpp:28-40) */
typedef struct {
  double P[MX2], p[MX];
} value_t;
typedef struct {
  double K[MX * 4], k[4];
} policy_t;
typedef struct {
  double P[MX2], p[MX], C[MX2], A[MX2], c[MX];
} belem_t; /* ScanElementBwd (lqr_scan.hpp:15-24) */
typedef struct {
  double A[MX2], c[MX];
} felem_t;

enum { E_OK = 0, E_INDEF = 1, E_FACT = 2 };

/* init_bwd_element (lqr_scan.hpp:28-49) */
static int init_bwd(int nx, int nu, const stage_t* s, belem_t* e) {
  ldlt_t f;
  ldlt(&f, nu, s->R);
  if (!ldlt_positive(&f)) return E_FACT;
  double RiMt[MX * 4], Bt[MX * 4], RiBt[MX * 4], Rir[4], t[MX2], v[MX];
  ldlt_solve(&f, nx, s->M, RiMt);
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nu; ++i) Bt[i + j * nu] = s->B[j + i * nx];
  ldlt_solve(&f, nx, Bt, RiBt);
  ldlt_solve(&f, 1, s->r, Rir);
  mtm(nx, nu, nx, s->M, RiMt, t);
  sub(nx * nx, s->Q, t, e->P);
  mtv(nx, nu, s->M, Rir, v);
  sub(nx, s->q, v, e->p);
  mm(nx, nu, nx, s->B, RiBt, e->C);
  mm(nx, nu, nx, s->B, RiMt, t);
  sub(nx * nx, s->A, t, e->A);
  mv(nx, nu, s->B, Rir, v);
  sub(nx, s->c, v, e->c);
  symmetrize(nx, e->P);
  symmetrize(nx, e->C);
  return E_OK;
}
/* embed_terminal (lqr_scan.hpp:55-66) */
static void embed(int nx, const value_t* v, belem_t* e) {
  memcpy(e->P, v->P, sizeof(double) * nx * nx);
  memcpy(e->p, v->p, sizeof(double) * nx);
  memset(e->C, 0, sizeof(double) * nx * nx);
  memset(e->A, 0, sizeof(double) * nx * nx);
  memset(e->c, 0, sizeof(double) * nx);
}
/* combine_bwd (lqr_scan.hpp:80-111) */
static int combine_bwd(int nx, const belem_t* a, const belem_t* b, belem_t* out) {
  double G[MX2], t[MX2], iGA[MX2], iGC[MX2], v[MX], iGv[MX], PA[MX2], iGtPA[MX2], w[MX], iGtw[MX];
  const int n2 = nx * nx;
  for (int i = 0; i < n2; ++i) G[i] = 0.0;
  for (int i = 0; i < nx; ++i) G[i + i * nx] = 1.0;
  mm(nx, nx, nx, a->C, b->P, t);
  for (int i = 0; i < n2; ++i) G[i] += t[i];
  lu_t lu;
  lu_compute(&lu, nx, G);
  lu_solve(&lu, nx, a->A, iGA);
  lu_solve(&lu, nx, a->C, iGC);
  mv(nx, nx, a->C, b->p, v);
  sub(nx, a->c, v, v);
  lu_solve(&lu, 1, v, iGv);
  mm(nx, nx, nx, b->P, a->A, PA);
  lu_solve_t(&lu, nx, PA, iGtPA);
  mv(nx, nx, b->P, a->c, w);
  add(nx, b->p, w, w);
  lu_solve_t(&lu, 1, w, iGtw);
  belem_t o;
  mm(nx, nx, nx, b->A, iGA, o.A);
  mv(nx, nx, b->A, iGv, o.c);
  add(nx, o.c, b->c, o.c);
  mm(nx, nx, nx, b->A, iGC, t);
  mmt(nx, nx, nx, t, b->A, o.C);
  add(n2, o.C, b->C, o.C);
  mtv(nx, nx, a->A, iGtw, o.p);
  add(nx, o.p, a->p, o.p);
  mtm(nx, nx, nx, a->A, iGtPA, o.P);
  add(n2, o.P, a->P, o.P);
  symmetrize(nx, o.C);
  symmetrize(nx, o.P);
  *out = o;
  if (!(finite(n2, o.P) && finite(nx, o.p) && finite(n2, o.C) && finite(n2, o.A) && finite(nx, o.c))) return E_FACT;
  return E_OK;
}
/* feedback_from_values (lqr_scan.hpp:146-157) */
static int feedback(int nx, int nu, const stage_t* s, const value_t* nv, policy_t* pol) {
  double BtP[MX * 4], H[16], X[MX * 4], t[MX * 4], pc[MX], y[4];
  mtm(nu, nx, nx, s->B, nv->P, BtP);
  mm(nu, nx, nu, BtP, s->B, H);
  add(nu * nu, s->R, H, H);
  symmetrize(nu, H);
  ldlt_t f;
  ldlt(&f, nu, H);
  if (!ldlt_positive(&f)) return E_INDEF;
  mm(nu, nx, nx, BtP, s->A, t);
  add(nu * nx, s->M, t, X);
  ldlt_solve(&f, nx, X, X);
  for (int i = 0; i < nu * nx; ++i) pol->K[i] = -X[i];
  mv(nx, nx, nv->P, s->c, pc);
  add(nx, nv->p, pc, pc);
  mtv(nu, nx, s->B, pc, y);
  add(nu, s->r, y, y);
  ldlt_solve(&f, 1, y, y);
  for (int i = 0; i < nu; ++i) pol->k[i] = -y[i];
  return E_OK;
}
/* riccati_step (riccati.hpp:22-43) */
static int riccati_step(int nx, int nu, const stage_t* s, const double* Pn, const double* pn, value_t* v,
                        policy_t* pol) {
  double AtP[MX2], Qxx[MX2], BtP[MX * 4], Quu[16], Qux[MX * 4], qx[MX], qu[4], t[MX2];
  mtm(nx, nx, nx, s->A, Pn, AtP);
  mm(nx, nx, nx, AtP, s->A, t);
  add(nx * nx, s->Q, t, Qxx);
  mtm(nu, nx, nx, s->B, Pn, BtP);
  mm(nu, nx, nu, BtP, s->B, t);
  add(nu * nu, s->R, t, Quu);
  mm(nu, nx, nx, BtP, s->A, t);
  add(nu * nx, s->M, t, Qux);
  mtv(nx, nx, s->A, pn, t);
  add(nx, s->q, t, qx);
  mtv(nu, nx, s->B, pn, t);
  add(nu, s->r, t, qu);
  symmetrize(nu, Quu);
  ldlt_t f;
  ldlt(&f, nu, Quu);
  if (!ldlt_positive(&f)) return E_INDEF;
  ldlt_solve(&f, nx, Qux, pol->K);
  for (int i = 0; i < nu * nx; ++i) pol->K[i] = -pol->K[i];
  ldlt_solve(&f, 1, qu, pol->k);
  for (int i = 0; i < nu; ++i) pol->k[i] = -pol->k[i];
  mtm(nx, nu, nx, Qux, pol->K, t);
  add(nx * nx, Qxx, t, v->P);
  mtv(nx, nu, Qux, pol->k, t);
  add(nx, qx, t, v->p);
  symmetrize(nx, v->P);
  return E_OK;
}

/* ------------------------------------------------------------ scan.hpp */
typedef int (*op_fn)(int nx, const void* a, const void* b, void* out, int flip);
/* detail::tree_prefix_inplace (scan.hpp:19-36), `flip` swaps the operands
 * (the suffix scan's flipped operator, scan.hpp:53-65). */
static int tree_prefix(int nx, char* a, int n, size_t es, op_fn op, int flip) {
  if (n < 2) return E_OK;
  const int np = (n + 1) / 2;
  char* pairs = (char*)malloc(es * (size_t)np);
  int err = E_OK, e;
  for (int i = 0; 2 * i + 1 < n; ++i) {
    e = op(nx, a + es * (2 * i), a + es * (2 * i + 1), pairs + es * i, flip);
    if (!err) err = e;
  }
  if (n % 2 == 1) memcpy(pairs + es * (np - 1), a + es * (n - 1), es);
  e = tree_prefix(nx, pairs, np, es, op, flip);
  if (!err) err = e;
  for (int i = (n - 1) / 2; i >= 1; --i) {
    e = op(nx, pairs + es * (i - 1), a + es * (2 * i), a + es * (2 * i), flip);
    if (!err) err = e;
    if (2 * i + 1 < n) memcpy(a + es * (2 * i + 1), pairs + es * i, es);
  }
  memcpy(a + es * 1, pairs, es);
  free(pairs);
  return err;
}
static int op_bwd(int nx, const void* a, const void* b, void* out, int flip) {
  belem_t o;
  const int e = flip ? combine_bwd(nx, (const belem_t*)b, (const belem_t*)a, &o)
                     : combine_bwd(nx, (const belem_t*)a, (const belem_t*)b, &o);
  *(belem_t*)out = o;
  return e;
}
static int op_fwd(int nx, const void* a, const void* b, void* out, int flip) { /* combine_fwd (lqr_scan.hpp:171) */
  const felem_t* f1 = (const felem_t*)(flip ? b : a);
  const felem_t* f2 = (const felem_t*)(flip ? a : b);
  felem_t o;
  mm(nx, nx, nx, f2->A, f1->A, o.A);
  mv(nx, nx, f2->A, f1->c, o.c);
  add(nx, o.c, f2->c, o.c);
  *(felem_t*)out = o;
  return E_OK;
}

/* backward_scan (lqr_scan.hpp:123-141), tree order. values: N+1 entries. */
static int backward_scan(int nx, int nu, const stage_t* st, int N, const value_t* term, value_t* values) {
  belem_t* el = (belem_t*)malloc(sizeof(belem_t) * (size_t)(N + 1));
  int err = E_OK;
  for (int k = 0; k < N; ++k) {
    const int e = init_bwd(nx, nu, &st[k], &el[k]);
    if (!err) err = e;
  }
  embed(nx, term, &el[N]);
  /* inclusive_suffix_scan: reverse, flipped prefix, reverse. */
  for (int i = 0, j = N; i < j; ++i, --j) {
    belem_t t = el[i];
    el[i] = el[j];
    el[j] = t;
  }
  const int e = tree_prefix(nx, (char*)el, N + 1, sizeof(belem_t), op_bwd, 1);
  if (!err) err = e;
  for (int i = 0, j = N; i < j; ++i, --j) {
    belem_t t = el[i];
    el[i] = el[j];
    el[j] = t;
  }
  for (int k = 0; k <= N; ++k) {
    memcpy(values[k].P, el[k].P, sizeof(double) * nx * nx);
    memcpy(values[k].p, el[k].p, sizeof(double) * nx);
  }
  free(el);
  return err;
}

/* ------------------------------------------------------------ models */
typedef struct {
  const bo_problem* p;
  int nx, nu, n;
  stage_t* stage;   /* per node */
  double* defect;   /* [n][nx] */
  value_t* leaf;    /* per node */
} models_t;

static int is_leaf(const bo_problem* p, int i) { return p->nchild[i] == 0; }

/* ---- unicycle (unicycle.hpp:19-74) */
static void uni_deriv(const double* x, const double* u, double* d) {
  d[0] = x[3] * cos(x[2]);
  d[1] = x[3] * sin(x[2]);
  d[2] = u[1];
  d[3] = u[0];
}
static void uni_step(const double* x, const double* u, double dt, double* out) {
  double k1[4], k2[4], k3[4], k4[4], t[4];
  uni_deriv(x, u, k1);
  for (int i = 0; i < 4; ++i) t[i] = x[i] + 0.5 * dt * k1[i];
  uni_deriv(t, u, k2);
  for (int i = 0; i < 4; ++i) t[i] = x[i] + 0.5 * dt * k2[i];
  uni_deriv(t, u, k3);
  for (int i = 0; i < 4; ++i) t[i] = x[i] + dt * k3[i];
  uni_deriv(t, u, k4);
  const double s = dt / 6.0;
  for (int i = 0; i < 4; ++i) out[i] = x[i] + s * (((k1[i] + 2.0 * k2[i]) + 2.0 * k3[i]) + k4[i]);
}
static void uni_jx(const double* x, double* J) {
  memset(J, 0, sizeof(double) * 16);
  J[0 + 2 * 4] = -x[3] * sin(x[2]);
  J[0 + 3 * 4] = cos(x[2]);
  J[1 + 2 * 4] = x[3] * cos(x[2]);
  J[1 + 3 * 4] = sin(x[2]);
}
static void uni_jacobians(const double* x, const double* u, double dt, double* A, double* B) {
  double k1[4], k2[4], k3[4], x2[4], x3[4], x4[4];
  uni_deriv(x, u, k1);
  for (int i = 0; i < 4; ++i) x2[i] = x[i] + 0.5 * dt * k1[i];
  uni_deriv(x2, u, k2);
  for (int i = 0; i < 4; ++i) x3[i] = x[i] + 0.5 * dt * k2[i];
  uni_deriv(x3, u, k3);
  for (int i = 0; i < 4; ++i) x4[i] = x[i] + dt * k3[i];
  double J1[16], J2[16], J3[16], J4[16], Ju[8] = {0, 0, 0, 1, 0, 0, 1, 0}, I[16], T[16];
  uni_jx(x, J1);
  uni_jx(x2, J2);
  uni_jx(x3, J3);
  uni_jx(x4, J4);
  for (int i = 0; i < 16; ++i) I[i] = (i % 5 == 0) ? 1.0 : 0.0;
  const double h = 0.5 * dt;
  double d1x[16], d2x[16], d3x[16], d4x[16], d1u[8], d2u[8], d3u[8], d4u[8], Tu[8];
  memcpy(d1x, J1, sizeof d1x);
  for (int i = 0; i < 16; ++i) T[i] = I[i] + h * d1x[i];
  mm(4, 4, 4, J2, T, d2x);
  for (int i = 0; i < 16; ++i) T[i] = I[i] + h * d2x[i];
  mm(4, 4, 4, J3, T, d3x);
  for (int i = 0; i < 16; ++i) T[i] = I[i] + dt * d3x[i];
  mm(4, 4, 4, J4, T, d4x);
  memcpy(d1u, Ju, sizeof d1u);
  for (int i = 0; i < 8; ++i) Tu[i] = h * d1u[i];
  mm(4, 4, 2, J2, Tu, d2u);
  for (int i = 0; i < 8; ++i) d2u[i] += Ju[i];
  for (int i = 0; i < 8; ++i) Tu[i] = h * d2u[i];
  mm(4, 4, 2, J3, Tu, d3u);
  for (int i = 0; i < 8; ++i) d3u[i] += Ju[i];
  for (int i = 0; i < 8; ++i) Tu[i] = dt * d3u[i];
  mm(4, 4, 2, J4, Tu, d4u);
  for (int i = 0; i < 8; ++i) d4u[i] += Ju[i];
  const double s = dt / 6.0;
  for (int i = 0; i < 16; ++i) A[i] = I[i] + s * (((d1x[i] + 2.0 * d2x[i]) + 2.0 * d3x[i]) + d4x[i]);
  for (int i = 0; i < 8; ++i) B[i] = s * (((d1u[i] + 2.0 * d2u[i]) + 2.0 * d3u[i]) + d4u[i]);
}
/* ego_constraints (scenarios.hpp:206-248). Jx row-major [m][4], Ju [m][2]. */
static int ego(const bo_problem* p, int i, int leaf, const double* x, const double* u, double* g, double* Jx,
               double* Ju) {
  const int nb = leaf ? 0 : 4, nc = nb + p->nv;
  if (Jx) {
    memset(Jx, 0, sizeof(double) * nc * 4);
    memset(Ju, 0, sizeof(double) * nc * 2);
  }
  if (!leaf) {
    g[0] = u[0] - p->a_max;
    g[1] = -u[0] - p->a_max;
    g[2] = u[1] - p->w_max;
    g[3] = -u[1] - p->w_max;
    if (Ju) {
      Ju[0] = 1.0;
      Ju[2 * 1 + 0] = -1.0;
      Ju[2 * 2 + 1] = 1.0;
      Ju[2 * 3 + 1] = -1.0;
    }
  }
  for (int v = 0; v < p->nv; ++v) {
    const double* vp = p->vehicles + ((size_t)i * p->nv + v) * 2;
    const double dx = x[0] - vp[0], dy = x[1] - vp[1];
    const double dist = sqrt(dx * dx + dy * dy + 1e-6);
    g[nb + v] = p->radius - dist;
    if (Jx) {
      Jx[(nb + v) * 4 + 0] = -dx / dist;
      Jx[(nb + v) * 4 + 1] = -dy / dist;
    }
  }
  return nc;
}
static int ncon(const bo_problem* p, int i) { return p->kind == 1 ? (is_leaf(p, i) ? 0 : 4) + p->nv : 0; }
static size_t lq_ss(int nx, int nu) { return (size_t)(2 * nx * nx + nx * nu + nx + nu * nu + nu * nx + nx + nu); }

static void unpack_stage(int nx, int nu, const double* s, stage_t* st) {
  const double* o = s;
  memcpy(st->A, o, sizeof(double) * nx * nx), o += nx * nx;
  memcpy(st->B, o, sizeof(double) * nx * nu), o += nx * nu;
  memcpy(st->c, o, sizeof(double) * nx), o += nx;
  memcpy(st->Q, o, sizeof(double) * nx * nx), o += nx * nx;
  memcpy(st->R, o, sizeof(double) * nu * nu), o += nu * nu;
  memcpy(st->M, o, sizeof(double) * nu * nx), o += nu * nx;
  memcpy(st->q, o, sizeof(double) * nx), o += nx;
  memcpy(st->r, o, sizeof(double) * nu);
}

/* NodeDynamics::value */
static void dynamics(const bo_problem* p, int i, const double* x, const double* u, double* out) {
  if (p->kind == 1) {
    uni_step(x, u, p->dt, out);
    return;
  }
  const int nx = p->nx, nu = p->nu;
  stage_t s;
  unpack_stage(nx, nu, p->lq_stage + lq_ss(nx, nu) * i, &s);
  double a[MX], b[MX]; /* (A x + B u) + c, oracles.hpp:342-344 */
  mv(nx, nx, s.A, x, a);
  mv(nx, nu, s.B, u, b);
  for (int j = 0; j < nx; ++j) out[j] = (a[j] + b[j]) + s.c[j];
}

/* Node objective value (weight not applied), evaluate (problem.hpp:115-123). */
static double node_cost(const bo_problem* p, int i, const double* x, const double* u) {
  const int nx = p->nx, nu = p->nu;
  double t[MX], e[MX];
  if (p->kind == 1) {
    const double* ref = p->reference + 4 * (size_t)i;
    sub(4, x, ref, e);
    if (is_leaf(p, i)) {
      mv(4, 4, p->Wf, e, t);
      return 0.5 * dot(4, e, t);
    }
    mv(4, 4, p->Wx, e, t);
    double tu[2];
    mv(2, 2, p->Wu, u, tu);
    return 0.5 * dot(4, e, t) + 0.5 * dot(2, u, tu);
  }
  if (is_leaf(p, i)) {
    const double* l = p->lq_leaf + (size_t)i * (nx * nx + nx);
    mv(nx, nx, l, x, t);
    return 0.5 * dot(nx, x, t) + dot(nx, l + nx * nx, x);
  }
  stage_t s;
  unpack_stage(nx, nu, p->lq_stage + lq_ss(nx, nu) * i, &s);
  double Qx[MX], Ru[4], Mx[4];
  mv(nx, nx, s.Q, x, Qx);
  mv(nu, nu, s.R, u, Ru);
  mv(nu, nx, s.M, x, Mx);
  return 0.5 * dot(nx, x, Qx) + dot(nx, s.q, x) + 0.5 * dot(nu, u, Ru) + dot(nu, s.r, u) + dot(nu, u, Mx);
}

/* detail::al_penalty (problem.hpp:85-93) */
static double al_penalty(const double* g, const double* eta, int nc, double rho) {
  double v = 0.0;
  for (int m = 0; m < nc; ++m)
    if (g[m] >= 0.0 || eta[m] > 0.0) v += eta[m] * g[m] + 0.5 * rho * g[m] * g[m];
  return v;
}

typedef struct {
  double cost, cost_al, defect_l1, max_violation;
  int finite;
} eval_t;

#define NCMAX 12
/* evaluate (problem.hpp:109-146) */
static eval_t evaluate(const bo_problem* p, const double* x, const double* u, const double* eta, double rho) {
  const int nx = p->nx, nu = p->nu;
  eval_t ev = {0, 0, 0, 0, 1};
  for (int i = 0; i < p->n; ++i) {
    const double w = p->weight[i];
    const double nc_ = node_cost(p, i, x + (size_t)i * nx, u + (size_t)i * nu);
    ev.cost += w * nc_;
    double pen = 0.0;
    const int nc = ncon(p, i);
    if (nc > 0) {
      double g[NCMAX];
      ego(p, i, is_leaf(p, i), x + (size_t)i * nx, u + (size_t)i * nu, g, NULL, NULL);
      pen = al_penalty(g, eta + (size_t)i * NCMAX, nc, rho);
      double gm = g[0];
      for (int m = 1; m < nc; ++m) gm = g[m] > gm ? g[m] : gm;
      ev.max_violation = ev.max_violation > gm ? ev.max_violation : gm;
    }
    ev.cost_al += w * (nc_ + pen);
  }
  ev.max_violation = ev.max_violation > 0.0 ? ev.max_violation : 0.0;
  for (int i = 1; i < p->n; ++i) {
    const int pa = p->parent[i];
    double f[MX];
    dynamics(p, pa, x + (size_t)pa * nx, u + (size_t)pa * nu, f);
    double s = 0.0;
    for (int j = 0; j < nx; ++j) s += fabs(f[j] - x[(size_t)i * nx + j]);
    ev.defect_l1 += s;
  }
  ev.finite = isfinite(ev.cost_al) && isfinite(ev.defect_l1);
  return ev;
}

/* linearize (solver.hpp:65-149). Returns node+1 of a non-finite expansion. */
static int linearize(const bo_problem* p, const double* x, const double* u, const double* eta, double rho,
                     models_t* m) {
  const int nx = p->nx, nu = p->nu;
  for (int i = 0; i < p->n; ++i) {
    const double w = p->weight[i];
    const double* xi = x + (size_t)i * nx;
    const double* ui = u + (size_t)i * nu;
    const int nc = ncon(p, i), leaf = is_leaf(p, i);
    double g[NCMAX], Jx[NCMAX * 4], Ju[NCMAX * 2], as[NCMAX], lam[NCMAX];
    if (nc > 0) {
      ego(p, i, leaf, xi, ui, g, Jx, Ju);
      for (int mm_ = 0; mm_ < nc; ++mm_) {
        as[mm_] = (g[mm_] >= 0.0 || eta[(size_t)i * NCMAX + mm_] > 0.0) ? rho : 0.0;
        lam[mm_] = eta[(size_t)i * NCMAX + mm_] + as[mm_] * g[mm_];
      }
    }
    if (leaf) {
      double Q[MX2], q[MX], e[MX];
      if (p->kind == 1) {
        memcpy(Q, p->Wf, sizeof(double) * 16);
        sub(4, xi, p->reference + 4 * (size_t)i, e);
        mv(4, 4, p->Wf, e, q);
      } else {
        const double* l = p->lq_leaf + (size_t)i * (nx * nx + nx);
        memcpy(Q, l, sizeof(double) * nx * nx);
        mv(nx, nx, l, xi, q);
        add(nx, q, l + nx * nx, q);
      }
      if (nc > 0) {
        double t[MX], T[MX2];
        for (int a = 0; a < nx; ++a) {
          double s = 0.0;
          for (int mm_ = 0; mm_ < nc; ++mm_) s += Jx[mm_ * 4 + a] * lam[mm_];
          t[a] = s;
        }
        add(nx, q, t, q);
        for (int b = 0; b < nx; ++b)
          for (int a = 0; a < nx; ++a) {
            double s = 0.0;
            for (int mm_ = 0; mm_ < nc; ++mm_) s += (Jx[mm_ * 4 + a] * as[mm_]) * Jx[mm_ * 4 + b];
            T[a + b * nx] = s;
          }
        add(nx * nx, Q, T, Q);
      }
      for (int k = 0; k < nx * nx; ++k) m->leaf[i].P[k] = w * Q[k];
      for (int k = 0; k < nx; ++k) m->leaf[i].p[k] = w * q[k];
      if (!finite(nx * nx, m->leaf[i].P) || !finite(nx, m->leaf[i].p)) return i + 1;
      continue;
    }
    stage_t* s = &m->stage[i];
    if (p->kind == 1) {
      uni_jacobians(xi, ui, p->dt, s->A, s->B);
      double e[4];
      memcpy(s->Q, p->Wx, sizeof(double) * 16);
      memcpy(s->R, p->Wu, sizeof(double) * 4);
      memset(s->M, 0, sizeof(double) * 8);
      sub(4, xi, p->reference + 4 * (size_t)i, e);
      mv(4, 4, p->Wx, e, s->q);
      mv(2, 2, p->Wu, ui, s->r);
    } else {
      stage_t d;
      unpack_stage(nx, nu, p->lq_stage + lq_ss(nx, nu) * i, &d);
      memcpy(s->A, d.A, sizeof d.A);
      memcpy(s->B, d.B, sizeof d.B);
      memcpy(s->Q, d.Q, sizeof d.Q);
      memcpy(s->R, d.R, sizeof d.R);
      memcpy(s->M, d.M, sizeof d.M);
      double t[MX]; /* q = Q x + q + M' u ; r = R u + r + M x (oracles.hpp:360-361) */
      mv(nx, nx, d.Q, xi, s->q);
      add(nx, s->q, d.q, s->q);
      mtv(nx, nu, d.M, ui, t);
      add(nx, s->q, t, s->q);
      mv(nu, nu, d.R, ui, s->r);
      add(nu, s->r, d.r, s->r);
      mv(nu, nx, d.M, xi, t);
      add(nu, s->r, t, s->r);
    }
    if (nc > 0) {
      double t[MX];
      for (int a = 0; a < nx; ++a) {
        double v = 0.0;
        for (int mm_ = 0; mm_ < nc; ++mm_) v += Jx[mm_ * 4 + a] * lam[mm_];
        t[a] = v;
      }
      add(nx, s->q, t, s->q);
      for (int a = 0; a < nu; ++a) {
        double v = 0.0;
        for (int mm_ = 0; mm_ < nc; ++mm_) v += Ju[mm_ * 2 + a] * lam[mm_];
        t[a] = v;
      }
      add(nu, s->r, t, s->r);
      for (int b = 0; b < nx; ++b)
        for (int a = 0; a < nx; ++a) {
          double v = 0.0;
          for (int mm_ = 0; mm_ < nc; ++mm_) v += (Jx[mm_ * 4 + a] * as[mm_]) * Jx[mm_ * 4 + b];
          s->Q[a + b * nx] += v;
        }
      for (int b = 0; b < nu; ++b)
        for (int a = 0; a < nu; ++a) {
          double v = 0.0;
          for (int mm_ = 0; mm_ < nc; ++mm_) v += (Ju[mm_ * 2 + a] * as[mm_]) * Ju[mm_ * 2 + b];
          s->R[a + b * nu] += v;
        }
      for (int b = 0; b < nx; ++b)
        for (int a = 0; a < nu; ++a) {
          double v = 0.0;
          for (int mm_ = 0; mm_ < nc; ++mm_) v += (Ju[mm_ * 2 + a] * as[mm_]) * Jx[mm_ * 4 + b];
          s->M[a + b * nu] += v;
        }
    }
    for (int k = 0; k < nx * nx; ++k) s->Q[k] *= w;
    for (int k = 0; k < nu * nu; ++k) s->R[k] *= w;
    for (int k = 0; k < nu * nx; ++k) s->M[k] *= w;
    for (int k = 0; k < nx; ++k) s->q[k] *= w;
    for (int k = 0; k < nu; ++k) s->r[k] *= w;
    memset(s->c, 0, sizeof(double) * nx);
    if (!finite(nx * nx, s->A) || !finite(nx * nu, s->B) || !finite(nx * nx, s->Q) || !finite(nu * nu, s->R) ||
        !finite(nx, s->q) || !finite(nu, s->r))
      return i + 1;
  }
  for (int i = 1; i < p->n; ++i) {
    const int pa = p->parent[i];
    double f[MX];
    dynamics(p, pa, x + (size_t)pa * nx, u + (size_t)pa * nu, f);
    for (int j = 0; j < nx; ++j) m->defect[(size_t)i * nx + j] = f[j] - x[(size_t)i * nx + j];
    if (!finite(nx, m->defect + (size_t)i * nx)) return i + 1;
  }
  return 0;
}

/* ------------------------------------------------------------ passes */
/* backward_pass (solver.hpp:203-318): P1 chain scans + P2 tree Riccati, or
 * strategy 2 = sequential tree Riccati (riccati_tree). */
static int backward_pass(const bo_problem* p, const models_t* min, double reg, int strategy, value_t* value,
                         policy_t* pol, double* max_ff) {
  const int nx = min->nx, nu = min->nu, n = p->n;
  stage_t* st = (stage_t*)malloc(sizeof(stage_t) * (size_t)n);
  value_t* lf = (value_t*)malloc(sizeof(value_t) * (size_t)n);
  memcpy(st, min->stage, sizeof(stage_t) * (size_t)n);
  memcpy(lf, min->leaf, sizeof(value_t) * (size_t)n);
  if (reg > 0.0) { /* solver.hpp:212-222 */
    for (int i = 0; i < n; ++i) {
      if (is_leaf(p, i))
        for (int j = 0; j < nx; ++j) lf[i].P[j + j * nx] += reg;
      else
        for (int j = 0; j < nu; ++j) st[i].R[j + j * nu] += reg;
    }
  }
  int err = E_OK;
  int boundary;
  if (strategy == 2) {
    boundary = p->horizon;
    for (int i = p->step_begin[boundary]; i < p->step_begin[boundary + 1]; ++i) value[i] = lf[i];
  } else {
    /* P1: chains from each node at step N_b + 1 to its leaf (solver.hpp:177-187, 235-286). */
    boundary = p->last_branch_step + 1;
    for (int h = p->step_begin[boundary]; h < p->step_begin[boundary + 1] && !err; ++h) {
      int len = 0;
      int* nodes = (int*)malloc(sizeof(int) * (size_t)(p->horizon + 2));
      for (int v = h;; v = p->first_child[v]) {
        nodes[len++] = v;
        if (is_leaf(p, v)) break;
      }
      const int steps = len - 1;
      if (steps == 0) {
        value[h] = lf[h];
        free(nodes);
        continue;
      }
      stage_t* cs = (stage_t*)malloc(sizeof(stage_t) * (size_t)steps);
      value_t* vals = (value_t*)malloc(sizeof(value_t) * (size_t)(steps + 1));
      for (int k = 0; k < steps; ++k) { /* chain_stage (solver.hpp:189-193) */
        cs[k] = st[nodes[k]];
        memcpy(cs[k].c, min->defect + (size_t)nodes[k + 1] * nx, sizeof(double) * nx);
      }
      int e = backward_scan(nx, nu, cs, steps, &lf[nodes[steps]], vals);
      if (!err) err = e;
      for (int k = 0; k < steps && !err; ++k) {
        e = feedback(nx, nu, &cs[k], &vals[k + 1], &pol[nodes[k]]);
        if (!err) err = e;
      }
      for (int k = 0; k <= steps; ++k) value[nodes[k]] = vals[k];
      free(cs);
      free(vals);
      free(nodes);
    }
  }
  /* P2: riccati_tree_from(models, boundary, values) (riccati.hpp:97-122). */
  for (int i = p->step_begin[boundary] - 1; i >= 0 && !err; --i) {
    double Pn[MX2] = {0}, pn[MX] = {0};
    for (int c = 0; c < p->nchild[i]; ++c) {
      const int ch = p->first_child[i] + c;
      double t[MX];
      for (int k = 0; k < nx * nx; ++k) Pn[k] += value[ch].P[k];
      mv(nx, nx, value[ch].P, min->defect + (size_t)ch * nx, t);
      add(nx, value[ch].p, t, t);
      add(nx, pn, t, pn);
    }
    const int e = riccati_step(nx, nu, &st[i], Pn, pn, &value[i], &pol[i]);
    if (!err) err = e;
  }
  double mff = 0.0;
  for (int i = 0; i < n && !err; ++i) {
    if (is_leaf(p, i)) continue;
    double m = 0.0;
    for (int j = 0; j < nu; ++j) m = fabs(pol[i].k[j]) > m ? fabs(pol[i].k[j]) : m;
    mff = m > mff ? m : mff;
  }
  *max_ff = mff;
  free(st);
  free(lf);
  return err;
}

/* linear_rollout (solver.hpp:330-387). */
static void linear_rollout(const bo_problem* p, const models_t* m, const policy_t* pol, const double* dx0, double* dx,
                           double* du, int strategy) {
  const int nx = m->nx, nu = m->nu;
  const int boundary = strategy == 2 ? p->horizon : p->last_branch_step + 1;
  memcpy(dx, dx0, sizeof(double) * nx);
  for (int i = 0; i < p->step_begin[boundary]; ++i) {
    const stage_t* s = &m->stage[i];
    double BK[MX2], Acl[MX2], Bk[MX];
    mm(nx, nu, nx, s->B, pol[i].K, BK);
    add(nx * nx, s->A, BK, Acl);
    mv(nx, nu, s->B, pol[i].k, Bk);
    for (int c = 0; c < p->nchild[i]; ++c) {
      const int ch = p->first_child[i] + c;
      double t[MX];
      mv(nx, nx, Acl, dx + (size_t)i * nx, t);
      add(nx, t, Bk, t);
      add(nx, t, m->defect + (size_t)ch * nx, dx + (size_t)ch * nx);
    }
  }
  for (int h = p->step_begin[boundary]; h < p->step_begin[boundary + 1] && boundary < p->horizon + 1; ++h) {
    int len = 0;
    int* nodes = (int*)malloc(sizeof(int) * (size_t)(p->horizon + 2));
    for (int v = h;; v = p->first_child[v]) {
      nodes[len++] = v;
      if (is_leaf(p, v)) break;
    }
    const int steps = len - 1;
    if (steps > 0) {
      felem_t* el = (felem_t*)malloc(sizeof(felem_t) * (size_t)steps);
      for (int k = 0; k < steps; ++k) { /* init_fwd_element (lqr_scan.hpp:166-168) on chain_stage */
        const stage_t* s = &m->stage[nodes[k]];
        double t[MX2];
        mm(nx, nu, nx, s->B, pol[nodes[k]].K, t);
        add(nx * nx, s->A, t, el[k].A);
        mv(nx, nu, s->B, pol[nodes[k]].k, t);
        add(nx, m->defect + (size_t)nodes[k + 1] * nx, t, el[k].c);
      }
      tree_prefix(nx, (char*)el, steps, sizeof(felem_t), op_fwd, 0);
      for (int k = 0; k < steps; ++k) { /* forward_scan: x = A x0 + c (lqr_scan.hpp:186) */
        double t[MX];
        mv(nx, nx, el[k].A, dx + (size_t)h * nx, t);
        add(nx, t, el[k].c, dx + (size_t)nodes[k + 1] * nx);
      }
      free(el);
    }
    free(nodes);
  }
  for (int i = 0; i < p->n; ++i) {
    if (is_leaf(p, i)) continue;
    double t[4];
    mv(nu, nx, pol[i].K, dx + (size_t)i * nx, t);
    add(nu, t, pol[i].k, du + (size_t)i * nu);
  }
}

/* expected_change_coefficients (solver.hpp:412-430). */
static void expected_change(const bo_problem* p, const models_t* m, const double* dx, const double* du, double* a1,
                            double* a2) {
  const int nx = m->nx, nu = m->nu;
  double s1 = 0.0, s2 = 0.0;
  for (int i = 0; i < p->n; ++i) {
    const double* x = dx + (size_t)i * nx;
    double t[MX];
    if (is_leaf(p, i)) {
      s1 += dot(nx, m->leaf[i].p, x);
      mv(nx, nx, m->leaf[i].P, x, t);
      s2 += 0.5 * dot(nx, x, t);
    } else {
      const stage_t* s = &m->stage[i];
      const double* u = du + (size_t)i * nu;
      double tm[4], tr[4];
      s1 += dot(nx, s->q, x) + dot(nu, s->r, u);
      mv(nx, nx, s->Q, x, t);
      mv(nu, nx, s->M, x, tm);
      mv(nu, nu, s->R, u, tr);
      s2 += 0.5 * dot(nx, x, t) + dot(nu, u, tm) + 0.5 * dot(nu, u, tr);
    }
  }
  *a1 = s1;
  *a2 = s2;
}

static int rollout(const bo_problem* p, const double* u_in, double* x, double* u) { /* problem.hpp:150-166 */
  const int nx = p->nx, nu = p->nu;
  memset(x, 0, sizeof(double) * (size_t)p->n * nx);
  memset(u, 0, sizeof(double) * (size_t)p->n * nu);
  memcpy(x, p->x0, sizeof(double) * nx);
  for (int i = 0; i < p->n; ++i) {
    if (is_leaf(p, i)) continue;
    if (u_in) memcpy(u + (size_t)i * nu, u_in + (size_t)i * nu, sizeof(double) * nu);
    double nxt[MX];
    dynamics(p, i, x + (size_t)i * nx, u + (size_t)i * nu, nxt);
    if (!finite(nx, nxt)) return -1;
    for (int c = 0; c < p->nchild[i]; ++c) memcpy(x + (size_t)(p->first_child[i] + c) * nx, nxt, sizeof(double) * nx);
  }
  return 0;
}

void bo_default_options(bo_options* o) { /* solver.hpp:35-57 */
  o->max_inner_iterations = 100;
  o->max_outer_iterations = 10;
  o->alpha_levels = 11;
  o->armijo_beta = 1e-4;
  o->merit_gamma = 0.5;
  o->merit_mu0 = 1.0;
  o->merit_mu_init = 1.0;
  o->defect_epsilon = 1e-8;
  o->tol_defect = 1e-8;
  o->tol_cost = 1e-8;
  o->tol_feedforward = 1e-6;
  o->tol_constraint = 1e-4;
  o->penalty_init = 10.0;
  o->penalty_growth = 10.0;
  o->penalty_max = 1e8;
  o->reg_init = 0.0;
  o->reg_min = 1e-6;
  o->reg_growth = 10.0;
  o->reg_decay = 10.0;
  o->reg_max = 1e10;
}

/* solve (solver.hpp:595-780) with the default pmsilqr strategy. */
int bo_solve(const bo_problem* p, const bo_options* o, const double* u_init, double* x_out, double* u_out,
             bo_report* rep, bo_record* recs, int max_recs) {
  const int n = p->n, nx = p->nx, nu = p->nu;
  double* x = (double*)calloc((size_t)n * nx, sizeof(double));
  double* u = (double*)calloc((size_t)n * nu, sizeof(double));
  double* xt = (double*)calloc((size_t)n * nx, sizeof(double));
  double* ut = (double*)calloc((size_t)n * nu, sizeof(double));
  double* dx = (double*)calloc((size_t)n * nx, sizeof(double));
  double* du = (double*)calloc((size_t)n * nu, sizeof(double));
  double* eta = (double*)calloc((size_t)n * NCMAX, sizeof(double));
  models_t m = {p, nx, nu, n, (stage_t*)calloc((size_t)n, sizeof(stage_t)), (double*)calloc((size_t)n * nx, sizeof(double)),
                (value_t*)calloc((size_t)n, sizeof(value_t))};
  value_t* val = (value_t*)calloc((size_t)n, sizeof(value_t));
  policy_t* pol = (policy_t*)calloc((size_t)n, sizeof(policy_t));
  memset(rep, 0, sizeof *rep);
  rep->status = 2;
  int rc = 0;
  if (rollout(p, u_init, x, u) != 0) {
    rc = -1;
    goto done;
  }
  {
    double rho = o->penalty_init, mu = o->merit_mu_init, reg = o->reg_init;
    int inner_conv = 0, failed = 0, status = 2;
    int has_con = 0;
    for (int i = 0; i < n; ++i) has_con = has_con || ncon(p, i) > 0;
    double dx0[MX];
    for (int outer = 0; outer < o->max_outer_iterations; ++outer) {
      ++rep->outer_iterations;
      inner_conv = 0;
      for (int pass = 0; pass < o->max_inner_iterations; ++pass) {
        const int bad = linearize(p, x, u, eta, rho, &m);
        if (bad) {
          rep->error_code = 4;
          failed = 1;
          break;
        }
        const eval_t ev = evaluate(p, x, u, eta, rho);
        for (int j = 0; j < nx; ++j) dx0[j] = p->x0[j] - x[j];
        double max_ff = 0.0;
        const int berr = backward_pass(p, &m, reg, 0, val, pol, &max_ff);
        if (berr) {
          reg = reg * o->reg_growth > o->reg_min ? reg * o->reg_growth : o->reg_min;
          if (reg > o->reg_max) {
            rep->error_code = berr == E_INDEF ? 1 : 2;
            failed = 1;
            break;
          }
          continue;
        }
        linear_rollout(p, &m, pol, dx0, dx, du, 0);
        double a1, a2;
        expected_change(p, &m, dx, du, &a1, &a2);
        const double ec_full = a1 + a2;
        if (ev.defect_l1 <= o->tol_defect && fabs(ec_full) <= o->tol_cost * (1.0 + fabs(ev.cost_al)) &&
            max_ff <= o->tol_feedforward) {
          inner_conv = 1;
          break;
        }
        { /* update_mu (solver.hpp:400-407) */
          double trial = mu;
          if (ev.defect_l1 > o->defect_epsilon) trial = ec_full / ((1.0 - o->merit_gamma) * ev.defect_l1) + o->merit_mu0;
          mu = trial > mu ? trial : mu;
        }
        const double merit0 = ev.cost_al + mu * ev.defect_l1;
        /* line_search, parallel mode (solver.hpp:459-518) */
        int acc = -1;
        double acc_alpha = 0, acc_merit = 0, acc_dec = 0;
        eval_t acc_ev = ev;
        for (int l = 0; l < o->alpha_levels; ++l) {
          const double alpha = pow(0.5, l);
          for (int i = 0; i < n * nx; ++i) xt[i] = x[i] + alpha * dx[i];
          for (int i = 0; i < n; ++i)
            for (int j = 0; j < nu; ++j)
              ut[(size_t)i * nu + j] = is_leaf(p, i) ? u[(size_t)i * nu + j]
                                                     : u[(size_t)i * nu + j] + alpha * du[(size_t)i * nu + j];
          const eval_t te = evaluate(p, xt, ut, eta, rho);
          const double mer = te.finite ? te.cost_al + mu * te.defect_l1 : INFINITY;
          const double ec = a1 * alpha + a2 * alpha * alpha;
          const double dec = o->armijo_beta * (ec - alpha * mu * ev.defect_l1);
          if (isfinite(mer) && mer <= merit0 + dec) {
            acc = l;
            acc_alpha = alpha;
            acc_merit = mer;
            acc_dec = dec;
            acc_ev = te;
            break; /* the first (largest) accepted alpha wins */
          }
        }
        bo_record rec;
        memset(&rec, 0, sizeof rec);
        rec.outer = outer;
        rec.merit_before = merit0;
        rec.mu = mu;
        rec.max_feedforward = max_ff;
        rec.regularization = reg;
        rec.accepted = acc >= 0;
        rec.alpha = acc_alpha;
        rec.model_decrease = acc_dec;
        if (acc < 0) {
          reg = reg * o->reg_growth > o->reg_min ? reg * o->reg_growth : o->reg_min;
          rec.merit_after = merit0;
          rec.cost = ev.cost;
          rec.cost_al = ev.cost_al;
          rec.defect_l1 = ev.defect_l1;
          rec.violation = ev.max_violation;
          if (recs && rep->n_records < max_recs) recs[rep->n_records] = rec;
          ++rep->n_records;
          if (reg > o->reg_max) {
            rep->error_code = 3;
            failed = 1;
            break;
          }
          continue;
        }
        for (int i = 0; i < n * nx; ++i) x[i] = x[i] + acc_alpha * dx[i];
        for (int i = 0; i < n; ++i)
          if (!is_leaf(p, i))
            for (int j = 0; j < nu; ++j) u[(size_t)i * nu + j] = u[(size_t)i * nu + j] + acc_alpha * du[(size_t)i * nu + j];
        reg = reg / o->reg_decay >= o->reg_min ? reg / o->reg_decay : 0.0;
        ++rep->inner_iterations;
        rec.merit_after = acc_merit;
        rec.cost = acc_ev.cost;
        rec.cost_al = acc_ev.cost_al;
        rec.defect_l1 = acc_ev.defect_l1;
        rec.violation = acc_ev.max_violation;
        if (recs && rep->n_records < max_recs) recs[rep->n_records] = rec;
        ++rep->n_records;
      }
      if (failed) break;
      const eval_t ev = evaluate(p, x, u, eta, rho);
      if (!has_con) {
        status = inner_conv ? 0 : 1;
        break;
      }
      if (inner_conv && ev.max_violation <= o->tol_constraint) {
        status = 0;
        break;
      }
      if (outer + 1 == o->max_outer_iterations) {
        status = 1;
        break;
      }
      for (int i = 0; i < n; ++i) { /* solver.hpp:764-769 */
        const int nc = ncon(p, i);
        if (!nc) continue;
        double g[NCMAX];
        ego(p, i, is_leaf(p, i), x + (size_t)i * nx, u + (size_t)i * nu, g, NULL, NULL);
        for (int k = 0; k < nc; ++k) {
          const double v = eta[(size_t)i * NCMAX + k] + rho * g[k];
          eta[(size_t)i * NCMAX + k] = v > 0.0 ? v : 0.0;
        }
      }
      rho = rho * o->penalty_growth < o->penalty_max ? rho * o->penalty_growth : o->penalty_max;
    }
    rep->status = failed ? 2 : status;
    const eval_t fin = evaluate(p, x, u, eta, rho);
    rep->final_cost = fin.cost;
    rep->final_violation = fin.max_violation;
    rep->final_defect_l1 = fin.defect_l1;
  }
done:
  if (x_out) memcpy(x_out, x, sizeof(double) * (size_t)n * nx);
  if (u_out) memcpy(u_out, u, sizeof(double) * (size_t)n * nu);
  free(x), free(u), free(xt), free(ut), free(dx), free(du), free(eta);
  free(m.stage), free(m.defect), free(m.leaf), free(val), free(pol);
  return rc;
}

int bo_lqr_tree(const bo_problem* tree, int nx, int nu, const double* stage, const double* defect, const double* leaf,
                double reg, int strategy, const double* dx0, double* K, double* k, double* P, double* pv, double* dx,
                double* du, double* scalars) {
  const int n = tree->n;
  models_t m = {tree, nx, nu, n, (stage_t*)calloc((size_t)n, sizeof(stage_t)), (double*)calloc((size_t)n * nx, sizeof(double)),
                (value_t*)calloc((size_t)n, sizeof(value_t))};
  for (int i = 0; i < n; ++i) {
    if (i > 0) memcpy(m.defect + (size_t)i * nx, defect + (size_t)i * nx, sizeof(double) * nx);
    if (is_leaf(tree, i)) {
      memcpy(m.leaf[i].P, leaf + (size_t)i * (nx * nx + nx), sizeof(double) * nx * nx);
      memcpy(m.leaf[i].p, leaf + (size_t)i * (nx * nx + nx) + nx * nx, sizeof(double) * nx);
    } else {
      unpack_stage(nx, nu, stage + lq_ss(nx, nu) * i, &m.stage[i]);
      memset(m.stage[i].c, 0, sizeof(double) * nx);
    }
  }
  value_t* val = (value_t*)calloc((size_t)n, sizeof(value_t));
  policy_t* pol = (policy_t*)calloc((size_t)n, sizeof(policy_t));
  double* ddx = (double*)calloc((size_t)n * nx, sizeof(double));
  double* ddu = (double*)calloc((size_t)n * nu, sizeof(double));
  double mff = 0.0;
  const int err = backward_pass(tree, &m, reg, strategy, val, pol, &mff);
  scalars[0] = mff;
  scalars[3] = err;
  if (!err) {
    linear_rollout(tree, &m, pol, dx0, ddx, ddu, strategy);
    expected_change(tree, &m, ddx, ddu, &scalars[1], &scalars[2]);
  }
  for (int i = 0; i < n; ++i) {
    if (P) memcpy(P + (size_t)i * nx * nx, val[i].P, sizeof(double) * nx * nx);
    if (pv) memcpy(pv + (size_t)i * nx, val[i].p, sizeof(double) * nx);
    if (!is_leaf(tree, i)) {
      if (K) memcpy(K + (size_t)i * nu * nx, pol[i].K, sizeof(double) * nu * nx);
      if (k) memcpy(k + (size_t)i * nu, pol[i].k, sizeof(double) * nu);
      if (du) memcpy(du + (size_t)i * nu, ddu + (size_t)i * nu, sizeof(double) * nu);
    }
    if (dx) memcpy(dx + (size_t)i * nx, ddx + (size_t)i * nx, sizeof(double) * nx);
  }
  free(m.stage), free(m.defect), free(m.leaf), free(val), free(pol), free(ddx), free(ddu);
  return 0;
}

/* ------------------------------------------------------------ tree */
int bo_tree_size(int horizon, int nb, const int* steps, const int* arities) {
  long long level = 1, total = 1;
  int b = 0;
  for (int k = 0; k < horizon; ++k) {
    if (b < nb && steps[b] == k) level *= arities[b++];
    total += level;
  }
  return (int)total;
}

int bo_build_tree(int horizon, int nb, const int* steps, const int* arities, const double* weights, int max_arity,
                  int* parent, int* time_step, double* weight, int* first_child, int* nchild, int* step_begin) {
  if (horizon < 1) return -1; /* tree.hpp:62-83 validation */
  for (int b = 0; b < nb; ++b) {
    if (steps[b] < 0 || steps[b] >= horizon) return -1;
    if (b > 0 && steps[b] <= steps[b - 1]) return -1;
    if (arities[b] < 2 || arities[b] > max_arity) return -1;
    double s = 0.0;
    for (int a = 0; a < arities[b]; ++a) {
      if (!(weights[b * max_arity + a] > 0.0)) return -1;
      s += weights[b * max_arity + a];
    }
    if (fabs(s - 1.0) > 1e-9) return -1;
  }
  /* Level expansion (tree.hpp:96-115). */
  int n = 1;
  parent[0] = -1;
  time_step[0] = 0;
  weight[0] = 1.0;
  int lvl_begin = 0, lvl_end = 1, next = 0;
  step_begin[0] = 0;
  for (int k = 0; k < horizon; ++k) {
    step_begin[k + 1] = n;
    int br = -1;
    if (next < nb && steps[next] == k) br = next++;
    for (int node = lvl_begin; node < lvl_end; ++node) {
      const int arity = br >= 0 ? arities[br] : 1;
      for (int a = 0; a < arity; ++a) {
        parent[n] = node;
        time_step[n] = k + 1;
        weight[n] = weight[node] * (br >= 0 ? weights[br * max_arity + a] : 1.0);
        ++n;
      }
    }
    lvl_begin = lvl_end;
    lvl_end = n;
  }
  step_begin[horizon + 1] = n;
  for (int i = 0; i < n; ++i) {
    first_child[i] = -1;
    nchild[i] = 0;
  }
  for (int i = 1; i < n; ++i) {
    if (first_child[parent[i]] < 0) first_child[parent[i]] = i;
    ++nchild[parent[i]];
  }
  return n;
}

/* ------------------------------------------------------------ random */
/* std::mt19937_64 (libstdc++). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;
static void mt_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}
static uint64_t mt_next(mt64_t* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
/* uniform_real_distribution<double>(-1, 1) via generate_canonical<double, 53>. */
static double uni(mt64_t* s) {
  double r = (double)mt_next(s) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r * 2.0 + -1.0;
}
void bo_mt_uniform(unsigned long long seed, int count, double* out) {
  mt64_t s;
  mt_seed(&s, seed);
  for (int i = 0; i < count; ++i) out[i] = uni(&s);
}
/* random_matrix: row-major fill (oracles.hpp:22-29) */
static void rmat(mt64_t* s, int r, int c, double scale, double* m) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m[i + j * r] = scale * uni(s);
}
static void rstage(mt64_t* s, int nx, int nu, double* out) { /* random_stage (oracles.hpp:39-54) */
  double A[MX2], B[MX * 4], c[MX], G[(MX + 4) * (MX + 4)], H[(MX + 4) * (MX + 4)], q[MX], r[4];
  const int m = nx + nu;
  rmat(s, nx, nx, 1.0 / sqrt((double)nx), A);
  rmat(s, nx, nu, 1.0, B);
  for (int i = 0; i < nx; ++i) c[i] = 0.5 * uni(s);
  rmat(s, m, m, 1.0, G);
  for (int j = 0; j < m; ++j) /* H = G G' / m, then diag += 1e-3 */
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += G[i + l * m] * G[j + l * m];
      H[i + j * m] = acc / (double)m;
    }
  for (int i = 0; i < m; ++i) H[i + i * m] += 1e-3;
  for (int i = 0; i < nx; ++i) q[i] = uni(s);
  for (int i = 0; i < nu; ++i) r[i] = uni(s);
  double* o = out;
  memcpy(o, A, sizeof(double) * nx * nx), o += nx * nx;
  memcpy(o, B, sizeof(double) * nx * nu), o += nx * nu;
  memcpy(o, c, sizeof(double) * nx), o += nx;
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nx; ++i) o[i + j * nx] = H[i + j * m];
  o += nx * nx;
  for (int j = 0; j < nu; ++j)
    for (int i = 0; i < nu; ++i) o[i + j * nu] = H[(nx + i) + (nx + j) * m] + (i == j ? 0.1 : 0.0);
  o += nu * nu;
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nu; ++i) o[i + j * nu] = H[(nx + i) + j * m];
  o += nu * nx;
  memcpy(o, q, sizeof(double) * nx), o += nx;
  memcpy(o, r, sizeof(double) * nu);
}
static void rterminal(mt64_t* s, int nx, double* out) { /* random_terminal (oracles.hpp:56-61) */
  double G[MX2];
  rmat(s, nx, nx, 1.0, G);
  for (int j = 0; j < nx; ++j)
    for (int i = 0; i < nx; ++i) {
      double acc = 0.0;
      for (int l = 0; l < nx; ++l) acc += G[i + l * nx] * G[j + l * nx];
      out[i + j * nx] = acc / (double)nx;
    }
  for (int i = 0; i < nx; ++i) out[i + i * nx] += 1e-3;
  for (int i = 0; i < nx; ++i) out[nx * nx + i] = uni(s);
}
void bo_random_lq(unsigned long long seed, int n, const int* nchild, int nx, int nu, double* x0, double* stage,
                  double* leaf) {
  mt64_t s;
  mt_seed(&s, seed);
  for (int i = 0; i < nx; ++i) x0[i] = uni(&s);
  const size_t ss = lq_ss(nx, nu), ls = (size_t)(nx * nx + nx);
  for (int i = 0; i < n; ++i) {
    if (nchild[i] == 0)
      rterminal(&s, nx, leaf + ls * i);
    else
      rstage(&s, nx, nu, stage + ss * i);
  }
}

int bo_init_bwd_element(int nx, int nu, const double* stage, double* e) {
  stage_t s;
  unpack_stage(nx, nu, stage, &s);
  belem_t el;
  const int rc = init_bwd(nx, nu, &s, &el);
  memcpy(e, el.P, sizeof(double) * nx * nx);
  memcpy(e + nx * nx, el.p, sizeof(double) * nx);
  memcpy(e + nx * nx + nx, el.C, sizeof(double) * nx * nx);
  memcpy(e + 2 * nx * nx + nx, el.A, sizeof(double) * nx * nx);
  memcpy(e + 3 * nx * nx + nx, el.c, sizeof(double) * nx);
  return rc;
}

int bo_combine_bwd(int nx, const double* e1, const double* e2, double* out) {
  belem_t a, b, o;
  const double* src[2] = {e1, e2};
  belem_t* dst[2] = {&a, &b};
  for (int t = 0; t < 2; ++t) {
    memcpy(dst[t]->P, src[t], sizeof(double) * nx * nx);
    memcpy(dst[t]->p, src[t] + nx * nx, sizeof(double) * nx);
    memcpy(dst[t]->C, src[t] + nx * nx + nx, sizeof(double) * nx * nx);
    memcpy(dst[t]->A, src[t] + 2 * nx * nx + nx, sizeof(double) * nx * nx);
    memcpy(dst[t]->c, src[t] + 3 * nx * nx + nx, sizeof(double) * nx);
  }
  const int rc = combine_bwd(nx, &a, &b, &o);
  memcpy(out, o.P, sizeof(double) * nx * nx);
  memcpy(out + nx * nx, o.p, sizeof(double) * nx);
  memcpy(out + nx * nx + nx, o.C, sizeof(double) * nx * nx);
  memcpy(out + 2 * nx * nx + nx, o.A, sizeof(double) * nx * nx);
  memcpy(out + 3 * nx * nx + nx, o.c, sizeof(double) * nx);
  return rc;
}

/* nonlinear_rollout (problem.hpp:150-166) and evaluate (problem.hpp:109-146)
 * with zero multipliers, for property checks. */
int bo_rollout(const bo_problem* p, const double* u, double* x_out) {
  double* ub = (double*)calloc((size_t)p->n * p->nu, sizeof(double));
  const int rc = rollout(p, u, x_out, ub);
  free(ub);
  return rc;
}

void bo_evaluate(const bo_problem* p, const double* x, const double* u, double rho, double* out) {
  double* eta = (double*)calloc((size_t)p->n * NCMAX, sizeof(double));
  const eval_t ev = evaluate(p, x, u, eta, rho);
  out[0] = ev.cost;
  out[1] = ev.cost_al;
  out[2] = ev.defect_l1;
  out[3] = ev.max_violation;
  out[4] = ev.finite;
  free(eta);
}
