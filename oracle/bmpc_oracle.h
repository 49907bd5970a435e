/* bmpc_oracle — plain-C restatement of the reference solve path.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker, never by the product.
 *
 * Restates /root/reference/proj/include/bmpc: tree.hpp (build_tree),
 * scan.hpp (tree schedule), lqr_scan.hpp (scan LQR), riccati.hpp (tree
 * Riccati), problem.hpp (evaluate, rollouts, tracking costs), unicycle.hpp,
 * scenarios.hpp (ego constraints), solver.hpp (linearize, backward_pass with
 * the P1 chain scans + P2 tree Riccati, linear_rollout, EC, merit, update_mu,
 * parallel line search, solve) and testing/oracles.hpp (random instances,
 * libstdc++ mt19937_64 + uniform_real_distribution). Eigen's LDLT and
 * PartialPivLU are restated in the same form as oracle/eigen_shim.
 * Pinned against the shim-built reference (oracle/_ref) by tests/test_oracle.py
 * and the committed fixtures in tests/golden/.
 */
#ifndef BMPC_ORACLE_H
#define BMPC_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

#define BO_MAXN 8 /* max state / input dimension */

typedef struct {
  /* tree (tree.hpp:28-44) */
  int n, horizon, last_branch_step;
  const int* parent;
  const int* first_child; /* -1 at leaves; children contiguous */
  const int* nchild;
  const double* weight;
  const int* step_begin; /* [horizon + 2] */
  /* model */
  int kind; /* 1 unicycle tracking, 2 affine-quadratic */
  int nx, nu;
  const double* x0;
  double dt;
  const double *Wx, *Wu, *Wf; /* column-major */
  double a_max, w_max, radius;
  int nv;
  const double* reference; /* [n][4] */
  const double* vehicles;  /* [n][nv][2] */
  const double* lq_stage;  /* [n][A B c Q R M q r] */
  const double* lq_leaf;   /* [n][P p] */
} bo_problem;

typedef struct {
  int max_inner_iterations, max_outer_iterations, alpha_levels;
  double armijo_beta, merit_gamma, merit_mu0, merit_mu_init, defect_epsilon;
  double tol_defect, tol_cost, tol_feedforward, tol_constraint;
  double penalty_init, penalty_growth, penalty_max;
  double reg_init, reg_min, reg_growth, reg_decay, reg_max;
} bo_options;

typedef struct {
  int outer, accepted;
  double cost, cost_al, merit_before, merit_after, model_decrease, defect_l1, violation, alpha, mu,
      max_feedforward, regularization;
} bo_record;

typedef struct {
  int status; /* 0 converged, 1 max-iter, 2 error */
  int error_code;
  int inner_iterations, outer_iterations, n_records;
  double final_cost, final_violation, final_defect_l1;
} bo_report;

void bo_default_options(bo_options* o);

/* solve (solver.hpp:595-780). u_init [n][nu] or NULL. Returns 0, or -1 when
 * the initial nonlinear rollout is non-finite (the reference throws). */
int bo_solve(const bo_problem* p, const bo_options* o, const double* u_init, double* x_out, double* u_out,
             bo_report* rep, bo_record* recs, int max_recs);

/* backward_pass + linear_rollout + EC (solver.hpp:203-430) on explicit
 * TreeStageModels; stage [n][A B c Q R M q r] (c ignored), defect [n][nx],
 * leaf [n][P p]. scalars = {max_ff, a1, a2, error}. strategy 0: scan + tree
 * Riccati (pmsilqr), 2: sequential tree Riccati. */
int bo_lqr_tree(const bo_problem* tree, int nx, int nu, const double* stage, const double* defect,
                const double* leaf, double reg, int strategy, const double* dx0, double* K, double* k, double* P,
                double* pv, double* dx, double* du, double* scalars);

/* build_tree (tree.hpp:61-128): outputs sized by bo_tree_size. Returns -1 on
 * an invalid spec. weights: nb rows of max_arity. */
int bo_tree_size(int horizon, int nb, const int* steps, const int* arities);
int bo_build_tree(int horizon, int nb, const int* steps, const int* arities, const double* weights, int max_arity,
                  int* parent, int* time_step, double* weight, int* first_child, int* nchild, int* step_begin);

/* testing::random_lq_problem draws (oracles.hpp:316-365) with libstdc++'s
 * mt19937_64 + uniform_real_distribution(-1, 1). */
void bo_random_lq(unsigned long long seed, int n, const int* nchild, int nx, int nu, double* x0, double* stage,
                  double* leaf);
/* Raw engine / distribution (for pinning against libstdc++). */
void bo_mt_uniform(unsigned long long seed, int count, double* out);

/* nonlinear_rollout of inputs u from x0; evaluate with zero multipliers:
 * out = {cost, cost_al, defect_l1, max_violation, finite}. */
int bo_rollout(const bo_problem* p, const double* u, double* x_out);
void bo_evaluate(const bo_problem* p, const double* x, const double* u, double rho, double* out);

/* Unit routines on single elements (lqr_scan.hpp), element = P p C A c. */
int bo_init_bwd_element(int nx, int nu, const double* stage /*A B c Q R M q r*/, double* e);
int bo_combine_bwd(int nx, const double* e1, const double* e2, double* out);

#ifdef __cplusplus
}
#endif
#endif
