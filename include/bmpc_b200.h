/* bmpc_b200 — C ABI of the B200-native branch-MPC solver.
 *
 * Drop-in boundary for the reference solve path (bmpc::solve,
 * /root/reference/proj/include/bmpc/solver.hpp:595-596). Every entry point
 * takes plain pointers and sizes; no exceptions cross it (int status +
 * bmpc_last_error()). Reference interfaces each entry replaces are cited.
 *
 * Ownership: the library owns everything it returns through a `**out`
 * argument; free it with the matching *_free / *_destroy call. Input arrays
 * are borrowed for the duration of the call only. A bmpc_ctx is bound to one
 * device and one CUDA stream and is not thread-safe (one host thread per ctx,
 * like the reference's single-owner solver).
 */
#ifndef BMPC_B200_H
#define BMPC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
#define BMPC_OK 0
#define BMPC_ERR_INVALID (-1)     /* bad argument (reference: std::invalid_argument) */
#define BMPC_ERR_CUDA (-2)        /* CUDA runtime failure / no device */
#define BMPC_ERR_UNSUPPORTED (-3) /* model kind or dimensions not compiled in */
#define BMPC_ERR_ROLLOUT (-4)     /* nonlinear_rollout non-finite state (problem.hpp:160-162 throws) */
#define BMPC_ERR_OUT_OF_RANGE (-5)

/* Solve status (SolveStatus, solver.hpp:536). */
#define BMPC_CONVERGED 0
#define BMPC_MAX_ITERATIONS 1
#define BMPC_ERROR 2

/* Model families (the reference's per-node callbacks, problem.hpp:15-40,
 * restated as device functions). */
#define BMPC_MODEL_UNICYCLE 1          /* unicycle RK4 + tracking + ego constraints (scenarios.hpp) */
#define BMPC_MODEL_AFFINE_QUADRATIC 2  /* affine dynamics + quadratic cost (oracles.hpp:316 random_lq_problem) */

const char* bmpc_last_error(void);
const char* bmpc_version(void);

/* ------------------------------------------------------------------ tree */
/* TreeTopology (tree.hpp:28-44) as flat arrays, bit-identical to build_tree
 * (tree.hpp:61-128). Children of a node are contiguous in BFS order, so they
 * are given as [first_child, first_child + child_count). */
typedef struct bmpc_tree {
  int node_count;
  int horizon;
  int last_branch_step; /* -1 for a path graph */
  int leaf_count;
  int* parent;      /* [node_count], -1 at the root */
  int* time_step;   /* [node_count] */
  double* weight;   /* [node_count] path probability */
  int* first_child; /* [node_count], -1 at leaves */
  int* child_count; /* [node_count] */
  int* step_begin;  /* [horizon + 2] */
  int* leaves;      /* [leaf_count] ascending */
} bmpc_tree;

/* build_tree(horizon, branchings) (tree.hpp:61). weights is n_branchings
 * rows of max_arity entries (row b holds arities[b] weights). */
int bmpc_tree_build(int horizon, int n_branchings, const int* steps, const int* arities, const double* weights,
                    int max_arity, bmpc_tree** out);
void bmpc_tree_free(bmpc_tree* tree);

/* -------------------------------------------------------------- problem */
/* Device model descriptor: what the reference captures inside its
 * std::function callbacks, as plain per-node arrays. */
typedef struct bmpc_model_desc {
  int kind;
  int state_dim;
  int input_dim;
  const double* initial_state; /* [state_dim] (BmpcProblem::initial_state) */
  /* BMPC_MODEL_UNICYCLE (state_dim 4, input_dim 2) */
  double dt;
  double state_weights[16];    /* Wx, column-major 4x4 (tracking_cost, problem.hpp:194) */
  double input_weights[4];     /* Wu, 2x2 */
  double terminal_weights[16]; /* Wf, 4x4 (tracking_terminal_cost, problem.hpp:211) */
  double accel_limit, yaw_rate_limit, safety_radius; /* ego_constraints (scenarios.hpp:206) */
  int num_vehicles;                                  /* <= 4 */
  const double* reference;        /* [node][4] tracking reference */
  const double* vehicle_position; /* [node][num_vehicles][2] */
  /* BMPC_MODEL_AFFINE_QUADRATIC: column-major blocks per node
   *   non-leaf: A[nx*nx] B[nx*nu] c[nx] Q[nx*nx] R[nu*nu] M[nu*nx] q[nx] r[nu]
   *   leaf:     P[nx*nx] p[nx]                                               */
  const double* lq_stage; /* [node][stage record] */
  const double* lq_leaf;  /* [node][nx*nx + nx] */
} bmpc_model_desc;

/* Host-side scenario builders (scenarios.hpp), producing a tree + model
 * descriptor whose arrays the returned object owns. */
#define BMPC_SCENARIO_INTERSECTION 0 /* build_intersection_case (scenarios.hpp:296) */
#define BMPC_SCENARIO_LATENCY 1      /* build_latency_case (scenarios.hpp:398) */
#define BMPC_SCENARIO_MULTISTAGE 2   /* multi-stage intersection (cfg2/cfg3) */
/* ScenarioSpec (scenarios.hpp:15-47): surrounding vehicles, tuning and
 * timing of a scene. The JSON form is scenario_spec_to_json /
 * scenario_spec_from_json (serialization.hpp:128-197). */
#define BMPC_MAX_TARGETS 8
typedef struct bmpc_vehicle {
  double position[2];
  double heading, speed;
  int n_targets;
  double target_speeds[BMPC_MAX_TARGETS];
} bmpc_vehicle;
typedef struct bmpc_scenario_spec {
  double total_time;
  int n_shared; /* 1 or 2 */
  double shared_times[2];
  int horizon;
  double ego_start[4];
  int n_vehicles; /* <= 4 */
  bmpc_vehicle vehicles[4];
  double state_weights[4], input_weights[2], terminal_weights[4];
  double accel_limit, yaw_rate_limit, safety_radius, prediction_tau;
  double reference_turn_rate, backup_deceleration, continue_deceleration;
} bmpc_scenario_spec;

typedef struct bmpc_scenario {
  int family;
  int horizon;
  double total_time;
  double shared_time[2]; /* intersection: [0]; latency: T_sh0, T_sh1 */
  int v1, v2;            /* intersection vehicle option counts */
  int n_branchings;      /* multistage: explicit uniform branchings */
  int branch_step[8];
  int branch_arity[8];
  int perturb;           /* perturb the measured initial state ... */
  unsigned long long perturb_seed; /* ... with std::mt19937_64(perturb_seed) */
  /* Full scene (vehicles, weights, limits, timing) as build_intersection_case /
   * build_latency_case take it; NULL = the family's reference preset
   * (intersection_spec / latency_spec) from the timing fields above. */
  const bmpc_scenario_spec* spec;
} bmpc_scenario;

typedef struct bmpc_problem_data {
  bmpc_tree* tree;
  bmpc_model_desc model;
} bmpc_problem_data;

int bmpc_scenario_build(const bmpc_scenario* spec, bmpc_problem_data** out);
void bmpc_problem_data_free(bmpc_problem_data* data);

/* -------------------------------------------------------- options/report */
/* SolverOptions (solver.hpp:28-58). The strategy enums keep the reference's
 * numbering (solver.hpp:23-26); defaults are pmsilqr (all 0):
 *   backward    0 scan_tree_riccati, 1 scan_condensed (hypmsilqr: the shared
 *               segment condensed into a dense QP over its inputs and solved
 *               by Cholesky / pivoted LU on the device, open-loop policies
 *               K = 0, k = u there, solver.hpp:297-307; at most 4096 stacked
 *               shared inputs, else BMPC_ERR_UNSUPPORTED), 2 sequential_riccati
 *               (team Riccati sweep on every segment);
 *   forward     0 linear_rollout, 1 nonlinear_rollout (single-shooting trials);
 *   line_search 0 parallel, 1 sequential (one step size per round; the
 *               accepted step is the same in both modes). */
#define BMPC_BACKWARD_SCAN_TREE_RICCATI 0
#define BMPC_BACKWARD_SCAN_CONDENSED 1
#define BMPC_BACKWARD_SEQUENTIAL_RICCATI 2
#define BMPC_FORWARD_LINEAR 0
#define BMPC_FORWARD_NONLINEAR 1
#define BMPC_LINE_SEARCH_PARALLEL 0
#define BMPC_LINE_SEARCH_SEQUENTIAL 1
typedef struct bmpc_options {
  int max_inner_iterations, max_outer_iterations, alpha_levels;
  double armijo_beta, merit_gamma, merit_mu0, merit_mu_init, defect_epsilon;
  double tol_defect, tol_cost, tol_feedforward, tol_constraint;
  double penalty_init, penalty_growth, penalty_max;
  double reg_init, reg_min, reg_growth, reg_decay, reg_max;
  int backward, forward, line_search;
} bmpc_options;
void bmpc_options_default(bmpc_options* opts);

/* IterationRecord (solver.hpp:547-561). */
typedef struct bmpc_record {
  int outer, accepted;
  double cost, cost_al, merit_before, merit_after, model_decrease, defect_l1, violation, alpha, mu,
      max_feedforward, regularization;
} bmpc_record;

/* SolveReport (solver.hpp:572-582); `times` = PhaseTimes (setup,
 * backward_p1 [= whole tree-scan backward pass], backward_p2 [= 0],
 * forward, line_search, total) in seconds of device time. */
typedef struct bmpc_report {
  int status, error_code, error_node, inner_iterations, outer_iterations, n_records;
  double final_cost, final_violation, final_defect_l1;
  double times[6];
  double final_penalty, final_mu, final_reg;
  char message[160];
  /* Work counter (not a SolveReport field): step sizes the line search
   * evaluated over all passes (see bmpc_ctx_set_line_search_block). */
  double alpha_evals;
} bmpc_report;

/* ------------------------------------------------------------- context */
typedef struct bmpc_ctx bmpc_ctx;
int bmpc_ctx_create(int device, bmpc_ctx** out);
/* Destroying a ctx that still has live batches only marks it; the last
 * bmpc_batch_destroy frees it (any destruction order is safe). */
void bmpc_ctx_destroy(bmpc_ctx* ctx);
int bmpc_ctx_set_stream(bmpc_ctx* ctx, void* cuda_stream); /* cudaStream_t; NULL = ctx-owned stream */
int bmpc_ctx_synchronize(bmpc_ctx* ctx);
/* Backward/forward strategy per tree segment: segments of at most `len`
 * nodes use the team-cooperative sequential Riccati sweep, longer ones the
 * associative scan (0 = scan everywhere; default 384, env BMPC_SEQ_MAX). */
int bmpc_ctx_set_seq_max_len(bmpc_ctx* ctx, int len);
/* Line search (solver.hpp:459-518) in rounds of `alphas` step sizes: a round
 * evaluates its alphas for every node and stops at the first accepted one, so
 * the chosen alpha and every reported value equal the all-at-once parallel
 * search; later rounds run only when a whole round is rejected
 * (0 = all alpha_levels in one round; default 2, env BMPC_LS_BLOCK). */
int bmpc_ctx_set_line_search_block(bmpc_ctx* ctx, int alphas);
/* Batch schedule for batches larger than one resident wave: a probe launch
 * runs every instance for `probe_passes` inner passes and suspends it, the
 * instances are ordered by their last constraint violation (largest first),
 * and a second launch resumes them; results are bit-identical to one launch
 * (0 = one FIFO launch; default 10, env BMPC_PROBE). */
int bmpc_ctx_set_schedule(bmpc_ctx* ctx, int probe_passes);
/* Number of kernels this ctx launched since creation (evidence counter). */
long long bmpc_ctx_launch_count(const bmpc_ctx* ctx);

/* ------------------------------------------------------ single solve */
/* solve(problem, opts, initial_inputs) (solver.hpp:595). initial_inputs:
 * [node][input_dim] or NULL (zeros). Outputs: x_out [node][state_dim],
 * u_out [node][input_dim] (leaf rows 0), report, up to max_records records.
 * Large trees run on the whole GPU (cooperative launch); small ones on one
 * thread block. Host buffers; synchronous. */
int bmpc_solve(bmpc_ctx* ctx, const bmpc_tree* tree, const bmpc_model_desc* model, const bmpc_options* opts,
               const double* initial_inputs, double* x_out, double* u_out, bmpc_report* report,
               bmpc_record* records, int max_records);

/* ------------------------------------------------------ batched solves */
/* A batch holds `count` independent instances sharing one tree shape and
 * model family, device-resident (one thread block per instance). */
typedef struct bmpc_batch bmpc_batch;
int bmpc_batch_create(bmpc_ctx* ctx, const bmpc_tree* tree, int count, const bmpc_model_desc* model_template,
                      int max_records, bmpc_batch** out);
void bmpc_batch_destroy(bmpc_batch* batch);
/* Host -> device copy of every instance's per-node data and initial state
 * (models[count], same kind/dims/num_vehicles as the template). Async on the
 * ctx stream. Returns the bytes copied in *h2d_bytes (may be NULL). */
int bmpc_batch_set_models(bmpc_batch* batch, const bmpc_model_desc* models, size_t* h2d_bytes);
/* Device-to-device replication of instance 0's data into all instances. */
/* Per-call measured states only: x0 [count][state_dim] (host) is uploaded
 * over the node data already resident from bmpc_batch_set_models /
 * bmpc_batch_replicate — the receding-horizon case where the scenario
 * (references, predictions) is fixed and each call brings new initial states.
 * h2d_bytes (optional) receives the bytes copied. */
int bmpc_batch_set_initial_states(bmpc_batch* batch, const double* x0, size_t* h2d_bytes);
int bmpc_batch_replicate(bmpc_batch* batch);
/* Device-side scene generation (the receding-horizon call where the ego state
 * and the surrounding vehicles change every control step): from scene specs
 * (one per instance, or n_specs = 1 for all), the device computes every
 * node's tracking reference (left_turn_reference / the latency references,
 * scenarios.hpp:201-214, 416-441), the vehicle predictions
 * (predict_vehicles, :87-113, with the family's branch choices), the model
 * scalars and x0 = ego_start. Each spec must imply the batch's tree (same
 * horizon and branch steps); family as in bmpc_scenario. h2d_bytes receives
 * the bytes uploaded (the specs and model scalars only). Async. */
int bmpc_batch_set_scenes(bmpc_batch* batch, int family, const bmpc_scenario_spec* specs, int n_specs, int v1,
                          int v2, size_t* h2d_bytes);
/* Per-node scene data of one instance (device -> host): reference [node][4],
 * vehicles [node][num_vehicles][2], x0 [nx]; any pointer may be NULL. */
int bmpc_batch_scene(bmpc_batch* batch, int instance, double* reference, double* vehicles, double* x0);
/* Per-instance thread-block shape: `threads` per block with at least
 * `min_blocks` resident per SM (compiled variants only). */
int bmpc_batch_set_launch(bmpc_batch* batch, int threads, int min_blocks);
/* Launch the solve of every instance (async on the ctx stream). */
int bmpc_batch_solve(bmpc_batch* batch, const bmpc_options* opts);
/* Device -> host copy of results and synchronize. Any pointer may be NULL.
 * x_out [count][node][nx], u_out [count][node][nu], reports [count]. */
int bmpc_batch_results(bmpc_batch* batch, double* x_out, double* u_out, bmpc_report* reports,
                       size_t* d2h_bytes);
/* Device pointers of the result trajectories (for an NVLink gather). */
int bmpc_batch_device_results(bmpc_batch* batch, double** d_x, double** d_u, size_t* bytes_x, size_t* bytes_u);
/* Packs every instance's [x (node*nx) | u (node*nu)] contiguously into the
 * device buffer d_dst (count * node * (nx + nu) doubles), async on the ctx
 * stream — the send buffer of the final NVLink gather. */
int bmpc_batch_pack_results(bmpc_batch* batch, double* d_dst, size_t* bytes);
/* Records of one instance (device -> host copy). */
int bmpc_batch_records(bmpc_batch* batch, int instance, bmpc_record* records, int max_records, int* n_records);
/* Kernel launches the batch solve issues (1) and the launch configuration. */
int bmpc_batch_info(const bmpc_batch* batch, int* threads_per_block, int* blocks, int* regs_per_thread);

/* ------------------------------------------- multi-device batched solves */
/* The reference's batched throughput path is a thread pool of independent
 * solve() calls (parallel_sweep, tools/bench.cpp:259-269). Here the instance
 * space is split into contiguous shards, one per ctx (device):
 * shard g = [g*count/n, (g+1)*count/n). No data-path collective: each device
 * solves its shard with its own launches; the only exchange is the final
 * gather of the packed trajectories to the first ctx's device. */
int bmpc_shard_range(int count, int n_shards, int g, int* begin, int* n);
typedef struct bmpc_multi bmpc_multi;
/* ctxs[n_ctx] (several ctxs may share a device); the template as in
 * bmpc_batch_create. */
int bmpc_multi_create(bmpc_ctx* const* ctxs, int n_ctx, const bmpc_tree* tree, int count,
                      const bmpc_model_desc* model_template, int max_records, bmpc_multi** out);
void bmpc_multi_destroy(bmpc_multi* multi);
int bmpc_multi_set_models(bmpc_multi* multi, const bmpc_model_desc* models, size_t* h2d_bytes);
int bmpc_multi_set_initial_states(bmpc_multi* multi, const double* x0, size_t* h2d_bytes);
/* Launches every shard's solve, asynchronously on each ctx's stream. */
int bmpc_multi_solve(bmpc_multi* multi, const bmpc_options* opts);
/* Final gather: d_dst is device memory on ctxs[0]'s device holding
 * count * node * (nx + nu) doubles ([x | u] per instance, global order).
 * Each shard's pack kernel stores its instances straight into d_dst over
 * peer-to-peer (NVLink/NVSwitch) mappings; devices that cannot map device 0
 * pack locally and copy peer-to-peer. Synchronizes every shard. */
int bmpc_multi_gather(bmpc_multi* multi, double* d_dst, size_t* bytes);
/* Host results in global instance order (as bmpc_batch_results). */
int bmpc_multi_results(bmpc_multi* multi, double* x_out, double* u_out, bmpc_report* reports, size_t* d2h_bytes);
/* Shard g's batch (borrowed; NULL for an empty shard) and its range. */
int bmpc_multi_shard(bmpc_multi* multi, int g, bmpc_batch** batch, int* begin, int* n);
/* One-shot: create + set_models + solve + results + destroy. */
int bmpc_solve_batch(bmpc_ctx* const* ctxs, int n_ctx, const bmpc_tree* tree, int count,
                     const bmpc_model_desc* models, const bmpc_options* opts, double* x_out, double* u_out,
                     bmpc_report* reports);

/* Measured FP64 FMA throughput of this device (TFLOP/s): the roofline
 * denominator of the FP64-bound solve path. */
int bmpc_fp64_peak_tflops(bmpc_ctx* ctx, double* tflops);
/* Diagnostic per-phase device timers (ns accumulated by the solve loop):
 * slots 0 linearize+evaluate, 1 backward terminals/elements, 2 backward
 * scans, 3 feedback, 4 forward elements, 5 forward scans, 6 forward sweep,
 * 7 line search, 8 merit/convergence, 9 step/AL bookkeeping. */
int bmpc_batch_set_profiling(bmpc_batch* batch, int on);
int bmpc_batch_phase_profile(bmpc_batch* batch, int instance, double* out, int n);
/* Diagnostic: dependent-latency probe {DFMA, LDS, FP64 division} in SM cycles. */
int bmpc_debug_latency_probe(bmpc_ctx* ctx, double* cycles3);
/* Diagnostic: SM cycles per team-cooperative Riccati step on a chain. */
/* prefetch == 2: stage-stamped run, cycles[0..5] = total, then per-stage cycles per step. */
int bmpc_debug_ric_step_cycles(bmpc_ctx* ctx, int steps, int prefetch, double* cycles);
/* Diagnostic: microseconds per cooperative grid barrier at this launch shape. */
int bmpc_debug_grid_sync_us(bmpc_ctx* ctx, int blocks, int threads, int iters, double* us);

/* ---------------------------------------------- kernel-level LQR tree */
/* backward_pass + linear_rollout + expected_change_coefficients
 * (solver.hpp:203-430) on explicit TreeStageModels (riccati.hpp:77-84):
 * stage [node][A B c Q R M q r] (c ignored), defect [node][nx], leaf
 * [node][P p]. Outputs K [node][nu*nx], k [node][nu], P [node][nx*nx],
 * p [node][nx], dx [node][nx], du [node][nu]; scalars = {max_feedforward,
 * a1, a2, error (0 ok, 1 IndefiniteHessian, 2 Factorization)}.
 * grid != 0 runs on the whole GPU (cooperative), else one thread block. */
int bmpc_lqr_tree(bmpc_ctx* ctx, const bmpc_tree* tree, int nx, int nu, const double* stage, const double* defect,
                  const double* leaf, double reg, const double* dx0, int grid, double* K, double* k, double* P,
                  double* p, double* dx, double* du, double* scalars);

/* Backward strategy of subsequent bmpc_lqr_tree calls on this ctx:
 * BMPC_BACKWARD_SCAN_TREE_RICCATI (default) or BMPC_BACKWARD_SCAN_CONDENSED
 * (the shared segment condensed into a dense QP; its nodes get K = 0, k = u,
 * backward_pass, solver.hpp:297-307). */
int bmpc_ctx_set_lqr_strategy(bmpc_ctx* ctx, int backward);

/* Batched scan-element primitives (lqr_scan.hpp), one GPU thread per element:
 *   op 0  init_bwd_element (:28-49): a = count records [A B c Q R M q r]
 *         (column-major; R gets + reg on its diagonal), out = elements;
 *   op 1  combine_bwd (:80-111): out = a (+) b, elements [P p C A c]
 *         (3 nx^2 + 2 nx doubles each, unpadded);
 *   op 2  combine_fwd (:171-173): out = a (+) b, elements [A c] (nx^2 + nx).
 * An element whose R is not positive definite comes back as NaN. */
int bmpc_lqr_elements(bmpc_ctx* ctx, int op, int nx, int nu, int count, const double* a, const double* b, double reg,
                      double* out);

#ifdef __cplusplus
}
#endif

#endif /* BMPC_B200_H */
