// Plain-old-data structs shared by the host runtime (host.cpp, host
// compiler) and the device solver (solver.cuh). No device code here.
#pragma once

namespace bmpc_b200 {

enum ModelKind : int { kModelUnicycle = 1, kModelAffineQuadratic = 2 };

constexpr int kMaxVehicles = 4;
constexpr int kMaxCon = 4 + kMaxVehicles;

// Per-instance model parameters (device pointers + shared scalars).
struct ModelParams {
  int kind;
  int nv;                  // vehicles (unicycle)
  double dt;
  double Wx[16], Wu[4], Wf[16];
  double a_max, w_max, radius;
  int w_diag;               // Wx, Wu, Wf all diagonal: structured (zero-skipping) expansion, same bits
  const double* reference;  // [node][4]
  const double* vehicles;   // [node][nv][2]
  // affine-quadratic
  const double* lq_stage;   // [node][stage_size]: A B c Q R M q r (column-major)
  const double* lq_leaf;    // [node][nx*nx + nx]: P p
};

constexpr int kMaxAlpha = 16;
constexpr int kProfSlots = 24;

// ------------------------------------------------------------------ options
struct DevOptions {  // SolverOptions (solver.hpp:28-58), device copy
  int max_inner_iterations, max_outer_iterations, alpha_levels;
  double armijo_beta, merit_gamma, merit_mu0, merit_mu_init, defect_epsilon;
  double tol_defect, tol_cost, tol_feedforward, tol_constraint;
  double penalty_init, penalty_growth, penalty_max;
  double reg_init, reg_min, reg_growth, reg_decay, reg_max;
  int zero_inputs;  // 1: initial inputs are zero (solver.hpp:604-609), skip the H2D
  int seq_max_len;  // segments of <= this many nodes use the team Riccati sweep, longer ones the scan
  int seq_wide_segs, seq_wide_max;  // ... and depths with >= seq_wide_segs segments of <= seq_wide_max
  int ls_block;     // step sizes evaluated per line-search round (<= 0: all alpha_levels at once)
  int pass_budget;  // > 0: suspend a solve after this many inner passes in this launch (Work::resume)
  const int* order; // optional block -> instance map of a batch launch (nullptr: identity)
  int keep_values;  // 1: store (P, p) of every node (kernel-level API); 0: segment heads only
  int fwd_scan_min; // segments of >= this length take the forward prefix scan (0: walk everywhere)
  int nonlinear_ls; // 1: ForwardMode::nonlinear_rollout trials (sssilqr, solver.hpp:463-467)
  int chunk_bwd;    // > 0: kChunk kernels sweep segments of >= this many nodes with the chunked scan
  int condensed;    // 1: BackwardStrategy::scan_condensed (hypmsilqr): P2 by condensing + dense solve
  int bwd_hs;       // > 0: Hillis-Steele backward scan where segments x length <= bwd_hs x teams
  int fwd_block_scan;  // > 0: wide blocks roll segments of >= this many transitions out by a block-local affine-map scan
};

// Suspended solve() loop state (batch scheduling): a solve can stop at the top
// of an inner pass and continue in a later launch with bit-identical results.
struct DevResume {
  int state;  // 0 fresh, 1 suspended, 2 finished
  int outer, pass, outer_count, inner, nrec, alpha_evals, pad;
  double mu, reg, rho, elapsed, key;  // key: last recorded constraint violation (scheduling priority)
  double times[6];
};

// IterationRecord (solver.hpp:547-561).
struct DevRecord {
  int outer, accepted;
  double cost, cost_al, merit_before, merit_after, model_decrease, defect_l1, violation, alpha, mu,
      max_feedforward, regularization;
};

enum SolveStatus : int { kConverged = 0, kMaxIterations = 1, kError = 2 };
enum ErrorCode : int {
  kErrNone = 0,
  kErrRegCap = 1,           // "regularization exceeded its cap" (IndefiniteHessianError)
  kErrFactorization = 2,    // FactorizationError what() at reg cap
  kErrLineSearch = 3,       // "line search failed at maximum regularization"
  kErrLinearizeNonfinite = 4,
  kErrRolloutNonfinite = 5,  // nonlinear_rollout throws (uncaught in the reference)
  kErrAlphaLevels = 6,
  kErrDefectNonfinite = 7,     // linearize: non-finite defect (solver.hpp:142-145)
  kErrLinearizeTerminal = 8,   // linearize: non-finite terminal expansion (solver.hpp:102-105)
};

struct DevResult {  // SolveReport (solver.hpp:572-582) minus the records
  int status, error_code, error_node, inner_iterations, outer_iterations, n_records;
  double final_cost, final_violation, final_defect_l1;
  double times[6];  // setup, backward (all), 0, forward, line search, total [s]
  double final_penalty, final_mu, final_reg;
  double alpha_evals;  // step sizes evaluated by the line search (all passes)
};

// ------------------------------------------------------------------ topology
// Segment plan of a TreeTopology (tree.hpp:28-44), built on the host.
struct Topo {
  int n;                     // node count
  const int* parent;         // [n], -1 at the root
  const double* weight;      // [n]
  const int* first_child;    // [n], -1 at leaves (children are contiguous in BFS order)
  const int* nchild;         // [n]
  int ndepth;                // segment depth levels (root segment = depth 0)
  const int* depth_begin;    // [ndepth+1] segment ranges per depth
  const int* depth_len;      // [ndepth] segment length at each depth (balanced tree)
  const int* seg_off;        // [nseg+1] CSR offsets into seg_nodes
  const int* seg_nodes;      // node ids head -> tail
  const int* seg_stride;     // [nseg] constant node-index stride along the segment (0: use seg_nodes)
  const int* seg_scratch;    // [nseg] first scratch slot (2*len + 32 slots reserved)
  const int* node_seg;       // [n]
  const int* node_pos;       // [n]
  const int* seg_depth;      // [nseg] depth level of each segment
  int has_constraints;
  int max_con;               // constraint rows stored per node (eta stride)
  int n_shared;              // nodes 0..n_shared-1 have step <= N_b (the shared segment), 0 for a path
  int n_bound;               // boundary nodes n_shared.. (step N_b + 1: heads of the deepest segments)
};

// Per-instance device state (layout strides depend on NX, NU; see lqr.cuh).
struct Work {
  const double* x0;  // [NX]
  double* x;         // [n*NX]
  double* u;         // [n*NU]
  double* eta;       // [n*max_con]
  double* stage;     // [n*StageLayout::stride]
  double* defect;    // [n*NX]
  double* policy;    // [n*PolicyLayout::stride]
  double* bwd;       // [scratch*BwdLayout::stride]
  double* fwd;       // [scratch*FwdLayout::stride]
  double* dx;        // [n*NX]
  double* du;        // [n*NU]
  double* value;     // optional [n*ValueLayout::stride] (kernel-level API)
  DevRecord* records;
  int max_records;
  DevResult* result;
  double* prof;  // optional [kProfSlots] per-phase device time (ns), leader-accumulated
  DevResume* resume;  // optional suspend / resume state
  double* cond;       // condensed strategy scratch (per-node records, H, H copy, h, u, pivots), else null
};

}  // namespace bmpc_b200
