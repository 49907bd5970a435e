// Device-resident MSiLQR-Tree + augmented-Lagrangian solve (the hot path of
// bmpc::solve, solver.hpp:595-780), written once over an execution group:
//   * CtaGroup  — one thread block solves one instance (small trees, batches;
//                 barriers are __syncthreads, no host round trips);
//   * GridGroup — every block of a cooperative launch solves ONE large
//                 instance (barriers are grid.sync()).
// Every decision the reference takes on the host (convergence, merit weight,
// Armijo acceptance, Levenberg regularization, AL outer loop) is taken on
// device from deterministic fixed-order reductions, so a solve is one kernel
// launch.
//
// Backward pass = tree-segmented associative scan. The tree is cut into
// segments (maximal single-child chains ending at a branch node or a leaf).
// Depth levels are processed leaves-first; within a level all segments are
// scanned concurrently with the reference's own work-efficient tree schedule
// (scan.hpp:19-65). Leaf segments reproduce the reference P1 chain scan
// exactly (lqr_scan.hpp:123-141 with the terminal appended); segments ending
// at a branch node take the branch node's value from one Bellman step over
// the summed children (riccati.hpp:97-122) as their terminal — this is where
// the reference's sequential P2 becomes parallel. Forward pass = prefix scan
// of the closed-loop affine maps of every segment at once (lqr_scan.hpp:
// 177-187), then one depth sweep to apply them to the head perturbations.
#pragma once

#include <cooperative_groups.h>

#include <type_traits>

#include "linalg.cuh"
#include "lqr.cuh"
#include "model.cuh"
#include "types.h"

namespace bmpc_b200 {

namespace cg = cooperative_groups;

constexpr int kRedSlots = 4 * kMaxAlpha;  // largest simultaneous reduction
constexpr int kMaxWarps = 32;  // blocks of <= 1024 threads

// Scan level bookkeeping (scan.hpp:19-36): n_0 = E, n_{l+1} = ceil(n_l / 2).
__device__ __forceinline__ int level_size(int E, int l) {
  int s = E;
  for (int i = 0; i < l; ++i) s = (s + 1) >> 1;
  return s;
}
__device__ __forceinline__ int level_offset(int E, int l) {
  int off = 0, s = E;
  for (int i = 0; i < l; ++i) {
    off += s;
    s = (s + 1) >> 1;
  }
  return off;
}
__host__ __device__ __forceinline__ int up_steps(int E) {
  int u = 0;
  for (int s = E; s >= 2; s = (s + 1) >> 1) ++u;
  return u;
}

// Lanes per cooperative team (combine_bwd needs NX*NX, the Riccati step
// NU*NX + NU); 0 = one thread per combination, scan path only.
template <int NX, int NU>
__host__ __device__ constexpr int team_size() {
  constexpr int need = NX * NX > NU * NX + NU ? NX * NX : NU * NX + NU;
  return need <= 4 ? 4 : (need <= 16 ? 16 : (need <= 32 ? 32 : 0));
}

// ------------------------------------------------------------------ groups
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct RedSmem {
  double* part;  // [kRedSlots][nwarps] warp partials (dynamic shared memory)
  double total[kRedSlots];
  double prof[kProfSlots];  // profiling accumulators (leader), flushed to Work::prof once per launch
  int flag;
};

// Reductions are two-stage and deterministic: warps butterfly-reduce (every
// lane ends with the same bits) into per-warp slots; slots are then folded
// in a fixed order. Slot k < nsum are sums, the rest maxima.
// kBlock > 0: block size known at compile time (per-instance kernels), so
// strides, warp counts and slot offsets fold to immediates.
template <int kBlock = 0>
struct CtaGroupT {
  RedSmem* sm;
  __device__ static int bdim() { return kBlock > 0 ? kBlock : static_cast<int>(blockDim.x); }
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return bdim(); }
  __device__ int block() const { return 0; }
  __device__ int nblocks() const { return 1; }
  __device__ bool leader() const { return threadIdx.x == 0; }
  __device__ void sync() const { __syncthreads(); }
  // Items of a phase over `total` items: this thread's first / end / step,
  // and the uniform round count with the k-th round's item (see GridGroup).
  __device__ int item0(int) const { return threadIdx.x; }
  __device__ int item_end(int total) const { return total; }
  __device__ int item_step() const { return bdim(); }
  __device__ int item_rounds(int total) const { return (total + bdim() - 1) / bdim(); }
  __device__ int item_at(int, int k) const { return k * bdim() + threadIdx.x; }
  // Fold warp partials sm->part[0..nslot) into sm->total (all threads see it).
  __device__ void finish(int nslot, int nsum) const {
    __syncthreads();
    const int nw = (bdim() + 31) >> 5;
    for (int k = threadIdx.x; k < nslot; k += bdim()) {
      const double* pk = sm->part + k * nw;
      double a = pk[0];
      for (int w = 1; w < nw; ++w) a = k < nsum ? a + pk[w] : fmax(a, pk[w]);
      sm->total[k] = a;
    }
    __syncthreads();
  }
};
using CtaGroup = CtaGroupT<0>;

struct GridGroup {
  RedSmem* sm;
  __device__ static int bdim() { return blockDim.x; }
  double* scratch;  // [2][gridDim.x][kRedSlots] global partials (double-buffered)
  int* parity;      // per-block private counter lives in smem via sm->flag
  __device__ int rank() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ int size() const { return gridDim.x * blockDim.x; }
  __device__ int block() const { return blockIdx.x; }
  __device__ int nblocks() const { return gridDim.x; }
  __device__ bool leader() const { return blockIdx.x == 0 && threadIdx.x == 0; }
  __device__ void sync() const { cg::this_grid().sync(); }
  // Items of a phase: every block takes a contiguous chunk of ceil(total /
  // blocks) items, so a phase over fewer items than grid threads (cfg1's
  // 3,971 nodes vs 37,888 threads) spreads over every SM instead of filling
  // the first blocks, and a warp still reads consecutive nodes.
  __device__ int item_chunk(int total) const { return (total + gridDim.x - 1) / gridDim.x; }
  __device__ int item0(int total) const { return blockIdx.x * item_chunk(total) + threadIdx.x; }
  __device__ int item_end(int total) const { return min(total, (blockIdx.x + 1) * item_chunk(total)); }
  __device__ int item_step() const { return blockDim.x; }
  __device__ int item_rounds(int total) const { return (item_chunk(total) + blockDim.x - 1) / blockDim.x; }
  // Round k's item (>= item_end when this thread has none in that round).
  __device__ int item_at(int total, int k) const {
    const int i = blockIdx.x * item_chunk(total) + k * blockDim.x + threadIdx.x;
    return i < item_end(total) ? i : total;
  }
  __device__ void finish(int nslot, int nsum) const {
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    const int buf = sm->flag & 1;
    double* out = scratch + (static_cast<size_t>(buf) * gridDim.x + blockIdx.x) * kRedSlots;
    for (int k = threadIdx.x; k < nslot; k += blockDim.x) {
      const double* pk = sm->part + k * nw;
      double a = pk[0];
      for (int w = 1; w < nw; ++w) a = k < nsum ? a + pk[w] : fmax(a, pk[w]);
      out[k] = a;
    }
    cg::this_grid().sync();
    // Warp w folds slots w, w+nw, ... over blocks: lane-strided then butterfly.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* in = scratch + static_cast<size_t>(buf) * gridDim.x * kRedSlots;
    for (int k = warp; k < nslot; k += nw) {
      const bool is_sum = k < nsum;
      double a = is_sum ? 0.0 : -INFINITY;
      for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
        const double v = in[static_cast<size_t>(b) * kRedSlots + k];
        a = is_sum ? a + v : fmax(a, v);
      }
      a = is_sum ? warp_sum(a) : warp_max(a);
      if (lane == 0) sm->total[k] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) sm->flag += 1;
    __syncthreads();
  }
};

// Contribute this thread's value to slot k (every thread of the block must call).
template <class G>
__device__ __forceinline__ void red_put(const G& g, int k, double v, bool is_sum) {
  v = is_sum ? warp_sum(v) : warp_max(v);
  if ((threadIdx.x & 31) == 0) g.sm->part[k * (G::bdim() >> 5) + (threadIdx.x >> 5)] = v;
}

// Like red_put, but accumulates into the warp's slot (first: overwrite).
template <class G>
__device__ __forceinline__ void red_acc(const G& g, int k, double v, bool is_sum, bool first) {
  v = is_sum ? warp_sum(v) : warp_max(v);
  if ((threadIdx.x & 31) == 0) {
    double* slot = g.sm->part + k * (G::bdim() >> 5) + (threadIdx.x >> 5);
    *slot = first ? v : (is_sum ? *slot + v : fmax(*slot, v));
  }
}

// ------------------------------------------------------------------ solver
// kSeqOnly: every segment takes the team Riccati sweep / walk; the scan path
// (and its register footprint) is compiled out — used for batches of trees
// whose segments are all short (e.g. cfg0/cfg4).
// kTeam > 0 overrides the team width (32 = one warp per segment, for blocks
// of >= 128 threads where the shorter per-step stages pay).
// kNL: the single-shooting line search (ForwardMode::nonlinear_rollout) is
// compiled in — only into the kernels launched for that mode, so the
// multiple-shooting solve loop keeps its register allocation.
// kFeat: optional paths compiled in only where they are launched, so the
// default solve kernels keep their register allocation and instruction
// footprint: bit 0 the single-shooting line search, bit 1 the condensed
// shared segment (scan_condensed), bit 2 the chunked backward sweep.
constexpr int kFeatNL = 1, kFeatCond = 2, kFeatChunk = 4;
template <int NX, int NU, class G, bool kSeqOnly = false, int kTeam = 0, int kFeat = 0>
struct Solver {
  static constexpr bool kNL = (kFeat & kFeatNL) != 0;
  static constexpr bool kCond = (kFeat & kFeatCond) != 0;
  static constexpr bool kChunk = (kFeat & kFeatChunk) != 0;
  using SL = StageLayout<NX, NU>;
  using BL = BwdLayout<NX>;
  using FL = FwdLayout<NX>;
  using PL = PolicyLayout<NX, NU>;
  using VL = ValueLayout<NX>;

  G g;
  const Topo& t;
  const ModelParams& mp;
  // By value: the pointers become registers / private stack slots, so a
  // generic store can no longer force reloading them from the block's
  // shared-memory copy (which it might alias) before every access.
  const Work w;
  const DevOptions& o;
  double g_rho{0.0};  // current AL penalty (uniform across the group)
  double* wbuf{nullptr};  // forward-walk elements (aliases tsm; wcap elements of kWE doubles)
  int wcap{0};
  void* tsm{nullptr};  // [blockDim / kTS] team scratch slots of slot_bytes() (kernel-provided)

  __device__ Solver(G g_, const Topo& t_, const ModelParams& mp_, Work& w_, const DevOptions& o_)
      : g(g_), t(t_), mp(mp_), w(w_), o(o_) {}

  __device__ bool is_leaf(int i) const { return t.first_child[i] < 0; }
  // Unicycle with diagonal weights: stage records hold UniRec's variable
  // entries per pass over per-solve constants (model.cuh).
  __device__ bool structured() const { return NX == 4 && NU == 2 && mp.kind == kModelUnicycle && mp.w_diag; }
  // Compact structured records in the default batch kernels (kSeqOnly, no
  // optional paths): 22 doubles per node instead of the 58-double dense
  // record, so a pass touches ~1.5 cache lines of stage data per node
  // instead of ~4 (the main launch's working set exceeds the L2).
  __device__ bool compact() const {
    if constexpr (kSeqOnly && kFeat == 0 && NX == 4 && NU == 2) return structured();
    return false;
  }
  __device__ double* stage(int i) const {
    return w.stage + static_cast<size_t>(i) * (compact() ? kCompactStride : SL::stride);
  }
  // Dense-layout entry k of a record r (compact records: the variable entry or the implied constant).
  __device__ double rec_at(const double* r, int k) const {
    if constexpr (NX == 4 && NU == 2) {
      if (compact()) {
        const int e = uni_var_of_rt(k);
        return e >= 0 ? r[e] : unicycle_stage_constant(mp.dt, k);
      }
    }
    return r[k];
  }
  __device__ static int uni_var_of_rt(int k) {
    int e = -1;
#pragma unroll
    for (int q = 0; q < UniRec::kVar; ++q) e = (UniRec::pos(q) == k) ? q : e;
    return e;
  }
  __device__ double* bwd(int slot) const { return w.bwd + static_cast<size_t>(slot) * BL::stride; }
  __device__ double* fwd(int slot) const { return w.fwd + static_cast<size_t>(slot) * FL::stride; }
  __device__ double* pol(int i) const { return w.policy + static_cast<size_t>(i) * PL::stride; }
  __device__ int seg_len(int s) const { return t.seg_off[s + 1] - t.seg_off[s]; }
  __device__ int seg_node(int s, int k) const { return t.seg_nodes[t.seg_off[s] + k]; }
  // Node k of a segment without a dependent index load when the stride is constant.
  struct SegIdx {
    int off, head, stride;
  };
  __device__ SegIdx seg_idx(int s) const {
    const int off = t.seg_off[s];
    return {off, t.seg_nodes[off], t.seg_stride[s]};
  }
  __device__ int node_at(const SegIdx& q, int k) const {
    return q.stride ? q.head + k * q.stride : t.seg_nodes[q.off + k];
  }

  // Value of node i during/after the backward pass: slot (L-1-pos) of its
  // segment's level-0 array (the reversed suffix scan).
  __device__ const double* value_of(int i) const {
    const int s = t.node_seg[i];
    return bwd(t.seg_scratch[s] + seg_len(s) - 1 - t.node_pos[i]);
  }
  __device__ double* val(int i) const { return w.value + static_cast<size_t>(i) * VL::stride; }
  // Segments of at most seq_max_len nodes take the team Riccati sweep.
  // Backward strategy per depth level: team sweep for short segments, or for
  // many long ones at one depth; the associative scan otherwise (host mirror:
  // seq_depth_host).
  __device__ bool seq_depth(int d) const {
    if (kSeqOnly) return true;
    if (kTS <= 0 || o.seq_max_len <= 0) return false;
    const int L = t.depth_len[d], ns = t.depth_begin[d + 1] - t.depth_begin[d];
    if constexpr (std::is_same<G, GridGroup>::value) {
      // Whole-GPU kernel: a depth with few segments leaves most teams idle
      // under the sweep; the Hillis-Steele scan takes ceil(log2 L) barrier-
      // separated levels of ceil(ns L / teams) team combines instead of L - 1
      // dependent steps. Measured costs (cycles): 32-lane team Riccati step
      // ~1,450 in this kernel, 16-lane team combine ~8,000, grid barrier
      // ~3,000, elements ~10,000.
      if (hs_bwd_depth(d)) {
        const int teams = g.size() / kTSC;
        const int rounds = (ns * L + teams - 1) / teams;
        const int levels = 32 - __clz(L - 1);
        const long long hs = static_cast<long long>(levels) * (rounds * 8000 + 3000) + 10000;
        if (hs * 5 < static_cast<long long>(L - 1) * 1450 * 4) return false;
      }
    }
    return L <= o.seq_max_len || (o.seq_wide_segs > 0 && ns >= o.seq_wide_segs && L <= o.seq_wide_max);
  }
  __device__ bool seq_seg(int s) const { return kSeqOnly || seq_depth(t.seg_depth[s]); }
  // Forward strategy, independent of the backward one: the closed-loop walk
  // (O(L) dependent steps of ~100 cycles out of shared memory) beats the
  // prefix scan of affine maps (2 log L grid-synchronised levels) at every
  // segment length measured; fwd_scan_min > 0 restores the scan from that length.
  __device__ bool fwd_walk(int L) const { return kSeqOnly || o.fwd_scan_min <= 0 || L < o.fwd_scan_min; }
  // (P, p) of node i after the backward pass (either path); P at +0, p at +NX*NX.
  __device__ const double* value_ptr(int i) const {
    const int s = t.node_seg[i];
    return seq_seg(s) ? val(i) : value_of(i);
  }

  // ------------------------------------------------------ nonlinear rollout
  // nonlinear_rollout (problem.hpp:150-166): one thread walks each segment;
  // depth levels in order. Returns false on a non-finite state.
  __device__ bool rollout() {
    // Leaves carry no input (TrajectoryTree, tree.hpp:159-173).
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      if (is_leaf(i) || o.zero_inputs) {
#pragma unroll
        for (int j = 0; j < NU; ++j) w.u[i * NU + j] = 0.0;
      }
    }
    if (g.leader()) {
#pragma unroll
      for (int j = 0; j < NX; ++j) w.x[j] = w.x0[j];
    }
    g.sync();
    double bad = 0.0;
    for (int d = 0; d < t.ndepth; ++d) {
      const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
      for (int s = sb + g.rank(); s < se; s += g.size()) {
        const int L = seg_len(s);
        int prev = t.parent[seg_node(s, 0)];
        for (int k = 0; k < L; ++k) {
          const int i = seg_node(s, k);
          if (prev >= 0) {
            double xn[NX];
            node_dynamics<NX, NU>(mp, prev, w.x + prev * NX, w.u + prev * NU, xn);
            // First failing node in index order (the reference throws there,
            // problem.hpp:160-162): reduce max of (n - node).
            if (!all_finite<NX>(xn)) bad = fmax(bad, static_cast<double>(t.n - prev));
            copy<NX>(xn, w.x + i * NX);
          }
          prev = i;
        }
      }
      g.sync();
    }
    red_put(g, 0, bad, false);
    g.finish(1, 0);
    if (g.sm->total[0] > 0.0) {
      if (g.leader()) w.result->error_node = t.n - static_cast<int>(g.sm->total[0]);
      return false;
    }
    return true;
  }

  // ---------------------------------------------- evaluate (problem.hpp:109)
  // Sums into slots base..base+3: cost, cost_al, defect_l1 (sums), violation (max).
  // With alpha >= 0 evaluates the trial x + alpha dx, u + alpha du.
  __device__ void node_eval(int i, double alpha, double* c, double* cal, double* dl1, double* vmax,
                            double* defect_out = nullptr) const {
    const bool leaf = is_leaf(i);
    double x[NX], u[NU];
#pragma unroll
    for (int j = 0; j < NX; ++j) x[j] = alpha > 0.0 ? fma(alpha, w.dx[i * NX + j], w.x[i * NX + j]) : w.x[i * NX + j];
    if (!leaf) {
#pragma unroll
      for (int j = 0; j < NU; ++j)
        u[j] = alpha > 0.0 ? fma(alpha, w.du[i * NU + j], w.u[i * NU + j]) : w.u[i * NU + j];
    } else {
#pragma unroll
      for (int j = 0; j < NU; ++j) u[j] = 0.0;
    }
    double nc, pen, gm;
    node_cost<NX, NU>(mp, i, leaf, x, u, w.eta + static_cast<size_t>(i) * t.max_con, g_rho, &nc, &pen, &gm);
    const double wi = t.weight[i];
    *c = wi * nc;
    *cal = wi * (nc + pen);
    *vmax = gm;
    *dl1 = 0.0;
    const int p = t.parent[i];
    if (p >= 0) {
      double xp[NX], up[NU], f[NX];
#pragma unroll
      for (int j = 0; j < NX; ++j)
        xp[j] = alpha > 0.0 ? fma(alpha, w.dx[p * NX + j], w.x[p * NX + j]) : w.x[p * NX + j];
#pragma unroll
      for (int j = 0; j < NU; ++j)
        up[j] = alpha > 0.0 ? fma(alpha, w.du[p * NU + j], w.u[p * NU + j]) : w.u[p * NU + j];
      node_dynamics<NX, NU>(mp, p, xp, up, f);
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        const double dj = f[j] - x[j];
        if (defect_out) defect_out[j] = dj;
        s += fabs(dj);
      }
      *dl1 = s;
    } else if (defect_out) {
#pragma unroll
      for (int j = 0; j < NX; ++j) defect_out[j] = 0.0;
    }
  }

  struct Eval {
    double cost, cost_al, defect_l1, max_violation;
  };

  __device__ Eval evaluate_current() {
    double c = 0, cal = 0, dl = 0, vm = -INFINITY;
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      double a, b, d, v;
      node_eval(i, 0.0, &a, &b, &d, &v);
      c += a;
      cal += b;
      dl += d;
      vm = fmax(vm, v);
    }
    red_put(g, 0, c, true);
    red_put(g, 1, cal, true);
    red_put(g, 2, dl, true);
    red_put(g, 3, vm, false);
    g.finish(4, 3);
    return {g.sm->total[0], g.sm->total[1], g.sm->total[2], fmax(g.sm->total[3], 0.0)};
  }

  // ------------------------------------ linearize + evaluate (fused, Phase L)
  // Returns the nominal evaluation. On a non-finite expansion or defect,
  // *bad_node = 1 + the node the reference throws at and *bad_code its error
  // (linearize, solver.hpp:76-149: every node's expansion is checked in index
  // order first, then every defect): the smallest failing expansion node, else
  // the smallest failing defect node.
  __device__ Eval linearize_evaluate(int* bad_node, int* bad_code) {
    double c = 0, cal = 0, dl = 0, vm = -INFINITY, bad = 0, badd = 0;
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      const bool leaf = is_leaf(i);
      const double* eta = w.eta + static_cast<size_t>(i) * t.max_con;
      const bool ok = node_linearize<NX, NU>(mp, i, leaf, t.weight[i], w.x + i * NX, w.u + i * NU, eta, g_rho,
                                             stage(i), compact());
      double a, b, d, v;
      // Nominal evaluate terms and the edge defect parent -> i
      // (models.defect, solver.hpp:138-147) from one dynamics evaluation.
      node_eval(i, 0.0, &a, &b, &d, &v, w.defect + i * NX);
      c += a;
      cal += b;
      dl += d;
      vm = fmax(vm, v);
      const bool dok = all_finite<NX>(w.defect + i * NX);
      if (!ok) bad = fmax(bad, static_cast<double>(t.n - i));
      if (!dok) badd = fmax(badd, static_cast<double>(t.n - i));
    }
    red_put(g, 0, c, true);
    red_put(g, 1, cal, true);
    red_put(g, 2, dl, true);
    red_put(g, 3, vm, false);
    red_put(g, 4, bad, false);
    red_put(g, 5, badd, false);
    g.finish(6, 3);
    const int be = static_cast<int>(g.sm->total[4]), bd = static_cast<int>(g.sm->total[5]);
    *bad_node = be > 0 ? t.n - be + 1 : (bd > 0 ? t.n - bd + 1 : 0);
    *bad_code = be > 0 ? (is_leaf(t.n - be) ? kErrLinearizeTerminal : kErrLinearizeNonfinite)
                       : kErrDefectNonfinite;
    return {g.sm->total[0], g.sm->total[1], g.sm->total[2], fmax(g.sm->total[3], 0.0)};
  }

  // ------------------------------------------------ tree scan machinery
  // Items of a per-segment phase over the segments of one depth level.
  template <class F>
  __device__ void for_depth_items(int d, int per_seg, F&& f) const {
    const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
    const int total = (se - sb) * per_seg;
    for (int q = g.item0(total), q_e = g.item_end(total); q < q_e; q += g.item_step()) f(sb + q / per_seg, q % per_seg);
  }

  // Backward suffix scan of segments at depth d, elements already in level 0
  // (reversed). f(a, b) = combine_bwd(first = b, second = a).
  // Team size of the cooperative combine (0: one thread per combination).
  static constexpr int kTS = kTeam > 0 ? kTeam : team_size<NX, NU>();
  // Team size of the scan's combines: the 16-lane teams the shared-memory
  // slots are sized for (twice the teams of the 32-lane sweep in the
  // 256-thread and whole-GPU kernels; a combine needs only NX*NX lanes).
  static constexpr int kTSC = team_size<NX, NU>() > 0 ? team_size<NX, NU>() : kTS;

  // Items of a per-segment phase, one kTSC-lane team per item.
  template <class F>
  __device__ void for_depth_items_team(int d, int per_seg, F&& f) const {
    const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
    const int total = (se - sb) * per_seg;
    const int team = g.rank() / kTSC, nteams = g.size() / kTSC;
    const int lane = threadIdx.x % kTSC;
    const unsigned mask =
        kTSC == 32 ? 0xffffffffu : (((1u << kTSC) - 1u) << ((threadIdx.x & 31) / kTSC * kTSC));
    for (int q = team; q < total; q += nteams) f(sb + q / per_seg, q % per_seg, lane, mask);
  }

  // Backward suffix scan of segments at depth d, elements already in level 0
  // (reversed). f(a, b) = combine_bwd(first = b, second = a).
  // Hillis-Steele form of the same suffix scan for depths whose elements fit
  // the group's teams in a couple of rounds (cfg1's 4 x 990 on the whole
  // grid): ceil(log2 E) levels of S_j = f(S_{j-o}, S_j) ping-ponged between
  // slots [0, E) and [E, 2E), one barrier per level, instead of the
  // work-efficient pairing's 2 log2 E barriers.
  __device__ bool hs_bwd_depth(int d) const {
    if constexpr (kTSC <= 0) return false;
    const int E = t.depth_len[d], ns = t.depth_begin[d + 1] - t.depth_begin[d];
    return o.bwd_hs > 0 && E >= 4 && ns * E <= o.bwd_hs * (g.size() / max(kTSC, 1));
  }
  __device__ int scan_bwd_depth_hs(int d) {
    const int E = t.depth_len[d];
    int err = kBwdOk;
    if constexpr (kTSC > 0) {
      TeamSmem<NX>& my = comb_smem();
      int src = 0;
      for (int off = 1; off < E; off <<= 1) {
        const int dst = E - src;  // the other half
        for_depth_items_team(d, E, [&](int s, int j, int lane, unsigned mask) {
          const int base = t.seg_scratch[s];
          double* out = bwd(base + dst + j);
          if (j >= off) {
            const int e = team_combine_bwd<NX, kTSC>(bwd(base + src + j), bwd(base + src + j - off), out, lane,
                                                     mask, my);
            err = err ? err : e;
          } else {
            const double* in = bwd(base + src + j);
            for (int k = lane; k < BL::size; k += kTSC) out[k] = in[k];
          }
        });
        g.sync();
        src = dst;
      }
      if (src != 0) {  // results back to slots [0, E) (value_of reads them there)
        for_depth_items_team(d, E, [&](int s, int j, int lane, unsigned) {
          const int base = t.seg_scratch[s];
          const double* in = bwd(base + src + j);
          double* out = bwd(base + j);
          for (int k = lane; k < BL::size; k += kTSC) out[k] = in[k];
        });
        g.sync();
      }
    }
    return err;
  }

  __device__ int scan_bwd_depth(int d) {
    if (hs_bwd_depth(d)) return scan_bwd_depth_hs(d);
    const int E = t.depth_len[d];
    const int U = up_steps(E);
    int err = kBwdOk;
    if constexpr (kTSC > 0) {
      TeamSmem<NX>& my = comb_smem();
      for (int l = 0; l < U; ++l) {
        const int nl = level_size(E, l), nn = (nl + 1) >> 1;
        const int ol = level_offset(E, l), on = ol + nl;
        for_depth_items_team(d, nn, [&](int s, int i, int lane, unsigned mask) {
          const int base = t.seg_scratch[s];
          double* dst = bwd(base + on + i);
          if (2 * i + 1 < nl) {
            const int e = team_combine_bwd<NX, kTSC>(bwd(base + ol + 2 * i + 1), bwd(base + ol + 2 * i), dst, lane,
                                                     mask, my);
            err = err ? err : e;
          } else {
            const double* src = bwd(base + ol + 2 * i);
            for (int k = lane; k < BL::size; k += kTSC) dst[k] = src[k];
          }
        });
        g.sync();
      }
      for (int l = U - 1; l >= 0; --l) {
        const int nl = level_size(E, l), nn = (nl + 1) >> 1;
        const int ol = level_offset(E, l), on = ol + nl;
        for_depth_items_team(d, nn, [&](int s, int i, int lane, unsigned mask) {
          const int base = t.seg_scratch[s];
          const double* S = bwd(base + on);
          if (2 * i + 1 < nl) {
            const double* src = S + static_cast<size_t>(i) * BL::stride;
            double* dst = bwd(base + ol + 2 * i + 1);
            for (int k = lane; k < BL::size; k += kTSC) dst[k] = src[k];
          }
          if (i >= 1) {
            double* a = bwd(base + ol + 2 * i);
            const int e = team_combine_bwd<NX, kTSC>(a, S + static_cast<size_t>(i - 1) * BL::stride, a, lane, mask, my);
            err = err ? err : e;
          }
        });
        g.sync();
      }
      return err;
    }
    for (int l = 0; l < U; ++l) {
      const int nl = level_size(E, l), nn = (nl + 1) >> 1;
      const int ol = level_offset(E, l), on = ol + nl;
      for_depth_items(d, nn, [&](int s, int i) {
        const int base = t.seg_scratch[s];
        double* dst = bwd(base + on + i);
        if (2 * i + 1 < nl) {
          double res[BL::size];
          const int e = combine_bwd<NX>(bwd(base + ol + 2 * i + 1), bwd(base + ol + 2 * i), res);
          err = err ? err : e;
          copy<BL::size>(res, dst);
        } else {
          copy<BL::size>(bwd(base + ol + 2 * i), dst);
        }
      });
      g.sync();
    }
    for (int l = U - 1; l >= 0; --l) {
      const int nl = level_size(E, l), nn = (nl + 1) >> 1;
      const int ol = level_offset(E, l), on = ol + nl;
      for_depth_items(d, nn, [&](int s, int i) {
        const int base = t.seg_scratch[s];
        const double* S = bwd(base + on);
        if (2 * i + 1 < nl) copy<BL::size>(S + static_cast<size_t>(i) * BL::stride, bwd(base + ol + 2 * i + 1));
        if (i >= 1) {
          double res[BL::size];
          double* a = bwd(base + ol + 2 * i);
          const int e = combine_bwd<NX>(a, S + static_cast<size_t>(i - 1) * BL::stride, res);
          err = err ? err : e;
          copy<BL::size>(res, a);
        }
      });
      g.sync();
    }
    return err;
  }

  // ---------------------------------------------------- backward pass (B)
  __device__ unsigned team_mask() const {
    return kTS == 32 ? 0xffffffffu : (((1u << kTS) - 1u) << ((threadIdx.x & 31) / kTS * kTS));
  }
  __device__ RicSmem<NX, NU>& ric_smem() const {
    return *reinterpret_cast<RicSmem<NX, NU>*>(reinterpret_cast<unsigned char*>(tsm) + (threadIdx.x / kTS) * slot_bytes());
  }
  __device__ TeamSmem<NX>& comb_smem() const {
    return *reinterpret_cast<TeamSmem<NX>*>(reinterpret_cast<unsigned char*>(tsm) + (threadIdx.x / kTSC) * slot_bytes());
  }
  __host__ __device__ static constexpr size_t slot_bytes() {
    constexpr size_t a = sizeof(TeamSmem<NX>) > sizeof(RicSmem<NX, NU>) ? sizeof(TeamSmem<NX>) : sizeof(RicSmem<NX, NU>);
    constexpr size_t b = sizeof(double) * RicFlat<NX, NU>::size;
    return ((a > b ? a : b) + 15) / 16 * 16;  // 16-byte aligned slots (vector loads)
  }

  // Team Bellman steps along one segment, nodes k_hi down to k_lo (positions
  // in the segment), starting from the value of node k_hi + 1 already staged
  // in the team's flat array Fm (P, PT, p). The next node's stage record and
  // edge offset are prefetched into registers while each step computes.
  // Values are stored at the segment head (the parent's branch step reads
  // them) or everywhere with keep_values; policies always.
  template <int TS>
  __device__ int team_chain(const SegIdx& sq, int k_hi, int k_lo, double reg, int lane, unsigned mask, double* Fm) {
    using F = RicFlat<NX, NU>;
    constexpr int PRE = (SL::size + TS - 1) / TS;
    int err = kBwdOk;
    __syncwarp(mask);
    if constexpr (NX == 4 && NU == 2) {
      if (compact()) return team_chain_compact<TS>(sq, k_hi, k_lo, reg, lane, mask, Fm);
    }
    {
      const double* s0 = stage(node_at(sq, k_hi));
      for (int k = lane; k < SL::size; k += TS) Fm[F::S + k] = s0[k];
      if (lane < NX) Fm[F::c + lane] = w.defect[node_at(sq, k_hi + 1) * NX + lane];
    }
    // Base pointers in registers: the step's generic stores could alias the
    // shared-memory Work struct, which would force a reload every step.
    const double* const stg = w.stage;
    const double* const dfc = w.defect;
    double* const vbase = w.value;
    double* const pbase = w.policy;
    for (int k = k_hi; k >= k_lo; --k) {
      const int i = node_at(sq, k);
      double pre[PRE];
      double prec = 0.0;
      if (k > k_lo) {
        const double* sp = stg + static_cast<size_t>(node_at(sq, k - 1)) * SL::stride;
#pragma unroll
        for (int j = 0; j < PRE; ++j) {
          const int idx = lane + j * TS;
          pre[j] = idx < SL::size ? sp[idx] : 0.0;
        }
        if (lane < NX) prec = dfc[i * NX + lane];
      }
      double* const vi = (k == 0 || o.keep_values) ? vbase + static_cast<size_t>(i) * VL::stride : nullptr;
      const int e = team_riccati_step_u<NX, NU, TS>(reg, mask, Fm, lane, vi, pbase + static_cast<size_t>(i) * PL::stride);
      err = err ? err : e;
      if (k > k_lo) {
        // No barrier needed: every lane passed the step's stage-2 __syncwarp,
        // after which nothing reads the stage record; the next step opens
        // with one before it reads what is staged here.
#pragma unroll
        for (int j = 0; j < PRE; ++j) {
          const int idx = lane + j * TS;
          if (idx < SL::size) Fm[F::S + idx] = pre[j];
        }
        if (lane < NX) Fm[F::c + lane] = prec;
      }
    }
    return err;
  }

  // team_chain over compact structured records: the constant entries of the
  // dense record are staged once, then each step stages only the 22 variable
  // entries (each lane's destination offsets held in registers).
  template <int TS>
  __device__ int team_chain_compact(const SegIdx& sq, int k_hi, int k_lo, double reg, int lane, unsigned mask,
                                    double* Fm) {
    using F = RicFlat<NX, NU>;
    constexpr int PRE = (UniRec::kVar + TS - 1) / TS;
    int err = kBwdOk;
    for (int k = lane; k < SL::size; k += TS)
      if (uni_var_of_rt(k) < 0) Fm[F::S + k] = unicycle_stage_constant(mp.dt, k);
    int dst[PRE];
#pragma unroll
    for (int j = 0; j < PRE; ++j) {
      const int idx = lane + j * TS;
      dst[j] = idx < UniRec::kVar ? kUniPosTab[idx] : 0;
    }
    {
      const double* s0 = stage(node_at(sq, k_hi));
#pragma unroll
      for (int j = 0; j < PRE; ++j)
        if (lane + j * TS < UniRec::kVar) Fm[F::S + dst[j]] = s0[lane + j * TS];
      if (lane < NX) Fm[F::c + lane] = w.defect[node_at(sq, k_hi + 1) * NX + lane];
    }
    const double* const stg = w.stage;
    const double* const dfc = w.defect;
    double* const vbase = w.value;
    double* const pbase = w.policy;
    for (int k = k_hi; k >= k_lo; --k) {
      const int i = node_at(sq, k);
      double pre[PRE];
      double prec = 0.0;
      if (k > k_lo) {
        const double* sp = stg + static_cast<size_t>(node_at(sq, k - 1)) * kCompactStride;
#pragma unroll
        for (int j = 0; j < PRE; ++j) {
          const int idx = lane + j * TS;
          pre[j] = idx < UniRec::kVar ? sp[idx] : 0.0;
        }
        if (lane < NX) prec = dfc[i * NX + lane];
      }
      double* const vi = (k == 0 || o.keep_values) ? vbase + static_cast<size_t>(i) * VL::stride : nullptr;
      const int e = team_riccati_step_u<NX, NU, TS>(reg, mask, Fm, lane, vi, pbase + static_cast<size_t>(i) * PL::stride);
      err = err ? err : e;
      if (k > k_lo) {
        // No barrier needed: every lane passed the step's stage-2 __syncwarp,
        // after which nothing reads the stage record; the next step opens
        // with one before it reads what is staged here.
#pragma unroll
        for (int j = 0; j < PRE; ++j)
          if (lane + j * TS < UniRec::kVar) Fm[F::S + dst[j]] = pre[j];
        if (lane < NX) Fm[F::c + lane] = prec;
      }
    }
    return err;
  }

  // ----------------------------------------- chunked (time-parallel) sweep
  // Block-local backward pass of the segments of depth d when the block has
  // more teams than the depth has segments: each segment is cut into J chunks
  // of Ck positions and
  //   A) every chunk folds its one-step elements (init_bwd_element, the
  //      terminal embedded at the last position) with combine_bwd
  //      (lqr_scan.hpp:28-111) into one chunk element G_j (one team per chunk);
  //   B) one team per segment forms the suffixes S_j = G_j (+) S_{j+1} of the
  //      chunk elements (J - 1 combinations), so the value function at every
  //      chunk boundary is known (the (P, p) of S_j, backward_scan,
  //      lqr_scan.hpp:123-141);
  //   C) every chunk runs its Bellman steps from the value at its right
  //      boundary (team_chain), producing the policies (feedback_from_values
  //      + the value update) and the head values.
  // Latency ~(Ck - 1 + J - 1) combinations + Ck steps instead of L - 1 steps:
  // the time-parallel form of the reference's P1 scan with only block
  // barriers between the phases.
  // Chunk length: a combination costs ~2.5 Bellman steps, so the latency
  // ~2.5 (Ck + J) + Ck with J = L / Ck is least near Ck = sqrt(0.7 L); J is
  // capped by the teams the depth can give each segment (block teams in a
  // CtaGroup, every block's in a GridGroup) so one round covers all chunks.
  static constexpr int kTC = team_size<NX, NU>();  // 16-lane teams (the allocated team slots)
  __device__ int chunk_count(int d) const {
    if (kTC <= 0 || G::bdim() < 256 || o.chunk_bwd <= 0) return 1;
    const int L = t.depth_len[d], ns = t.depth_begin[d + 1] - t.depth_begin[d];
    if (L < 8 || L < o.chunk_bwd) return 1;
    const int ck = max(4, static_cast<int>(sqrtf(0.7f * static_cast<float>(L))));
    const int J = min((g.size() / kTC) / max(ns, 1), min((L + ck - 1) / ck, L / 4));
    return J >= 2 ? J : 1;
  }

  __device__ int chunked_bwd_depth(int d, double reg) {
    int err = kBwdOk;
    if constexpr (kTC > 0) {
      using F = RicFlat<NX, NU>;
      const int L = t.depth_len[d];
      const int sb = t.depth_begin[d], se = t.depth_begin[d + 1], ns = se - sb;
      int J = chunk_count(d);
      const int Ck = (L + J - 1) / J;
      J = (L + Ck - 1) / Ck;
      // Element of position pos (chain step pos, the terminal at L - 1) in
      // slot L - 1 - pos; chunk elements G_j in slots L + j, suffixes S_j in L + J + j.
      // 0a: terminals (regularized leaf cost / branch-node Bellman step over the summed children).
      for_depth_items(d, 1, [&](int s, int) {
        const int b = seg_node(s, L - 1);
        double P[NX * NX], p[NX];
        if (is_leaf(b)) {
          copy<NX * NX>(stage(b) + SL::Q, P);
          copy<NX>(stage(b) + SL::q, p);
#pragma unroll
          for (int j = 0; j < NX; ++j) P[j + j * NX] += reg;
        } else {
          double Pn[NX * NX], pn[NX];
#pragma unroll
          for (int j = 0; j < NX * NX; ++j) Pn[j] = 0.0;
#pragma unroll
          for (int j = 0; j < NX; ++j) pn[j] = 0.0;
          const int c0 = t.first_child[b], nc = t.nchild[b];
          for (int ch = c0; ch < c0 + nc; ++ch) {
            const double* v = value_ptr(ch);
            double Pd[NX];
            mv<NX, NX>(v, w.defect + ch * NX, Pd);
#pragma unroll
            for (int j = 0; j < NX * NX; ++j) Pn[j] += v[j];
#pragma unroll
            for (int j = 0; j < NX; ++j) pn[j] += v[NX * NX + j] + Pd[j];
          }
          const int e = riccati_step<NX, NU>(stage(b), reg, Pn, pn, P, p, pol(b) + PL::K, pol(b) + PL::k);
          err = err ? err : e;
        }
        if (o.keep_values) {
          copy<NX * NX>(P, val(b) + VL::P);
          copy<NX>(p, val(b) + VL::p);
        }
        embed_terminal<NX>(P, p, bwd(t.seg_scratch[s] + 0));
      });
      // 0b: one-step elements of the chain nodes (chain_stage, solver.hpp:189-193).
      for_depth_items(d, L - 1, [&](int s, int k) {
        const int i = seg_node(s, k), nxt = seg_node(s, k + 1);
        const int e = init_bwd_element<NX, NU>(stage(i), reg, w.defect + nxt * NX, bwd(t.seg_scratch[s] + L - 1 - k));
        err = err ? err : e;
      });
      g.sync();
      const int team = g.rank() / kTC, nteams = g.size() / kTC, lane = threadIdx.x % kTC;
      const unsigned mask = kTC == 32 ? 0xffffffffu : (((1u << kTC) - 1u) << ((threadIdx.x & 31) / kTC * kTC));
      unsigned char* slot = reinterpret_cast<unsigned char*>(tsm) + (threadIdx.x / kTC) * slot_bytes();  // block-local slot
      TeamSmem<NX>& cs = *reinterpret_cast<TeamSmem<NX>*>(slot);
      // A: chunk elements.
      for (int q = team; q < ns * J; q += nteams) {
        const int s = sb + q / J, j = q % J, base = t.seg_scratch[s];
        const int a = j * Ck, b = min(L, a + Ck);
        __syncwarp(mask);
        for (int k = lane; k < BL::size; k += kTC) cs.e2[k] = bwd(base + L - 1 - (b - 1))[k];
        for (int pos = b - 2; pos >= a; --pos) {
          const int e = team_combine_bwd<NX, kTC>(bwd(base + L - 1 - pos), cs.e2, cs.e2, lane, mask, cs);
          err = err ? err : e;
        }
        __syncwarp(mask);
        for (int k = lane; k < BL::size; k += kTC) bwd(base + L + j)[k] = cs.e2[k];
      }
      g.sync();
      // B: suffixes of the chunk elements, S_{J-1} .. S_1 (S_0 is not needed).
      for (int q = team; q < ns; q += nteams) {
        const int base = t.seg_scratch[sb + q];
        __syncwarp(mask);
        for (int k = lane; k < BL::size; k += kTC) {
          const double v = bwd(base + L + J - 1)[k];
          cs.e2[k] = v;
          bwd(base + L + J + J - 1)[k] = v;
        }
        for (int j = J - 2; j >= 1; --j) {
          const int e = team_combine_bwd<NX, kTC>(bwd(base + L + j), cs.e2, cs.e2, lane, mask, cs);
          err = err ? err : e;
          __syncwarp(mask);
          for (int k = lane; k < BL::size; k += kTC) bwd(base + L + J + j)[k] = cs.e2[k];
        }
      }
      g.sync();
      // C: Bellman steps of every chunk from the value at its right boundary.
      double* Fm = reinterpret_cast<double*>(slot);
      for (int q = team; q < ns * J; q += nteams) {
        const int s = sb + q / J, j = q % J, base = t.seg_scratch[s];
        const int a = j * Ck, b = min(L, a + Ck);
        const SegIdx sq = seg_idx(s);
        // Value at position b (chunk j + 1's head), or the terminal itself.
        const double* vb = j == J - 1 ? bwd(base + 0) : bwd(base + L + J + j + 1);
        __syncwarp(mask);
        for (int k = lane; k < NX * NX; k += kTC) ric_put_P<NX, NU>(Fm, k, vb[BL::P + k]);
        for (int k = lane; k < NX; k += kTC) Fm[F::p + k] = vb[BL::p + k];
        if (lane < NX) Fm[F::ZERO + lane] = 0.0;
        const int k_hi = (j == J - 1 ? L - 1 : b) - 1;
        if (k_hi >= a) {
          const int e = team_chain<kTC>(sq, k_hi, a, reg, lane, mask, Fm);
          err = err ? err : e;
        }
      }
    }
    g.sync();
    return err;
  }

  // Team Riccati sweep of every (short) segment at depth d: terminal (leaf
  // cost + reg, or the branch-node step over the summed children), then the
  // chain nodes tail -> head. Produces values (w.value) and policies.
  __device__ int riccati_sweep_depth(int d, double reg) {
    if constexpr (kChunk) {
      if (chunk_count(d) > 1) return chunked_bwd_depth(d, reg);
    }
    int err = kBwdOk;
    if constexpr (kTS > 0) {
      using F = RicFlat<NX, NU>;
      const int L = t.depth_len[d];
      const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
      const int team = g.rank() / kTS, nteams = g.size() / kTS, lane = threadIdx.x % kTS;
      const unsigned mask = team_mask();
      double* Fm = reinterpret_cast<double*>(&ric_smem());
      constexpr int PRE = (SL::size + kTS - 1) / kTS;
      for (int s = sb + team; s < se; s += nteams) {
        const SegIdx sq = seg_idx(s);
        const int b = node_at(sq, L - 1);
        __syncwarp(mask);
        if (lane < NX) Fm[F::ZERO + lane] = 0.0;
        if (is_leaf(b)) {
          // Values are read back only at segment heads (the parent's branch
          // step); the kernel-level API keeps every node's.
          const bool keep = o.keep_values || L == 1;
          for (int k = lane; k < NX * NX; k += kTS) {
            const double v = rec_at(stage(b), SL::Q + k) + ((k % (NX + 1)) == 0 ? reg : 0.0);
            ric_put_P<NX, NU>(Fm, k, v);
            if (keep) val(b)[VL::P + k] = v;
          }
          for (int k = lane; k < NX; k += kTS) {
            const double v = rec_at(stage(b), SL::q + k);
            Fm[F::p + k] = v;
            if (keep) val(b)[VL::p + k] = v;
          }
        } else {
          // riccati_tree_from (riccati.hpp:112-116): children in index order.
          const int c0 = t.first_child[b], nc = t.nchild[b];
          for (int k = lane; k < NX * NX; k += kTS) {
            double a = 0.0;
            for (int ch = c0; ch < c0 + nc; ++ch) a += value_ptr(ch)[k];
            ric_put_P<NX, NU>(Fm, k, a);
          }
          for (int k = lane; k < NX; k += kTS) {
            double a = 0.0;
            for (int ch = c0; ch < c0 + nc; ++ch) {
              const double* v = value_ptr(ch);
              double pd = 0.0;
#pragma unroll
              for (int l = 0; l < NX; ++l) pd = fma(v[k + l * NX], w.defect[ch * NX + l], pd);
              a += v[NX * NX + k] + pd;
            }
            Fm[F::p + k] = a;
          }
          for (int k = lane; k < SL::size; k += kTS) Fm[F::S + k] = rec_at(stage(b), k);
          if (lane < NX) Fm[F::c + lane] = 0.0;
          const int e = team_riccati_step_u<NX, NU, kTS>(reg, mask, Fm, lane,
                                                         (o.keep_values || L == 1) ? val(b) : nullptr, pol(b));
          err = err ? err : e;
        }
        // Chain nodes tail -> head.
        long long tc0 = 0;
        if (w.prof && threadIdx.x == 0) tc0 = clock64();
        if (L >= 2) {
          const int e = team_chain<kTS>(sq, L - 2, 0, reg, lane, mask, Fm);
          err = err ? err : e;
        }
        if (w.prof && threadIdx.x == 0 && L >= 2) {  // diagnostic: cycles per chain step
          g.sm->prof[12] += static_cast<double>(clock64() - tc0);
          g.sm->prof[13] += L - 1;
        }
      }
    }
    g.sync();
    return err;
  }

  // backward_pass (solver.hpp:203-318) with Levenberg shift `reg` on R
  // (non-leaves) and P (leaves). Depth levels leaves-first; each level by the
  // team Riccati sweep (short segments) or the associative scan (long ones).
  // Returns error code and max_feedforward.
  // ------------------------------------------- condensed P2 ("hypmsilqr")
  // backward_pass with BackwardStrategy::scan_condensed (solver.hpp:297-307):
  // P1 (the leaf segments, steps > N_b) as in the tree scan; the shared
  // segment (nodes 0..m-1, steps <= N_b) is condensed against the P1 values at
  // the boundary nodes (step N_b + 1) into one dense QP over the stacked
  // shared inputs, min 1/2 u'Hu + h'u (condense_tree, condensed.hpp:205-279),
  // solved by solve_dense (condensed.hpp:122-137: Cholesky, pivoted LU when
  // H is not positive definite, residual bound 1e-9 (|H| |u| + |h|) else
  // FactorizationError), and every shared node gets the open-loop policy
  // K = 0, k = u (solver.hpp:301-307).
  // H and h are formed on the tree instead of per root-to-boundary path: with
  // z the zero-input perturbation (z_0 = dx0, z_ch = A z + d_ch), V_j the
  // cost-to-go Hessian without control (V_b = P_b at the boundary,
  // V_i = Q_i + A_i' (sum_ch V_ch) A_i), lam_j its gradient, and
  // S_ba = dx_b / du_a = (A_{..} ... A_{a's child}) B_a for an ancestor a of b:
  //   H_aa = R_a + B_a' Vs_a B_a,  H_ab = S_ba' (A_b' Vs_b B_b + M_b'),
  //   h_a  = B_a' lams_a + M_a z_a + r_a,
  // which is G' diag(H^p) G / G' stack(h^p) of condense_tree (the per-path
  // split of the shared costs by multiplicity sums back to each cost once).
  struct CondL {  // per-node scratch record of nodes [0, m + nb)
    static constexpr int z = 0, V = NX, lam = V + NX * NX, Vs = lam + NX, lams = Vs + NX * NX, W = lams + NX,
                         size = W + NX * NU, stride = (size + 1) & ~1;
  };
  __device__ double* crec(int i) const { return w.cond + static_cast<size_t>(i) * CondL::stride; }
  __device__ int cond_n() const { return t.n_shared * NU; }
  __device__ double* cH() const { return w.cond + static_cast<size_t>(t.n_shared + t.n_bound) * CondL::stride; }
  __device__ double* cHc() const { return cH() + static_cast<size_t>(cond_n()) * cond_n(); }
  __device__ double* ch() const { return cHc() + static_cast<size_t>(cond_n()) * cond_n(); }
  __device__ double* cu() const { return ch() + cond_n(); }
  __device__ double* cpiv() const { return cu() + cond_n(); }
  __device__ double* cflag() const { return cpiv() + cond_n(); }

  // Stage blocks of a non-leaf node (structured records: constants included).
  __device__ void load_QRMqr(int i, double* Q, double* R, double* M, double* q, double* r) const {
    const double* si = stage(i);
    copy<NX * NX>(si + SL::Q, Q);
    copy<NU * NU>(si + SL::R, R);
    copy<NU * NX>(si + SL::M, M);
    copy<NX>(si + SL::q, q);
    copy<NU>(si + SL::r, r);
  }

  // solve_dense (condensed.hpp:122-137) over the whole group: u = -H^-1 h
  // with H = cHc() (symmetric, both triangles). Eigen::LLT as a right-looking
  // column Cholesky (each column: scale, then the trailing rank-1 update, one
  // warp per trailing column so the column-major rows stream coalesced; the
  // pivot sqrt is recomputed by every thread, so two group barriers per
  // column), the two triangular solves with one barrier per column. A
  // non-positive pivot (LLT info() != Success) falls back to
  // Eigen::PartialPivLU on one block. Returns kBwdOk or kFactorization
  // (non-finite u or residual |Hu + h| > 1e-9 (|H|_F |u| + |h|)); u in cu().
  __device__ int dense_solve() {
    const int n = cond_n();
    double* H = cH();
    double* Hc = cHc();
    double* h = ch();
    double* u = cu();
    double* y = cpiv();  // forward-solve workspace (pivots in the LU fallback)
    double* dg = cflag() + 2;  // [n] Cholesky diagonal
    auto at = [n](double* A, int i, int j) -> double& { return A[i + static_cast<size_t>(j) * n]; };
    const int rank = g.rank(), size = g.size();
    const int gw = rank >> 5, nw = size >> 5, lane = threadIdx.x & 31;
    for (int k = rank; k < n * n; k += size) H[k] = Hc[k];
    for (int k = rank; k < n; k += size) u[k] = -h[k];
    g.sync();
    bool llt_ok = true;
    for (int k = 0; k < n; ++k) {
      const double d = at(H, k, k);
      if (!(d > 0.0)) {
        llt_ok = false;  // every thread reads the same value: a uniform exit
        break;
      }
      const double lkk = sqrt(d);
      if (rank == 0) dg[k] = lkk;
      for (int i = k + 1 + rank; i < n; i += size) at(H, i, k) /= lkk;
      g.sync();
      for (int j = k + 1 + gw; j < n; j += nw) {
        const double ljk = at(H, j, k);
        for (int i = j + lane; i < n; i += 32) at(H, i, j) = fma(-at(H, i, k), ljk, at(H, i, j));
      }
      g.sync();
    }
    if (llt_ok) {
      for (int k = 0; k < n; ++k) {  // L y = -h
        const double yk = u[k] / dg[k];
        if (rank == 0) y[k] = yk;
        for (int i = k + 1 + rank; i < n; i += size) u[i] = fma(-at(H, i, k), yk, u[i]);
        g.sync();
      }
      for (int k = n - 1; k >= 0; --k) {  // L' u = y
        const double xk = y[k] / dg[k];
        if (rank == 0) u[k] = xk;
        for (int i = rank; i < k; i += size) y[i] = fma(-at(H, k, i), xk, y[i]);
        g.sync();
      }
    } else if (g.block() == 0) {
      // Eigen::PartialPivLU of the original H, one block.
      const int tid = threadIdx.x, nt = blockDim.x;
      double* piv = y;
      for (int k = tid; k < n * n; k += nt) H[k] = Hc[k];
      for (int k = tid; k < n; k += nt) u[k] = -h[k];
      __syncthreads();
      for (int k = 0; k < n; ++k) {
        if (tid == 0) {
          int p = k;
          double best = fabs(at(H, k, k));
          for (int i = k + 1; i < n; ++i) {
            const double v = fabs(at(H, i, k));
            if (v > best) best = v, p = i;
          }
          piv[k] = p;
        }
        __syncthreads();
        const int p = static_cast<int>(piv[k]);
        if (p != k)
          for (int j = tid; j < n; j += nt) {
            const double a = at(H, k, j);
            at(H, k, j) = at(H, p, j);
            at(H, p, j) = a;
          }
        __syncthreads();
        const double ukk = at(H, k, k);
        if (ukk != 0.0)
          for (int i = k + 1 + tid; i < n; i += nt) at(H, i, k) /= ukk;
        __syncthreads();
        for (int j = k + 1 + (tid >> 5); j < n; j += nt >> 5) {
          const double ukj = at(H, k, j);
          for (int i = k + 1 + lane; i < n; i += 32) at(H, i, j) = fma(-at(H, i, k), ukj, at(H, i, j));
        }
        __syncthreads();
      }
      if (tid == 0)
        for (int k = 0; k < n; ++k) {
          const int p = static_cast<int>(piv[k]);
          const double a = u[k];
          u[k] = u[p];
          u[p] = a;
        }
      __syncthreads();
      for (int k = 0; k < n; ++k) {  // unit-lower L
        const double yk = u[k];
        for (int i = k + 1 + tid; i < n; i += nt) u[i] = fma(-at(H, i, k), yk, u[i]);
        __syncthreads();
      }
      for (int k = n - 1; k >= 0; --k) {
        if (tid == 0) u[k] /= at(H, k, k);
        __syncthreads();
        const double xk = u[k];
        for (int i = tid; i < k; i += nt) u[i] = fma(-at(H, i, k), xk, u[i]);
        __syncthreads();
      }
    }
    g.sync();
    // Residual bound (condensed.hpp:128-135); 2-norms, Frobenius |H|.
    double r2 = 0.0, H2 = 0.0, u2 = 0.0, h2 = 0.0, bad = 0.0;
    for (int i = rank; i < n; i += size) {
      double ri = h[i];
      for (int j = 0; j < n; ++j) {
        const double hij = at(Hc, i, j);
        ri = fma(hij, u[j], ri);
        H2 = fma(hij, hij, H2);
      }
      r2 = fma(ri, ri, r2);
      u2 = fma(u[i], u[i], u2);
      h2 = fma(h[i], h[i], h2);
      if (!isfinite(u[i])) bad = 1.0;
    }
    red_put(g, 0, r2, true);
    red_put(g, 1, H2, true);
    red_put(g, 2, u2, true);
    red_put(g, 3, h2, true);
    red_put(g, 4, bad, false);
    g.finish(5, 4);
    const double bound = 1e-9 * (sqrt(g.sm->total[1]) * sqrt(g.sm->total[2]) + sqrt(g.sm->total[3]));
    return (g.sm->total[4] > 0.0 || !(sqrt(g.sm->total[0]) <= bound)) ? kFactorization : kBwdOk;
  }

  __device__ int condensed_p2(double reg) {
    const int m = t.n_shared, nb = t.n_bound, n = cond_n();
    const int D = t.ndepth;
    double* H = cHc();
    double* h = ch();
    for (int k = g.item0(n * n), k_e = g.item_end(n * n); k < k_e; k += g.item_step()) H[k] = 0.0;
    // (1) zero-input perturbations z, depth by depth (the boundary: heads of depth D-1).
    for (int d = 0; d < D; ++d) {
      const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
      const int L = d == D - 1 ? 1 : t.depth_len[d];
      for (int sg = sb + g.rank(); sg < se; sg += g.size()) {
        const SegIdx sq = seg_idx(sg);
        double z[NX];
        const int hd = sq.head, p = t.parent[hd];
        if (p < 0) {
#pragma unroll
          for (int j = 0; j < NX; ++j) z[j] = w.x0[j] - w.x[j];
        } else {
          double A[NX * NX], Bm[NX * NU], t1[NX];
          load_AB(p, A, Bm);
          mv<NX, NX>(A, crec(p) + CondL::z, t1);
#pragma unroll
          for (int j = 0; j < NX; ++j) z[j] = t1[j] + w.defect[hd * NX + j];
        }
        copy<NX>(z, crec(hd) + CondL::z);
        for (int k = 1; k < L; ++k) {
          const int prev = node_at(sq, k - 1), i = node_at(sq, k);
          double A[NX * NX], Bm[NX * NU], t1[NX];
          load_AB(prev, A, Bm);
          mv<NX, NX>(A, z, t1);
#pragma unroll
          for (int j = 0; j < NX; ++j) z[j] = t1[j] + w.defect[i * NX + j];
          copy<NX>(z, crec(i) + CondL::z);
        }
      }
      g.sync();
    }
    // (2) boundary values V_b = P_b, lam_b = p_b + P_b z_b (P1 results).
    for (int b = m + g.rank(); b < m + nb; b += g.size()) {
      const double* v = value_ptr(b);
      double* c = crec(b);
      double Pz[NX];
      mv<NX, NX>(v, c + CondL::z, Pz);
      copy<NX * NX>(v, c + CondL::V);
#pragma unroll
      for (int j = 0; j < NX; ++j) c[CondL::lam + j] = v[NX * NX + j] + Pz[j];
    }
    g.sync();
    // (3) shared nodes, leaves-first: Vs, lams, V, lam, W; diagonal blocks of H and h.
    for (int d = D - 2; d >= 0; --d) {
      const int sb = t.depth_begin[d], se = t.depth_begin[d + 1], L = t.depth_len[d];
      for (int sg = sb + g.rank(); sg < se; sg += g.size()) {
        const SegIdx sq = seg_idx(sg);
        for (int k = L - 1; k >= 0; --k) {
          const int i = node_at(sq, k);
          double* c = crec(i);
          double Vs[NX * NX], ls[NX];
#pragma unroll
          for (int q = 0; q < NX * NX; ++q) Vs[q] = 0.0;
#pragma unroll
          for (int q = 0; q < NX; ++q) ls[q] = 0.0;
          const int c0 = t.first_child[i], nc = t.nchild[i];
          for (int ch = c0; ch < c0 + nc; ++ch) {  // children in index order
            const double* cc = crec(ch);
#pragma unroll
            for (int q = 0; q < NX * NX; ++q) Vs[q] += cc[CondL::V + q];
#pragma unroll
            for (int q = 0; q < NX; ++q) ls[q] += cc[CondL::lam + q];
          }
          double A[NX * NX], Bm[NX * NU], Q[NX * NX], R[NU * NU], M[NU * NX], q[NX], r[NU];
          load_AB(i, A, Bm);
          load_QRMqr(i, Q, R, M, q, r);
          double AtV[NX * NX], V[NX * NX], BtV[NU * NX], Hd[NU * NU], W[NX * NU], t1[NX], t2[NU], t3[NU];
          mtm<NX, NX, NX>(A, Vs, AtV);
          mm<NX, NX, NX>(AtV, A, V);
#pragma unroll
          for (int e = 0; e < NX * NX; ++e) V[e] += Q[e];
          symmetrize<NX>(V);
          mm<NX, NX, NU>(AtV, Bm, W);
#pragma unroll
          for (int a = 0; a < NU; ++a)
#pragma unroll
            for (int j = 0; j < NX; ++j) W[j + a * NX] += M[a + j * NU];
          mtm<NU, NX, NX>(Bm, Vs, BtV);
          mm<NU, NX, NU>(BtV, Bm, Hd);
#pragma unroll
          for (int e = 0; e < NU * NU; ++e) Hd[e] += R[e];
#pragma unroll
          for (int a = 0; a < NU; ++a) Hd[a + a * NU] += reg;  // regularized R (solver.hpp:212-222)
          symmetrize<NU>(Hd);
          // lam = q + Q z + A' lams ; h_i = B' lams + M z + r
          mv<NX, NX>(Q, c + CondL::z, t1);
          double Atl[NX];
          mtv<NX, NX>(A, ls, Atl);
#pragma unroll
          for (int j = 0; j < NX; ++j) c[CondL::lam + j] = (q[j] + t1[j]) + Atl[j];
          mtv<NU, NX>(Bm, ls, t2);
          mv<NU, NX>(M, c + CondL::z, t3);
#pragma unroll
          for (int a = 0; a < NU; ++a) h[i * NU + a] = (t2[a] + t3[a]) + r[a];
          copy<NX * NX>(V, c + CondL::V);
          copy<NX * NU>(W, c + CondL::W);
#pragma unroll
          for (int a = 0; a < NU; ++a)
#pragma unroll
            for (int b2 = 0; b2 < NU; ++b2) H[(i * NU + a) + static_cast<size_t>(i * NU + b2) * n] = Hd[a + b2 * NU];
        }
      }
      g.sync();
    }
    // (4) off-diagonal blocks: every shared node b against each ancestor a.
    for (int b = 1 + g.rank(); b < m; b += g.size()) {
      const double* W = crec(b) + CondL::W;
      double T[NX * NX];
#pragma unroll
      for (int q = 0; q < NX * NX; ++q) T[q] = (q % (NX + 1)) == 0 ? 1.0 : 0.0;
      for (int y = b, a = t.parent[b]; a >= 0; y = a, a = t.parent[a]) {
        double A[NX * NX], Bm[NX * NU], S[NX * NU], Hab[NU * NU], T2[NX * NX];
        load_AB(a, A, Bm);
        mm<NX, NX, NU>(T, Bm, S);    // dx_b / du_a
        mtm<NU, NX, NU>(S, W, Hab);  // (a, b) block
#pragma unroll
        for (int r = 0; r < NU; ++r)
#pragma unroll
          for (int c2 = 0; c2 < NU; ++c2) {
            H[(a * NU + r) + static_cast<size_t>(b * NU + c2) * n] = Hab[r + c2 * NU];
            H[(b * NU + c2) + static_cast<size_t>(a * NU + r) * n] = Hab[r + c2 * NU];
          }
        mm<NX, NX, NX>(T, A, T2);
        copy<NX * NX>(T2, T);
      }
    }
    g.sync();
    // (5) solve_dense.
    const int err = dense_solve();
    // (6) open-loop policies of the shared nodes.
    if (err == kBwdOk) {
      const double* u = cu();
      for (int i = g.item0(m), i_e = g.item_end(m); i < i_e; i += g.item_step()) {
#pragma unroll
        for (int q = 0; q < NU * NX; ++q) pol(i)[PL::K + q] = 0.0;
#pragma unroll
        for (int a = 0; a < NU; ++a) pol(i)[PL::k + a] = u[i * NU + a];
      }
    }
    g.sync();
    return err;
  }

  __device__ int backward(double reg, double* max_ff) {
    int err = kBwdOk;
    // Condensed strategy: only the leaf segments (P1) take the tree scan.
    const bool condensed = kCond && o.condensed && t.n_shared > 0;
    for (int d = t.ndepth - 1; d >= (condensed ? t.ndepth - 1 : 0); --d) {
      const int L = t.depth_len[d];
      if (seq_depth(d)) {
        const int e = riccati_sweep_depth(d, reg);
        err = err ? err : e;
        mark(2);
        continue;
      }
      if constexpr (!kSeqOnly) {
      // Terminal of each segment: regularized leaf cost or the branch-node
      // Bellman step over the summed children (riccati.hpp:107-120).
      for_depth_items(d, 1, [&](int s, int) {
        const int b = seg_node(s, L - 1);
        double* term = bwd(t.seg_scratch[s] + 0);
        double P[NX * NX], p[NX];
        if (is_leaf(b)) {
          copy<NX * NX>(stage(b) + SL::Q, P);
          copy<NX>(stage(b) + SL::q, p);
#pragma unroll
          for (int j = 0; j < NX; ++j) P[j + j * NX] += reg;
        } else {
          double Pn[NX * NX], pn[NX];
#pragma unroll
          for (int j = 0; j < NX * NX; ++j) Pn[j] = 0.0;
#pragma unroll
          for (int j = 0; j < NX; ++j) pn[j] = 0.0;
          const int c0 = t.first_child[b], nc = t.nchild[b];
          for (int ch = c0; ch < c0 + nc; ++ch) {
            const double* v = value_ptr(ch);
            double Pd[NX];
            mv<NX, NX>(v, w.defect + ch * NX, Pd);
#pragma unroll
            for (int j = 0; j < NX * NX; ++j) Pn[j] += v[j];
#pragma unroll
            for (int j = 0; j < NX; ++j) pn[j] += v[NX * NX + j] + Pd[j];
          }
          const int e = riccati_step<NX, NU>(stage(b), reg, Pn, pn, P, p, pol(b) + PL::K, pol(b) + PL::k);
          err = err ? err : e;
        }
        embed_terminal<NX>(P, p, term);
      });
      // One-step elements of the chain nodes (chain_stage, solver.hpp:189-193:
      // offset = defect of the next node), stored reversed.
      if (L >= 2) {
        for_depth_items(d, L - 1, [&](int s, int k) {
          const int i = seg_node(s, k), nxt = seg_node(s, k + 1);
          const int e = init_bwd_element<NX, NU>(stage(i), reg, w.defect + nxt * NX,
                                                  bwd(t.seg_scratch[s] + L - 1 - k));
          err = err ? err : e;
        });
      }
      g.sync();
      mark(1);
      const int e = scan_bwd_depth(d);
      mark(2);
      err = err ? err : e;
      }
    }
    if constexpr (kCond) {
      if (condensed && err == kBwdOk) {
        g.sync();
        err = condensed_p2(reg);
      }
    }
    // Policies of scanned chain nodes from their successor's value
    // (feedback_from_values, lqr_scan.hpp:146); max_feedforward.
    double mff = 0.0;
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      if (is_leaf(i)) continue;
      const int s = t.node_seg[i], k = t.node_pos[i];
      if constexpr (!kSeqOnly) {
        if (!seq_seg(s) && k + 1 < seg_len(s) && !(condensed && i < t.n_shared)) {
          const int nxt = seg_node(s, k + 1);
          const double* v = value_of(nxt);
          const int e = feedback<NX, NU>(stage(i), reg, w.defect + nxt * NX, v + BL::P, v + BL::p,
                                         pol(i) + PL::K, pol(i) + PL::k);
          err = err ? err : e;
        }
      }
      if constexpr (!kSeqOnly) {  // the parallel forward scan's element of transition (i, nxt)
        const int d = t.seg_depth[s];
        if (block_scan_fwd(d) && k + 1 < seg_len(s)) {
          const int T = t.depth_len[d] - 1;
          const FwdRuns fr = fwd_runs(T);
          double e[kWE];
          walk_element(i, seg_node(s, k + 1), e);
          double* p = fwd(t.seg_scratch[s]) + fr.pos(k);
#pragma unroll
          for (int f = 0; f < kWE; ++f) p[f * fr.stride()] = e[f];
        }
      }
      double m = 0.0;
#pragma unroll
      for (int j = 0; j < NU; ++j) m = fmax(m, fabs(pol(i)[PL::k + j]));
      mff = fmax(mff, m);
    }
    red_put(g, 0, mff, false);
    red_put(g, 1, static_cast<double>(err), false);
    g.finish(2, 0);
    mark(3);
    *max_ff = g.sm->total[0];
    return static_cast<int>(g.sm->total[1]);
  }

  // Items of a phase spanning several depths, numbered contiguously across
  // depths so each thread gets at most its share (per_seg(d) items/segment;
  // 0 skips the depth).
  template <class PerSeg, class F>
  __device__ void for_multi_depth_items(PerSeg&& per_seg, F&& f) const {
    int total = 0;
    for (int d = 0; d < t.ndepth; ++d) total += (t.depth_begin[d + 1] - t.depth_begin[d]) * per_seg(d);
    for (int q = g.item0(total), q_e = g.item_end(total); q < q_e; q += g.item_step()) {
      int r = q, d = 0;
      for (; d < t.ndepth; ++d) {
        const int cnt = (t.depth_begin[d + 1] - t.depth_begin[d]) * per_seg(d);
        if (r < cnt) break;
        r -= cnt;
      }
      const int ps = per_seg(d);
      f(d, t.depth_begin[d] + r / ps, r % ps);
    }
  }

  // --------------------------------------------------- forward pass (F)
  // linear_rollout (solver.hpp:330-387) + expected_change_coefficients
  // (:412-430). Long segments: prefix scan of the closed-loop maps
  // (lqr_scan.hpp:177-187, all depths at once) then a per-node depth sweep;
  // short segments: a team walk dx_{k+1} = A dx + B du + d. Returns (a1, a2).
  __device__ void forward(double* a1_out, double* a2_out) {
    auto scan_E = [&](int d) { return fwd_walk(t.depth_len[d]) ? 0 : t.depth_len[d] - 1; };
    if constexpr (!kSeqOnly) {
    for_multi_depth_items([&](int d) { return scan_E(d); }, [&](int d, int s, int k) {
      const int i = seg_node(s, k), nxt = seg_node(s, k + 1);
      init_fwd_element<NX, NU>(stage(i), w.defect + nxt * NX, pol(i) + PL::K, pol(i) + PL::k,
                               fwd(t.seg_scratch[s] + k));
    });
    g.sync();
    mark(4);
    // Prefix scans (scan.hpp:19-50), all scanned depths in the same phases.
    int maxU = 0;
    for (int d = 0; d < t.ndepth; ++d) maxU = max(maxU, up_steps(scan_E(d)));
    for (int l = 0; l < maxU; ++l) {
      for_multi_depth_items(
          [&](int d) { return l < up_steps(scan_E(d)) ? (level_size(scan_E(d), l) + 1) >> 1 : 0; },
          [&](int d, int s, int i) {
            const int E = scan_E(d);
            const int nl = level_size(E, l);
            const int ol = level_offset(E, l), on = ol + nl;
            const int base = t.seg_scratch[s];
            if (2 * i + 1 < nl)
              combine_fwd<NX>(fwd(base + ol + 2 * i), fwd(base + ol + 2 * i + 1), fwd(base + on + i));
            else
              copy<FL::size>(fwd(base + ol + 2 * i), fwd(base + on + i));
          });
      g.sync();
    }
    for (int l = maxU - 1; l >= 0; --l) {
      for_multi_depth_items(
          [&](int d) { return l < up_steps(scan_E(d)) ? (level_size(scan_E(d), l) + 1) >> 1 : 0; },
          [&](int d, int s, int i) {
            const int E = scan_E(d);
            const int nl = level_size(E, l);
            const int ol = level_offset(E, l), on = ol + nl;
            const int base = t.seg_scratch[s];
            const double* S = fwd(base + on);
            if (2 * i + 1 < nl) copy<FL::size>(S + static_cast<size_t>(i) * FL::stride, fwd(base + ol + 2 * i + 1));
            if (i >= 1) {
              double* a = fwd(base + ol + 2 * i);
              combine_fwd<NX>(S + static_cast<size_t>(i - 1) * FL::stride, a, a);
            }
          });
      g.sync();
    }
    }
    mark(5);
    // Depth sweep.
    for (int d = 0; d < t.ndepth; ++d) {
      const int L = t.depth_len[d];
      if (fwd_walk(L)) {
        long long tf0 = 0, nf0 = 0;
        if (w.prof && threadIdx.x == 0) {
          tf0 = clock64();
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(nf0));
        }
        if (block_scan_fwd(d))
          forward_scan_block_depth(d);
        else
          forward_walk_depth(d);
        if (w.prof && threadIdx.x == 0) {
          long long nf1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(nf1));
          g.sm->prof[11] += static_cast<double>(clock64() - tf0);
          g.sm->prof[18] += static_cast<double>(nf1 - nf0);
        }
        continue;
      }
      if constexpr (!kSeqOnly) {
      for_depth_items(d, L, [&](int s, int k) {
        const int head = seg_node(s, 0);
        double h[NX];
        head_dx(head, h);
        const int i = seg_node(s, k);
        double dxi[NX];
        if (k == 0) {
          copy<NX>(h, dxi);
        } else {
          const double* F = fwd(t.seg_scratch[s] + k - 1);
          double t1[NX];
          mv<NX, NX>(F + FL::A, h, t1);
#pragma unroll
          for (int j = 0; j < NX; ++j) dxi[j] = t1[j] + F[FL::c + j];
        }
        copy<NX>(dxi, w.dx + i * NX);
        if (!is_leaf(i)) {
          double dui[NU];
          mv<NU, NX>(pol(i) + PL::K, dxi, dui);
#pragma unroll
          for (int j = 0; j < NU; ++j) w.du[i * NU + j] = dui[j] + pol(i)[PL::k + j];
        }
      });
      g.sync();
      }
    }
    mark(6);
    // EC terms per node (solver.hpp:416-428).
    double a1 = 0.0, a2 = 0.0;
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      const double* si = stage(i);
      const double* dxi = w.dx + i * NX;
      if constexpr (NX == 4 && NU == 2) {
        if (structured()) {
          ec_structured(i, si, dxi, &a1, &a2);
          continue;
        }
      }
      double Qdx[NX];
      mv<NX, NX>(si + SL::Q, dxi, Qdx);
      if (is_leaf(i)) {
        a1 += dot<NX>(si + SL::q, dxi);
        a2 += 0.5 * dot<NX>(dxi, Qdx);
      } else {
        double* dui = w.du + i * NU;
        if (fwd_walk(seg_len(t.node_seg[i]))) {  // walked segment: du = K dx + k
          const double* po = pol(i);
          double du[NU];
          mv<NU, NX>(po + PL::K, dxi, du);
#pragma unroll
          for (int j = 0; j < NU; ++j) dui[j] = du[j] + po[PL::k + j];
        }
        double Mdx[NU], Rdu[NU];
        mv<NU, NX>(si + SL::M, dxi, Mdx);
        mv<NU, NU>(si + SL::R, dui, Rdu);
        a1 += dot<NX>(si + SL::q, dxi) + dot<NU>(si + SL::r, dui);
        a2 += (0.5 * dot<NX>(dxi, Qdx) + dot<NU>(dui, Mdx)) + 0.5 * dot<NU>(dui, Rdu);
      }
    }
    red_put(g, 0, a1, true);
    red_put(g, 1, a2, true);
    g.finish(2, 2);
    mark(10);
    *a1_out = g.sm->total[0];
    *a2_out = g.sm->total[1];
  }

  // Head perturbation of a segment: dx0 at the root, else the parent's
  // closed loop dx_ch = (A + B K) dx_p + B k + defect_ch (solver.hpp:344-348).
  __device__ void head_dx(int head, double* h) const {
    const int p = t.parent[head];
    if (p < 0) {
#pragma unroll
      for (int j = 0; j < NX; ++j) h[j] = w.x0[j] - w.x[j];
      return;
    }
    double A[NX * NX], Bm[NX * NU];
    load_AB(p, A, Bm);
    double BK[NX * NX], Acl[NX * NX], Bk[NX], t1[NX];
    mm<NX, NU, NX>(Bm, pol(p) + PL::K, BK);
#pragma unroll
    for (int j = 0; j < NX * NX; ++j) Acl[j] = A[j] + BK[j];
    mv<NX, NU>(Bm, pol(p) + PL::k, Bk);
    mv<NX, NX>(Acl, w.dx + p * NX, t1);
#pragma unroll
    for (int j = 0; j < NX; ++j) h[j] = (t1[j] + Bk[j]) + w.defect[head * NX + j];
  }

  // Walk of every short segment at depth d (solver.hpp:341-350 closed loop):
  // dx_{k+1} = (A_k + B_k K_k) dx_k + B_k k_k + d_{k+1}. The per-step affine
  // maps do not depend on dx, so the whole block first builds them in shared
  // memory (one element per thread, a chunk of every segment at once); one
  // thread per segment then runs the dependent chain out of shared memory.
  // du = K dx + k is formed per node in the EC phase. Block-local: under a
  // GridGroup each block walks its own share of the depth's segments.
  static constexpr int kWE = NX * NX + 2 * NX;  // walk element: Acl, B k, defect of the next node
  // EC terms of one node from a structured record (variable entries only):
  // the dense products below with the exact-zero terms dropped, same bits.
  __device__ void ec_structured(int i, const double* si, const double* dxi, double* a1, double* a2) {
    const bool cmp = compact();
    // Variable entry at dense offset K of either layout (K is a compile-time constant).
    auto sv = [&](auto K) -> double {
      constexpr int k = decltype(K)::value;
      return cmp ? si[uni_var_of(k)] : si[k];
    };
    const double d0 = dxi[0], d1 = dxi[1], d2 = dxi[2], d3 = dxi[3];
    const double Q00 = sv(std::integral_constant<int, SL::Q + 0>{}), Q10 = sv(std::integral_constant<int, SL::Q + 1>{}),
                 Q01 = sv(std::integral_constant<int, SL::Q + 4>{}), Q11 = sv(std::integral_constant<int, SL::Q + 5>{});
    const double Qdx[4] = {fma(Q01, d1, Q00 * d0), fma(Q11, d1, Q10 * d0),
                           sv(std::integral_constant<int, SL::Q + 10>{}) * d2,
                           sv(std::integral_constant<int, SL::Q + 15>{}) * d3};
    const double qdx = dot<4>(si + (cmp ? uni_var_of(SL::q) : SL::q), dxi);
    const double xQx = dot<4>(dxi, Qdx);
    if (is_leaf(i)) {
      *a1 += qdx;
      *a2 += 0.5 * xQx;
      return;
    }
    double* dui = w.du + i * NU;
    if (fwd_walk(seg_len(t.node_seg[i]))) {  // walked segment: du = K dx + k
      const double* po = pol(i);
      double du[NU];
      mv<NU, NX>(po + PL::K, dxi, du);
#pragma unroll
      for (int j = 0; j < NU; ++j) dui[j] = du[j] + po[PL::k + j];
    }
    const double u0 = dui[0], u1 = dui[1];
    const double Rdu[2] = {sv(std::integral_constant<int, SL::R + 0>{}) * u0,
                           sv(std::integral_constant<int, SL::R + 3>{}) * u1};
    const double Mdx[2] = {0.0, 0.0};
    *a1 += qdx + fma(sv(std::integral_constant<int, SL::r + 1>{}), u1, sv(std::integral_constant<int, SL::r + 0>{}) * u0);
    *a2 += (0.5 * xQx + dot<2>(dui, Mdx)) + 0.5 * dot<2>(dui, Rdu);
  }

  // A, B of node i's stage record (structured records: variable entries only).
  __device__ void load_AB(int i, double* A, double* Bm) const {
    const double* si = stage(i);
    if constexpr (NX == 4 && NU == 2) {
      if (compact()) {
#pragma unroll
        for (int k = 0; k < NX * NX; ++k)
          A[k] = uni_var_of(SL::A + k) >= 0 ? si[uni_var_of(SL::A + k)] : unicycle_stage_constant(mp.dt, SL::A + k);
#pragma unroll
        for (int k = 0; k < NX * NU; ++k)
          Bm[k] = uni_var_of(SL::B + k) >= 0 ? si[uni_var_of(SL::B + k)] : unicycle_stage_constant(mp.dt, SL::B + k);
        return;
      }
      if (structured()) {
        unicycle_load_AB(si, mp.dt, A, Bm);
        return;
      }
    }
#pragma unroll
    for (int q = 0; q < NX * NX; ++q) A[q] = si[SL::A + q];
#pragma unroll
    for (int q = 0; q < NX * NU; ++q) Bm[q] = si[SL::B + q];
  }

  __device__ void walk_element(int i, int nxt, double* e) const {
    const double* po = pol(i);
    double A[NX * NX], Bm[NX * NU];
    load_AB(i, A, Bm);
    double BK[NX * NX], Bk[NX];
    mm<NX, NU, NX>(Bm, po + PL::K, BK);
#pragma unroll
    for (int q = 0; q < NX * NX; ++q) e[q] = A[q] + BK[q];
    mv<NX, NU>(Bm, po + PL::k, Bk);
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      e[NX * NX + j] = Bk[j];
      e[NX * NX + NX + j] = w.defect[nxt * NX + j];
    }
  }

  // Parallel forward pass of long segments (wide blocks of the non-lean
  // kernels): linear_rollout's forward_scan (lqr_scan.hpp:177-187) with no
  // group barrier inside instead of 2 log L grid-synchronised levels.
  //   E) backward()'s closing policy loop (all threads) already wrote the
  //      walk element (Acl, B k, defect) of every transition of the depth into
  //      the segment's forward scratch, field-major (coalesced reads below);
  //   S) block-locally, each segment gets whole warps and each thread
  //      1) composes the affine maps x -> (Acl x + B k) + d of its run of
  //         R <= 4 consecutive transitions,
  //      2) the warp scans the run maps with shuffles (5 levels),
  //      3) warp totals go through shared memory and each warp carries the
  //         segment's incoming dx across the earlier warps' totals,
  //      4) each thread takes its start state from lane - 1 and re-walks its
  //         run with the walk's arithmetic, writing dx.
  // Rounding differs from the one-thread walk, so the lean (population)
  // kernels keep the walk.
  static constexpr int kFE = NX * NX + NX;  // affine map (A, b)
  __device__ bool block_scan_fwd(int d) const {
    if constexpr (kSeqOnly) return false;
    return G::bdim() >= 128 && o.fwd_block_scan > 0 && t.depth_len[d] - 1 >= o.fwd_block_scan;
  }
  // Walk elements of a segment's T transitions in its forward scratch,
  // field-major and run-major: with R = ceil(T / block) transitions per
  // thread and W = ceil(T / R) threads, transition k = R t + q sits at
  // position q W + t of each field (stride R W < T + R), so the threads of a
  // warp read consecutive doubles.
  struct FwdRuns {
    int R, W;
    __device__ int pos(int k) const { return (k % R) * W + k / R; }
    __device__ int stride() const { return R * W; }
  };
  __device__ FwdRuns fwd_runs(int T) const {
    const int R = max(1, (T + G::bdim() - 1) / G::bdim());
    return {R, (T + R - 1) / R};
  }
  __device__ void load_walk_element(int base, const FwdRuns& fr, int k, double* e) const {
    const double* p = fwd(base) + fr.pos(k);
    const int st = fr.stride();
#pragma unroll
    for (int f = 0; f < kWE; ++f) e[f] = p[f * st];
  }
  // (A, b) <- E o (A, b) for the walk element e (Acl, B k, defect).
  __device__ static void compose_walk(const double* e, double* A, double* bb) {
    double An[NX * NX], bn[NX];
    mm<NX, NX, NX>(e, A, An);
    mv<NX, NX>(e, bb, bn);
#pragma unroll
    for (int j = 0; j < NX; ++j) bb[j] = (bn[j] + e[NX * NX + j]) + e[NX * NX + NX + j];
#pragma unroll
    for (int k = 0; k < NX * NX; ++k) A[k] = An[k];
  }
  __device__ void forward_scan_block_depth(int d) {
    const int L = t.depth_len[d], T = L - 1;
    const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
    long long tp = 0;  // diagnostic phase clocks (thread 0 of the block): prof[21..23]
    if (w.prof && threadIdx.x == 0) tp = clock64();
    auto tick = [&](int slot) {
      if (w.prof && threadIdx.x == 0) {
        const long long now = clock64();
        g.sm->prof[slot] += static_cast<double>(now - tp);
        tp = now;
      }
    };
    // E) the elements were written by backward()'s policy loop (scratch:
    //    2L + 32 slots of FL::stride doubles >= kWE (T + R)).
    const FwdRuns fr = fwd_runs(T);
    tick(21);
    const int nb = g.nblocks(), b = g.block();
    const int ls = G::bdim(), lr = threadIdx.x, lane = lr & 31, warp = lr >> 5, nw = ls >> 5;
    const int nmine = se - sb > b ? (se - sb - b + nb - 1) / nb : 0;
    const int R = fr.R, span = T;                            // transitions per thread; one round
    const int wps = (fr.W + 31) / 32;                        // warps per segment
    const int ng = nw / wps;                                 // segments per round
    double* tot = wbuf;                                      // [nw][kFE] warp totals
    double* carry = wbuf + nw * kFE;                         // [ng][NX]
    const int r = warp / wps, wg = warp - r * wps, tq = wg * 32 + lane;
    for (int j0 = 0; j0 < nmine; j0 += ng) {
      const int ngc = min(ng, nmine - j0);
      for (int rr = lr; rr < ngc; rr += ls) {
        const SegIdx qs = seg_idx(sb + b + (j0 + rr) * nb);
        double h[NX];
        head_dx(qs.head, h);
#pragma unroll
        for (int j = 0; j < NX; ++j) {
          w.dx[qs.head * NX + j] = h[j];
          carry[rr * NX + j] = h[j];
        }
      }
      __syncthreads();
      const bool seg_ok = r < ng && r < ngc;
      SegIdx qs{0, 0, 0};
      int base = 0;
      if (seg_ok) {
        const int s = sb + b + (j0 + r) * nb;
        qs = seg_idx(s);
        base = t.seg_scratch[s];
      }
      for (int c0 = 0; c0 < T; c0 += span) {
        const int cn = min(span, T - c0);
        const int k0 = c0 + tq * R;
        const int nk = seg_ok ? max(0, min(R, c0 + cn - k0)) : 0;
        // 1) run map
        double A[NX * NX], bb[NX];
#pragma unroll
        for (int k = 0; k < NX * NX; ++k) A[k] = (k % (NX + 1)) == 0 ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < NX; ++j) bb[j] = 0.0;
        for (int q = 0; q < nk; ++q) {
          double e[kWE];
          load_walk_element(base, fr, k0 + q, e);
          compose_walk(e, A, bb);
        }
        tick(22);
        // 2) warp inclusive scan: mine o lane-off's
        for (int off = 1; off < 32; off <<= 1) {
          double Ap[NX * NX], bp[NX];
#pragma unroll
          for (int k = 0; k < NX * NX; ++k) Ap[k] = __shfl_up_sync(0xffffffffu, A[k], off);
#pragma unroll
          for (int j = 0; j < NX; ++j) bp[j] = __shfl_up_sync(0xffffffffu, bb[j], off);
          if (lane >= off) {
            double An[NX * NX], bn[NX];
            mm<NX, NX, NX>(A, Ap, An);
            mv<NX, NX>(A, bp, bn);
#pragma unroll
            for (int j = 0; j < NX; ++j) bb[j] = bn[j] + bb[j];
#pragma unroll
            for (int k = 0; k < NX * NX; ++k) A[k] = An[k];
          }
        }
        // 3) warp totals; the segment's state at this warp's start
        if (lane == 31) {
#pragma unroll
          for (int k = 0; k < NX * NX; ++k) tot[warp * kFE + k] = A[k];
#pragma unroll
          for (int j = 0; j < NX; ++j) tot[warp * kFE + NX * NX + j] = bb[j];
        }
        __syncthreads();
        double x[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) x[j] = seg_ok ? carry[r * NX + j] : 0.0;
        for (int v = 0; v < wg; ++v) {
          const double* tv = tot + (r * wps + v) * kFE;
          double t1[NX];
          mv<NX, NX>(tv, x, t1);
#pragma unroll
          for (int j = 0; j < NX; ++j) x[j] = t1[j] + tv[NX * NX + j];
        }
        // 4) own end state; start state = lane - 1's end state; re-walk
        double y[NX];
        {
          double t1[NX];
          mv<NX, NX>(A, x, t1);
#pragma unroll
          for (int j = 0; j < NX; ++j) y[j] = t1[j] + bb[j];
        }
        double st[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) {
          const double v = __shfl_up_sync(0xffffffffu, y[j], 1);
          st[j] = lane == 0 ? x[j] : v;
        }
        for (int q = 0; q < nk; ++q) {
          double e[kWE];
          load_walk_element(base, fr, k0 + q, e);
          double t1[NX];
          mv<NX, NX>(e, st, t1);
          const int nxt = node_at(qs, k0 + q + 1);
#pragma unroll
          for (int j = 0; j < NX; ++j) {
            st[j] = (t1[j] + e[NX * NX + j]) + e[NX * NX + NX + j];
            w.dx[nxt * NX + j] = st[j];
          }
        }
        __syncthreads();  // carry / totals consumed
        if (nk > 0 && k0 + nk == c0 + cn)
#pragma unroll
          for (int j = 0; j < NX; ++j) carry[r * NX + j] = st[j];
        __syncthreads();
        tick(23);
      }
    }
    g.sync();
  }

  __device__ void forward_walk_depth(int d) {
    const int L = t.depth_len[d];
    const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
    const int nb = g.nblocks(), b = g.block();
    const int T = L - 1;  // transitions inside a segment
    const int lr = threadIdx.x, ls = G::bdim();
    const int nmine = se - sb > b ? (se - sb - b + nb - 1) / nb : 0;
    const int grp = min(ls, wcap);
    for (int j0 = 0; j0 < nmine; j0 += grp) {
      const int ng = min(grp, nmine - j0);
      const int C = max(1, wcap / ng);
      const bool walker = lr < ng;
      SegIdx sq{0, 0, 0};
      double dx[NX];
      long long th0 = 0;
      if (w.prof && lr == 0) th0 = clock64();
      if (walker) {
        sq = seg_idx(sb + b + (j0 + lr) * nb);
        head_dx(sq.head, dx);
#pragma unroll
        for (int j = 0; j < NX; ++j) w.dx[sq.head * NX + j] = dx[j];
      }
      if (w.prof && lr == 0) {  // diagnostic (shared-memory accumulators)
        const long long now = clock64();
        g.sm->prof[14] += static_cast<double>(now - th0);
        th0 = now;
      }
      for (int c0 = 0; c0 < T; c0 += C) {
        const int cn = min(C, T - c0);
        long long tq0 = 0;
        if (w.prof && lr == 0) tq0 = clock64();
        for (int q = lr; q < ng * cn; q += ls) {
          const int r = q / cn, kk = q - r * cn;
          const SegIdx qs = seg_idx(sb + b + (j0 + r) * nb);
          walk_element(node_at(qs, c0 + kk), node_at(qs, c0 + kk + 1), wbuf + (r * C + kk) * kWE);
        }
        __syncthreads();
        if (w.prof && lr == 0) {
          const long long now = clock64();
          g.sm->prof[19] += static_cast<double>(now - tq0);
          tq0 = now;
        }
        if (walker) {
          // The chain touches shared memory only: dx_{k+1} replaces the
          // consumed element's B k slot, copied out block-wide below.
          double* e = wbuf + lr * C * kWE;
          for (int kk = 0; kk < cn; ++kk, e += kWE) {
            double t1[NX];
            mv<NX, NX>(e, dx, t1);
#pragma unroll
            for (int j = 0; j < NX; ++j) {
              dx[j] = (t1[j] + e[NX * NX + j]) + e[NX * NX + NX + j];
              e[NX * NX + j] = dx[j];
            }
          }
        }
        if (w.prof && lr == 0) g.sm->prof[20] += static_cast<double>(clock64() - tq0);
        __syncthreads();
        for (int q = lr; q < ng * cn * NX; q += ls) {
          const int r = q / (cn * NX), rem = q - r * cn * NX, kk = rem / NX, j = rem - kk * NX;
          const SegIdx qs = seg_idx(sb + b + (j0 + r) * nb);
          w.dx[node_at(qs, c0 + kk + 1) * NX + j] = wbuf[(r * C + kk) * kWE + NX * NX + j];
        }
        __syncthreads();
      }
      if (w.prof && lr == 0) g.sm->prof[15] += static_cast<double>(clock64() - th0);
    }
    g.sync();
  }

  // ------------------------------------------------- line search (S)
  // Parallel line search (solver.hpp:459-518): every alpha evaluated, sums in
  // slots [4l .. 4l+3]; returns the first accepted level or -1.
  // Parallel line search (solver.hpp:459-518) with the reference's
  // first-accepted-alpha semantics, evaluated in rounds of o.ls_block step
  // sizes: a round evaluates its alphas for every node, reduces them, and
  // stops at the first accepted one. The chosen alpha and every reported
  // value are identical to evaluating all levels at once (each alpha's sums
  // are independent of the rounds); later rounds only run when every alpha of
  // the earlier ones was rejected.
  // One node per thread per chunk; the node's and its parent's x, dx, u, du
  // are loaded once per round and the round's alphas evaluated from
  // registers. Per-alpha sums are butterfly-reduced per chunk into the warp
  // slots (fixed order, deterministic). Returns the accepted level or -1.
  __device__ int line_search(int levels, double merit0, double a1, double a2, double mu, double dl1_nom,
                             Eval* chosen, double* merit_chosen, double* decrease_chosen, int* evals) {
    const int blk = o.ls_block > 0 ? min(o.ls_block, kMaxAlpha) : levels;
    for (int l0 = 0; l0 < levels; l0 += blk) {
      const int nl = min(blk, levels - l0);
      *evals += nl;
      for (int rnd = 0, nrnd = g.item_rounds(t.n); rnd < nrnd; ++rnd) {
        const int i = g.item_at(t.n, rnd);
        const bool valid = i < t.n;
        const bool leaf = valid ? is_leaf(i) : true;
        const int p = valid ? t.parent[i] : -1;
        double x[NX], dx[NX], u[NU], du[NU], xp[NX], dxp[NX], up[NU], dup[NU];
#pragma unroll
        for (int j = 0; j < NX; ++j) {
          x[j] = valid ? w.x[i * NX + j] : 0.0;
          dx[j] = valid ? w.dx[i * NX + j] : 0.0;
          xp[j] = p >= 0 ? w.x[p * NX + j] : 0.0;
          dxp[j] = p >= 0 ? w.dx[p * NX + j] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < NU; ++j) {
          u[j] = valid && !leaf ? w.u[i * NU + j] : 0.0;
          du[j] = valid && !leaf ? w.du[i * NU + j] : 0.0;
          up[j] = p >= 0 ? w.u[p * NU + j] : 0.0;
          dup[j] = p >= 0 ? w.du[p * NU + j] : 0.0;
        }
        const double wi = valid ? t.weight[i] : 0.0;
        const double* eta = w.eta + static_cast<size_t>(valid ? i : 0) * t.max_con;
#pragma unroll 1
        for (int q = 0; q < nl; ++q) {
          const double alpha = ldexp(1.0, -(l0 + q));
          double c = 0.0, cal = 0.0, dl = 0.0, vm = -INFINITY;
          if (valid) {
            double xt[NX], ut[NU];
#pragma unroll
            for (int j = 0; j < NX; ++j) xt[j] = fma(alpha, dx[j], x[j]);
#pragma unroll
            for (int j = 0; j < NU; ++j) ut[j] = leaf ? 0.0 : fma(alpha, du[j], u[j]);
            double nc, pen, gm;
            node_cost<NX, NU>(mp, i, leaf, xt, ut, eta, g_rho, &nc, &pen, &gm);
            c = wi * nc;
            cal = wi * (nc + pen);
            vm = gm;
            if (p >= 0) {
              double xpt[NX], upt[NU], f[NX];
#pragma unroll
              for (int j = 0; j < NX; ++j) xpt[j] = fma(alpha, dxp[j], xp[j]);
#pragma unroll
              for (int j = 0; j < NU; ++j) upt[j] = fma(alpha, dup[j], up[j]);
              node_dynamics<NX, NU>(mp, p, xpt, upt, f);
              double sd = 0.0;
#pragma unroll
              for (int j = 0; j < NX; ++j) sd += fabs(f[j] - xt[j]);
              dl = sd;
            }
          }
          const bool first = rnd == 0;
          red_acc(g, 3 * q + 0, c, true, first);
          red_acc(g, 3 * q + 1, cal, true, first);
          red_acc(g, 3 * q + 2, dl, true, first);
          red_acc(g, 3 * nl + q, vm, false, first);
        }
      }
      g.finish(4 * nl, 3 * nl);
      for (int q = 0; q < nl; ++q) {
        const double alpha = ldexp(1.0, -(l0 + q));
        const double cal = g.sm->total[3 * q + 1], dl = g.sm->total[3 * q + 2];
        const bool finite = isfinite(cal) && isfinite(dl);
        const double m = finite ? cal + mu * dl : INFINITY;
        const double ec = a1 * alpha + a2 * alpha * alpha;
        const double dec = o.armijo_beta * (ec - alpha * mu * dl1_nom);
        if (isfinite(m) && m <= merit0 + dec) {
          *chosen = {g.sm->total[3 * q + 0], cal, dl, fmax(g.sm->total[3 * nl + q], 0.0)};
          *merit_chosen = m;
          *decrease_chosen = dec;
          return l0 + q;
        }
      }
      // (finish() opens with a barrier, so the next round cannot overwrite
      // the totals while a thread still reads them.)
    }
    return -1;
  }

  // ------------------------------ single-shooting line search (sssilqr)
  // ForwardMode::nonlinear_rollout (solver.hpp:463-467): each trial is
  // nonlinear_rollout(problem, nominal, policies, alpha, x0)
  // (problem.hpp:170-191): u_i = u_nom_i + K_i (x_i - x_nom_i) + alpha k_i,
  // x_child = f(x_i, u_i), walked one thread per segment, depth levels in
  // order. The trial lands in (dx, du) — the linear step is not needed once
  // EC is formed, and a rejected pass recomputes it. A non-finite state (the
  // reference throws, evaluate_trial catches) rejects the trial. Alphas are
  // tried largest first; the first accepted is the parallel mode's answer too.
  __device__ bool rollout_policy(double alpha) {
    if (g.leader()) {
#pragma unroll
      for (int j = 0; j < NX; ++j) w.dx[j] = w.x0[j];
    }
    g.sync();
    double bad = 0.0;
    for (int d = 0; d < t.ndepth; ++d) {
      const int sb = t.depth_begin[d], se = t.depth_begin[d + 1];
      for (int s = sb + g.rank(); s < se; s += g.size()) {
        // The walked state / input stay in registers along the segment; only
        // the head reads its parent's (written one depth level earlier).
        const int L = seg_len(s);
        int prev = t.parent[seg_node(s, 0)];
        double xp[NX], up[NU];
        if (prev >= 0) {
#pragma unroll
          for (int j = 0; j < NX; ++j) xp[j] = w.dx[prev * NX + j];
#pragma unroll
          for (int j = 0; j < NU; ++j) up[j] = w.du[prev * NU + j];
        }
        const SegIdx sq = seg_idx(s);
        for (int k = 0; k < L; ++k) {
          const int i = node_at(sq, k);
          // The node's nominal point and policy are loaded before the
          // dynamics of the step that produces its state, so their latency
          // hides under the RK4 arithmetic of the dependency chain.
          const bool leaf = is_leaf(i);
          double xn[NX], un[NU], Kp[NU * NX], kp[NU];
          if (!leaf) {
            const double* pk = pol(i);
#pragma unroll
            for (int j = 0; j < NX; ++j) xn[j] = w.x[i * NX + j];
#pragma unroll
            for (int j = 0; j < NU; ++j) un[j] = w.u[i * NU + j];
#pragma unroll
            for (int j = 0; j < NU * NX; ++j) Kp[j] = pk[PL::K + j];
#pragma unroll
            for (int j = 0; j < NU; ++j) kp[j] = pk[PL::k + j];
          }
          double xi[NX];
          if (prev >= 0) {
            node_dynamics<NX, NU>(mp, prev, xp, up, xi);
            if (!all_finite<NX>(xi)) bad = 1.0;
            copy<NX>(xi, w.dx + i * NX);
          } else {
#pragma unroll
            for (int j = 0; j < NX; ++j) xi[j] = w.dx[i * NX + j];
          }
          if (leaf) {
#pragma unroll
            for (int j = 0; j < NU; ++j) up[j] = 0.0;
          } else {
            double e[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) e[j] = xi[j] - xn[j];
#pragma unroll
            for (int r = 0; r < NU; ++r) {
              double kv = 0.0;
#pragma unroll
              for (int j = 0; j < NX; ++j) kv += Kp[r + j * NU] * e[j];  // K column-major NU x NX
              up[r] = (un[r] + kv) + alpha * kp[r];
            }
          }
#pragma unroll
          for (int j = 0; j < NU; ++j) w.du[i * NU + j] = up[j];
#pragma unroll
          for (int j = 0; j < NX; ++j) xp[j] = xi[j];
          prev = i;
        }
      }
      g.sync();
    }
    red_put(g, 0, bad, false);
    g.finish(1, 0);
    return g.sm->total[0] == 0.0;
  }

  // evaluate (problem.hpp:109-146) of the trajectory held in (dx, du).
  __device__ Eval evaluate_trial() {
    double c = 0, cal = 0, dl = 0, vm = -INFINITY;
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      const bool leaf = is_leaf(i);
      const double* xi = w.dx + i * NX;
      double u[NU];
#pragma unroll
      for (int j = 0; j < NU; ++j) u[j] = leaf ? 0.0 : w.du[i * NU + j];
      double nc, pen, gm;
      node_cost<NX, NU>(mp, i, leaf, xi, u, w.eta + static_cast<size_t>(i) * t.max_con, g_rho, &nc, &pen, &gm);
      const double wi = t.weight[i];
      c += wi * nc;
      cal += wi * (nc + pen);
      vm = fmax(vm, gm);
      const int p = t.parent[i];
      if (p >= 0) {
        double f[NX];
        node_dynamics<NX, NU>(mp, p, w.dx + p * NX, w.du + p * NU, f);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NX; ++j) s += fabs(f[j] - xi[j]);
        dl += s;
      }
    }
    red_put(g, 0, c, true);
    red_put(g, 1, cal, true);
    red_put(g, 2, dl, true);
    red_put(g, 3, vm, false);
    g.finish(4, 3);
    return {g.sm->total[0], g.sm->total[1], g.sm->total[2], fmax(g.sm->total[3], 0.0)};
  }

  __device__ int line_search_nonlinear(int levels, double merit0, double a1, double a2, double mu, double dl1_nom,
                                       Eval* chosen, double* merit_chosen, double* decrease_chosen, int* evals) {
    for (int l = 0; l < levels; ++l) {
      const double alpha = ldexp(1.0, -l);
      ++*evals;
      if (!rollout_policy(alpha)) continue;
      const Eval ev = evaluate_trial();
      const bool finite = isfinite(ev.cost_al) && isfinite(ev.defect_l1);
      const double m = finite ? ev.cost_al + mu * ev.defect_l1 : INFINITY;
      const double ec = a1 * alpha + a2 * alpha * alpha;
      const double dec = o.armijo_beta * (ec - alpha * mu * dl1_nom);
      if (isfinite(m) && m <= merit0 + dec) {
        *chosen = ev;
        *merit_chosen = m;
        *decrease_chosen = dec;
        return l;
      }
    }
    return -1;
  }

  // Accept the trial held in (dx, du).
  __device__ void take_trial() {
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
#pragma unroll
      for (int j = 0; j < NX; ++j) w.x[i * NX + j] = w.dx[i * NX + j];
#pragma unroll
      for (int j = 0; j < NU; ++j) w.u[i * NU + j] = w.du[i * NU + j];
    }
    g.sync();
  }

  __device__ void take_step(double alpha) {
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
#pragma unroll
      for (int j = 0; j < NX; ++j) w.x[i * NX + j] = fma(alpha, w.dx[i * NX + j], w.x[i * NX + j]);
      if (!is_leaf(i)) {
#pragma unroll
        for (int j = 0; j < NU; ++j) w.u[i * NU + j] = fma(alpha, w.du[i * NU + j], w.u[i * NU + j]);
      }
    }
    g.sync();
  }

  // Projected multiplier update (solver.hpp:764-769).
  __device__ void update_multipliers(double rho) {
    for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
      double gv[kMaxCon];
      const int nc = node_constraints<NX, NU>(mp, i, is_leaf(i), w.x + i * NX, w.u + i * NU, gv);
      double* eta = w.eta + static_cast<size_t>(i) * t.max_con;
      for (int m = 0; m < nc; ++m) eta[m] = fmax(eta[m] + rho * gv[m], 0.0);
    }
    g.sync();
  }

  // Per-phase device time (diagnostic): the leader charges the time since
  // the previous mark to slot `id` (Work::prof, optional).
  unsigned long long prof_last{0};
  __device__ void mark(int id) {
    if (w.prof && g.leader()) {
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      if (prof_last) g.sm->prof[id] += static_cast<double>(ns - prof_last);
      prof_last = ns;
    }
  }

  __device__ static double now_s() {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    return static_cast<double>(ns) * 1e-9;
  }

  // ------------------------------------------------------------- solve
  __device__ void solve() {
    long long c0 = 0, n0 = 0;
    if (w.prof && g.leader()) {
      for (int k = 0; k < kProfSlots; ++k) g.sm->prof[k] = 0.0;
      c0 = clock64();
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n0));
    }
    solve_body();
    if (w.prof && g.leader()) {  // SM clock check: cycles and ns of this launch
      long long n1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n1));
      g.sm->prof[16] += static_cast<double>(clock64() - c0);
      g.sm->prof[17] += static_cast<double>(n1 - n0);
    }
    if (w.prof && g.leader())  // one flush per launch (a global RMW per mark costs ~1 us)
      for (int k = 0; k < kProfSlots; ++k) w.prof[k] += g.sm->prof[k];
  }

  __device__ void solve_body() {
    double t_start = now_s();
    double times[6] = {0, 0, 0, 0, 0, 0};
    DevResult* res = w.result;
    DevResume* rs = w.resume;
    const int rstate = rs ? rs->state : 0;
    if (rstate == 2) return;  // finished in an earlier launch
    double mu, reg, last_viol = 0.0;
    bool inner_converged = false, failed = false;
    int status = kError, err_code = kErrNone, err_node = -1;
    int inner = 0, outer_count = 0, nrec = 0, alpha_evals = 0, outer0 = 0, pass0 = 0;
    if (rstate == 1) {  // resume at the top of inner pass (outer0, pass0)
      outer0 = rs->outer;
      pass0 = rs->pass;
      outer_count = rs->outer_count;
      inner = rs->inner;
      nrec = rs->nrec;
      alpha_evals = rs->alpha_evals;
      mu = rs->mu;
      reg = rs->reg;
      g_rho = rs->rho;
      last_viol = rs->key;
      t_start -= rs->elapsed;
      for (int k = 0; k < 6; ++k) times[k] = rs->times[k];
    } else {
      if (g.leader()) {
        res->status = kError;
        res->error_code = kErrNone;
        res->error_node = -1;
        res->inner_iterations = 0;
        res->outer_iterations = 0;
        res->n_records = 0;
      }
      if (o.alpha_levels < 1 || o.alpha_levels > kMaxAlpha) {
        if (g.leader()) {
          res->error_code = kErrAlphaLevels;
          if (rs) rs->state = 2;
        }
        return;
      }
      // eta = 0; the caller filled w.u with the initial inputs.
      for (int i = g.item0(t.n * t.max_con), i_e = g.item_end(t.n * t.max_con); i < i_e; i += g.item_step()) w.eta[i] = 0.0;
      if constexpr (NX == 4 && NU == 2) {
        if (structured())  // constant part of every stage record, once per solve
          if (!compact())
            for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) unicycle_stage_constants(mp.dt, is_leaf(i), stage(i));
      }
      g_rho = o.penalty_init;
      if (!rollout()) {
        if (g.leader()) {
          res->error_code = kErrRolloutNonfinite;
          if (rs) rs->state = 2;
        }
        return;
      }
      mu = o.merit_mu_init;
      reg = o.reg_init;
    }
    int budget_used = 0;
    bool resumed = rstate == 1;

    for (int outer = outer0; outer < o.max_outer_iterations; ++outer) {
      int pass_start = 0;
      if (resumed) {
        pass_start = pass0;
        resumed = false;
      } else {
        ++outer_count;
        inner_converged = false;
      }
      for (int pass = pass_start; pass < o.max_inner_iterations; ++pass) {
        if (rs && o.pass_budget > 0 && budget_used++ >= o.pass_budget) {
          // Suspend: everything the loop carries lives in (x, u, eta, records) or here.
          if (g.leader()) {
            rs->state = 1;
            rs->outer = outer;
            rs->pass = pass;
            rs->outer_count = outer_count;
            rs->inner = inner;
            rs->nrec = nrec;
            rs->alpha_evals = alpha_evals;
            rs->mu = mu;
            rs->reg = reg;
            rs->rho = g_rho;
            rs->key = last_viol;
            rs->elapsed = now_s() - t_start;
            for (int k = 0; k < 6; ++k) rs->times[k] = times[k];
          }
          return;
        }
        double t0 = now_s();
        int bad = 0, bad_code = kErrNone;
        mark(9);
        const Eval ev = linearize_evaluate(&bad, &bad_code);
        mark(0);
        if (bad) {
          err_code = bad_code;
          err_node = bad - 1;
          failed = true;
          break;
        }
        double t1 = now_s();
        times[0] += t1 - t0;
        double max_ff = 0.0;
        const int berr = backward(reg, &max_ff);
        double t2 = now_s();
        times[1] += t2 - t1;
        if (berr != kBwdOk) {
          reg = fmax(reg * o.reg_growth, o.reg_min);
          if (reg > o.reg_max) {
            err_code = berr == kIndefinite ? kErrRegCap : kErrFactorization;
            failed = true;
            break;
          }
          continue;
        }
        double a1, a2;
        forward(&a1, &a2);
        double t3 = now_s();
        times[3] += t3 - t2;
        const double ec_full = a1 + a2;
        if (ev.defect_l1 <= o.tol_defect && fabs(ec_full) <= o.tol_cost * (1.0 + fabs(ev.cost_al)) &&
            max_ff <= o.tol_feedforward) {
          inner_converged = true;
          break;
        }
        // update_mu (solver.hpp:400-407)
        {
          double trial = mu;
          if (ev.defect_l1 > o.defect_epsilon) trial = ec_full / ((1.0 - o.merit_gamma) * ev.defect_l1) + o.merit_mu0;
          mu = fmax(trial, mu);
        }
        const double merit0 = ev.cost_al + mu * ev.defect_l1;
        Eval after;
        double merit_after = 0.0, dec = 0.0;
        mark(8);
        int lvl;
        if constexpr (kNL)
          lvl = line_search_nonlinear(o.alpha_levels, merit0, a1, a2, mu, ev.defect_l1, &after, &merit_after, &dec,
                                      &alpha_evals);
        else
          lvl = line_search(o.alpha_levels, merit0, a1, a2, mu, ev.defect_l1, &after, &merit_after, &dec, &alpha_evals);
        mark(7);
        double t4 = now_s();
        times[4] += t4 - t3;
        DevRecord rec;
        rec.outer = outer;
        rec.merit_before = merit0;
        rec.mu = mu;
        rec.max_feedforward = max_ff;
        rec.regularization = reg;
        rec.accepted = lvl >= 0 ? 1 : 0;
        rec.alpha = lvl >= 0 ? ldexp(1.0, -lvl) : 0.0;
        rec.model_decrease = lvl >= 0 ? dec : 0.0;
        if (lvl < 0) {
          reg = fmax(reg * o.reg_growth, o.reg_min);
          rec.merit_after = merit0;
          rec.cost = ev.cost;
          rec.cost_al = ev.cost_al;
          rec.defect_l1 = ev.defect_l1;
          rec.violation = ev.max_violation;
          if (g.leader() && nrec < w.max_records) w.records[nrec] = rec;
          ++nrec;
          last_viol = rec.violation;
          if (reg > o.reg_max) {
            err_code = kErrLineSearch;
            failed = true;
            break;
          }
          continue;
        }
        if constexpr (kNL)
          take_trial();
        else
          take_step(rec.alpha);
        reg = reg / o.reg_decay >= o.reg_min ? reg / o.reg_decay : 0.0;
        ++inner;
        rec.merit_after = merit_after;
        rec.cost = after.cost;
        rec.cost_al = after.cost_al;
        rec.defect_l1 = after.defect_l1;
        rec.violation = after.max_violation;
        if (g.leader() && nrec < w.max_records) w.records[nrec] = rec;
        ++nrec;
        last_viol = rec.violation;
      }
      if (failed) break;
      const Eval ev = evaluate_current();
      if (!t.has_constraints) {
        status = inner_converged ? kConverged : kMaxIterations;
        break;
      }
      if (inner_converged && ev.max_violation <= o.tol_constraint) {
        status = kConverged;
        break;
      }
      if (outer + 1 == o.max_outer_iterations) {
        status = kMaxIterations;
        break;
      }
      update_multipliers(g_rho);
      g_rho = fmin(g_rho * o.penalty_growth, o.penalty_max);
    }
    const Eval fin = evaluate_current();
    times[5] = now_s() - t_start;
    if (g.leader()) {
      res->status = failed ? kError : status;
      res->error_code = err_code;
      res->error_node = err_node;
      res->inner_iterations = inner;
      res->outer_iterations = outer_count;
      res->n_records = nrec;
      res->final_cost = fin.cost;
      res->final_violation = fin.max_violation;
      res->final_defect_l1 = fin.defect_l1;
      for (int k = 0; k < 6; ++k) res->times[k] = times[k];
      res->final_penalty = g_rho;
      if (rs) rs->state = 2;
      res->alpha_evals = alpha_evals;
      res->final_mu = mu;
      res->final_reg = reg;
    }
  }

  // Kernel-level LQR-tree entry (tests): stage records / defects already in
  // place; backward + forward + EC, values copied out.
  __device__ void lqr_tree(double reg, double* scalars) {
    double max_ff = 0.0;
    const int err = backward(reg, &max_ff);
    if (w.value) {
      for (int i = g.item0(t.n), i_e = g.item_end(t.n); i < i_e; i += g.item_step()) {
        if (!seq_seg(t.node_seg[i])) {
          const double* v = value_of(i);
          copy<NX * NX>(v + BL::P, w.value + static_cast<size_t>(i) * VL::stride + VL::P);
          copy<NX>(v + BL::p, w.value + static_cast<size_t>(i) * VL::stride + VL::p);
        }
      }
    }
    g.sync();
    double a1 = 0, a2 = 0;
    if (err == kBwdOk) forward(&a1, &a2);
    if (g.leader()) {
      scalars[0] = max_ff;
      scalars[1] = a1;
      scalars[2] = a2;
      scalars[3] = err;
    }
  }
};


}  // namespace bmpc_b200
