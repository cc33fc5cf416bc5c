// device_state.h — layouts shared by the host runtime and the kernels.
#pragma once

#include <stdint.h>

#include "tiles.h"

namespace pdlp {

// Which branch the primal kernel takes (set by the dual kernel's decision).
enum PMode : int32_t { kPNone = 0, kPAccept = 1, kPRetry = 2, kPRestart = 3 };

// Scalar solver state resident in HBM. The host owns the fields above the
// marker between windows (uploads them before a window), the kernels own the
// rest during a window (downloaded after it).
struct DevState {
  double eta;       // step size of the next trial (eta-hat at a step start)
  double omega;     // primal weight
  double wsum;      // WeightedAverage weight sum (vector_ops.hpp:95-107)
  int64_t total;    // k
  int64_t inner;    // t
  int64_t table_base;  // total at window start (index base of the factor table)
  int32_t window_target;
  int32_t p_mode;
  int32_t ix_cur, ix_prev, ix_trial;  // rotation of the three x buffers
  int32_t iy_cur, iy_prev, iy_trial;  // rotation of the three y buffers
  int32_t ikx_cur, ikty_cur;          // rotation of the two Kx / K'y buffers
  int32_t record_log;
  int32_t pad0;
  // ---- kernel-owned during a window ----
  int32_t window_accepts;
  int32_t trials_in_step;
  int64_t trials_total;
  int32_t failure;
  int32_t accepted;
  double avg_ratio;
  int32_t avg_first;
  int32_t pad1;
  double eta_acc, eta_bar, eta_next, mov, inter;  // last accepted step
  unsigned ctr_dual;
  unsigned ctr_eval;
  int32_t window_cont;  // unused (layout)
  int32_t pad2;
  // ---- window chaining (graph engine, fast mode; chain_decide_kernel) ----
  double kkt_epoch_start;  // the host's restart-test values, mirrored for the device
  double kkt_last;
  int32_t chain_left;      // windows the chain may still start after this one
  int32_t chain_stop;      // 0 running; 1 the last evaluation needs the host; 2 handled
  int32_t chain_evals;     // evaluations decided on the device in this chain
  int32_t pad3;
};

// Constants of the evaluation block's decisions (SolverParams and the
// instance's termination norms), for the device-side chain decision.
struct ChainConsts {
  double eps_optimal, eps_infeasible, eps_zero;
  double beta_sufficient, beta_necessary, beta_artificial;
  double rhs_norm, obj_norm;
  int64_t iteration_limit;
  int32_t freq;
  int32_t pad;
};

// Results of one evaluation block (evaluate_candidates + the infeasibility
// rays, solver.hpp:705-739, :853-885) for four points carried side by side:
// slot 0 = current, 1 = average, 2 = last-step delta ray, 3 = normalized ray.
struct EvalOut {
  // KKT points (slots 0, 1): KktResiduals (solver.hpp:109-123)
  double prn[2], drn[2], pobj[2], dobj[2];
  // rays (slots 2, 3): certificate_from_ray (solver.hpp:503-574)
  double y_norm[2], kty_resid[2], ray_dobj[2];
  double x_norm[2], ax_norm[2], gx_negmax[2], xl_negmax[2], xu_max[2], cx[2];
  // restart displacement of each candidate vs the epoch start (scaled space)
  double dx2[2], dy2[2];
};

// ---------------------------------------------------------------------------
// Row sharding across ranks (one rank per GPU)
// ---------------------------------------------------------------------------
constexpr int kMaxShards = 8;
constexpr int kEvalReduceCtas = 32;  // first level of the evaluation reductions

// Barrier kinds: each participating launch of a producer kernel bumps its
// local count and publishes it to every peer's flag slot; a consumer waits
// until every rank's flag reached its own local count (BSP epochs).
enum SyncKind : int32_t {
  kSyncDual = 0,    // y', K x' rows, dual partials
  kSyncPrimal = 1,  // x', primal partials
  kSyncAvg = 2,     // average slices (once per window, before the evaluation)
  kSyncEvRows = 3,  // evaluation partials over K
  kSyncEvCols = 4,  // evaluation partials over K^T (and reduced costs at finish)
  kSyncKinds = 5
};

// Per-rank synchronisation block in the rank's own HBM, mapped by the peers.
struct ShardSync {
  unsigned long long flag[kSyncKinds][kMaxShards];  // written remotely by rank q
  unsigned long long count[kSyncKinds];             // local participating launches
  unsigned ticket[kSyncKinds];                      // local last-CTA tickets
  int timeout;                                      // a wait gave up (peer lost)
  int pad;
};

// Device pointers (valid on this rank: local, or CUDA-IPC-mapped peer memory)
// of every rank's exchanged buffers. Entry `rank` is the rank's own buffer.
struct ShardView {
  double* x_all[kMaxShards];   // the three x buffers, 3 n
  double* y_all[kMaxShards];   // the three y buffers, 3 m
  double* d_part[kMaxShards];  // dual partials [K tiles * 3]
  double* p_part[kMaxShards];  // primal partials [2][K^T tiles * 2]
  double* avg_x[kMaxShards];
  double* avg_y[kMaxShards];
  double* part1[kMaxShards];   // evaluation partials over K
  double* part2[kMaxShards];   // evaluation partials over K^T
  double* lam[kMaxShards];     // [4][n] reduced costs
  ShardSync* sync[kMaxShards];
};

// Device pointers of one CSR operator with its tile plan.
struct DevCsr {
  const int* rp;
  const int* col;
  const double* val;       // scaled (iteration) values
  const double* val_orig;  // original values (evaluation)
  int rows;
  int cols;
  int64_t nnz;
  const Tile* tiles;       // the GLOBAL tile list of the operator
  int ntiles;              // tiles this rank runs: tiles[tile0 .. tile0 + ntiles)
  int tile0;               // global index of the first (partials are indexed globally)
  int chunk_slots;
  double* chunk_part;     // [chunk_slots * 8]
  unsigned* chunk_ctr;    // [split_rows]
};

// Vectors of the iteration (all device pointers, fixed for the graph's life).
struct DevIter {
  double* x[3];
  double* y[3];
  double* kx[2];
  double* kty[2];
  double* avg_x;
  double* avg_y;
  double* x_start;
  double* y_start;
  const double* c;   // scaled objective
  const double* l;   // scaled bounds
  const double* u;
  const double* q;   // scaled rhs (h; b)
  int n, m, m1;
  int p_grid;        // CTAs of the primal kernel (own K^T tiles + avg_y blocks)
  int p_tiles;       // global K^T tiles = primal partials per parity half
  int nonneg;        // every scaled bound is l = +0, u = +inf: clamp is max(v, 0)
  int avg_blocks;    // trailing CTAs of the primal kernel that update avg_y
  double* d_part;    // [K tiles * 3]
  double* p_part;    // [2][p_grid * 2], ping-pong by trial parity
  double* px_total;  // unused (kept for layout stability)
  DevState* snap;    // state the current trial's dual kernel ran on (fast mode)
  int d_tiles;       // global K tiles (dual partials the decision sums)
  int kty_lazy;      // 1: accepted steps do not store K'y' (recomputed by a retry)
  int prefetch;      // 1: kernels pull their tile (and the primal its operands) to L2 early
  int decide_sep;    // 1: the step decision runs in its own one-CTA kernel (many
                     //    tiles); 0: every primal CTA recomputes it at its head
  double* seq_dy2;   // parity-mode per-row terms (m)
  double* seq_inter; // (m)
  double* seq_dx2;   // (n)
  // step factors of the window, interleaved: red_tab[2i] = 1-(k+1)^-0.3,
  // red_tab[2i+1] = 1+(k+1)^-0.6 for k = table_base + i (uploaded with the state)
  const double* red_tab;
  void* step_log;         // pdlp_step_log_entry[window capacity]
  DevState* st;
  // ---- sharding (world == 1: single device, everything below unused) ----
  int world, rank;
  int spin;                // 1: consumers wait on peer flags in-kernel (one process per GPU)
  int row0, row1;          // own rows of K (y, K x, avg_y slices)
  int col0, col1;          // own rows of K^T = columns (x, K'y, avg_x slices)
  const ShardView* shv;    // peer table (device memory)
  ShardSync* sync;         // own sync block
  // per value, the peers whose rows read it (bit q: rank q), so a trial pushes
  // x' / y' only where it is gathered; nullptr: every peer
  const unsigned* xmask;   // (n) ranks whose rows of K hold column j
  const unsigned* ymask;   // (m) ranks whose rows of K^T (columns of K) hold row i
};

// Vectors of the evaluation block.
struct DevEval {
  double* X4;   // [n][4] unscaled x of the four points
  double* Y4;   // [m][4] unscaled y (rays projected onto the dual cone)
  double* lam;  // [4][n] reduced costs lambda of the four points
  const double* c;   // original objective
  const double* l;   // original bounds
  const double* u;
  const double* q;   // original rhs (h; b)
  const double* d1;  // row scale
  const double* d2;  // col scale
  double objective_constant;
  double* part0;  // EV0 partials [grid0 * 4]
  double* part1;  // EV1 partials [K tiles * 14]
  double* part2;  // EV2 partials [KT tiles * 18]
  int grid0;
  double* seq_r;  // parity: [4][m] row residual terms
  double* seq_d;  // parity: [4][n] column residual terms
  EvalOut* out;
  int ev1_tiles, ev2_tiles;  // global evaluation tile counts (partials summed)
  double* stage;             // [36][kEvalReduceCtas] first-level sums of the partials
  int world, rank;           // sharding (see DevIter)
  const ShardView* shv;
  ShardSync* sync;
};

}  // namespace pdlp
