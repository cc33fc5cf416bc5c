/* pdlp_b200.h — C-ABI boundary of the B200-native restarted-PDHG solver.
 *
 * The reference (`pdhglp`, /root/reference/proj/include/pdhglp) is a
 * header-only C++20 library with no FFI. Its drop-in boundary for the hot
 * path is the C++ API below; every entry point here replaces one of them:
 *
 *   pdlp_create + pdlp_solve      <- pdhglp::solve(const GeneralFormLp&, const SolverParams&)
 *                                    solver.hpp:935-940 (SolveLoop ctor :636-646, run :759-929)
 *   pdlp_get_solution             <- SolveResult::point / ::reduced (solver.hpp:618-630)
 *   pdlp_get_step_log             <- SolveResult::step_log   (StepLogEntry, solver.hpp:596-604)
 *   pdlp_get_restart_log          <- SolveResult::restart_log (RestartEvent, solver.hpp:606-616)
 *   pdlp_spmv                     <- spmv / spmv_transpose (sparse_matrix.hpp:117-165)
 *   pdlp_get_scaling              <- make_scaling(vstack(G,A), ...) (scaling.hpp:117-132)
 *   pdlp_iterate_begin/run/get    <- SolveLoop::run's loop body, exposed for iterate parity
 *                                    (solver.hpp:759-841; detail::adaptive_step_cached :381-467)
 *   pdlp_read_mps / pdlp_parse_mps <- read_mps_file / parse_mps + to_general_form
 *                                    (mps_io.hpp:163-585), host C++ inside the library
 *   pdlp_write_solution           <- write_solution (solution_io.hpp:70-95)
 *
 * Conventions (mirroring the reference):
 *   - plain pointers and sizes, no C++/torch types; caller-owned inputs are
 *     read-only and may be freed once pdlp_create returns (they are copied to HBM);
 *   - every function returns PDLP_OK (0) or an error code and never throws;
 *     PDLP_EINVAL corresponds to std::invalid_argument in the reference
 *     (lp_model.hpp:45-72, solver.hpp:79-93), PDLP_ERUNTIME to std::runtime_error;
 *   - numerical trouble is a *status* (PDLP_STATUS_NUMERICAL_ERROR), not an error code
 *     (solver.hpp:811-817);
 *   - one handle per host thread; distinct handles may run concurrently.
 */
#ifndef PDLP_B200_H_
#define PDLP_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDLP_ABI_VERSION 1

/* ---- return codes ---------------------------------------------------- */
enum {
  PDLP_OK = 0,
  PDLP_EINVAL = 1,   /* std::invalid_argument in the reference */
  PDLP_ERUNTIME = 2, /* std::runtime_error */
  PDLP_ECUDA = 3,    /* CUDA / NCCL failure */
  PDLP_ESTATE = 4    /* call order violated (e.g. get_solution before solve) */
};

/* ---- SolveStatus (solver.hpp:26-33), same order ----------------------- */
enum {
  PDLP_STATUS_OPTIMAL = 0,
  PDLP_STATUS_PRIMAL_INFEASIBLE = 1,
  PDLP_STATUS_DUAL_INFEASIBLE = 2,
  PDLP_STATUS_ITERATION_LIMIT = 3,
  PDLP_STATUS_TIME_LIMIT = 4,
  PDLP_STATUS_NUMERICAL_ERROR = 5,
  PDLP_STATUS_RUNNING = 6 /* only returned by pdlp_iterate_run */
};

/* ---- RestartCriterion (solver.hpp:47) -------------------------------- */
enum {
  PDLP_RESTART_NONE = 0,
  PDLP_RESTART_SUFFICIENT_DECAY = 1,
  PDLP_RESTART_NECESSARY_DECAY = 2,
  PDLP_RESTART_LONG_INNER_LOOP = 3
};

/* ---- ScalingMode (scaling.hpp:16) ------------------------------------ */
enum { PDLP_SCALING_NONE = 0, PDLP_SCALING_RUIZ = 1, PDLP_SCALING_RUIZ_PC = 2 };

/* ---- MpsFormat (mps_io.hpp:40) --------------------------------------- */
enum { PDLP_MPS_FIXED = 0, PDLP_MPS_FREE = 1, PDLP_MPS_AUTO = 2 };

/* ---- execution modes (B200 extension) -------------------------------- */
enum {
  /* Fast deterministic mode: load-balanced tiled SpMV, tree reductions in a
   * fixed order. Bitwise identical run to run, ~1e-16 relative from the CPU. */
  PDLP_MODE_FAST = 0,
  /* Parity mode: every sum is accumulated in the reference's sequential index
   * order and no FMA is contracted, so iterates are bitwise identical to the
   * CPU reference. Intended for verification on small instances. */
  PDLP_MODE_PARITY = 1
};

/* ---- iteration engines (B200 extension) ----------------------------- */
enum {
  /* GRAPH (STREAM if use_cuda_graph == 0) */
  PDLP_ENGINE_AUTO = 0,
  /* reserved: a removed persistent window engine (measured 2x slower than
   * GRAPH); rejected with PDLP_EINVAL */
  PDLP_ENGINE_PERSISTENT = 1,
  /* CUDA graph: WHILE(conditional node) { dual kernel; primal kernel } */
  PDLP_ENGINE_GRAPH = 2,
  /* plain stream launches of the per-trial kernels */
  PDLP_ENGINE_STREAM = 3
};

/* CSR of one constraint block; mirrors CsrMatrix (sparse_matrix.hpp:35-55).
 * Invariants expected (as produced by CsrMatrix::from_triplets):
 * row_offsets[0]==0, row_offsets[num_rows]==nnz, nondecreasing; column indices
 * strictly increasing within a row; no stored zeros. Indices are 64-bit like
 * the reference's index_t (sparse_matrix.hpp:21); `col_indices32` may be given
 * instead of `col_indices` to skip the device-side narrowing. */
typedef struct {
  int64_t num_rows;
  int64_t num_cols;
  int64_t nnz;
  const int64_t* row_offsets; /* num_rows + 1 */
  const int64_t* col_indices; /* nnz, or NULL when col_indices32 is set */
  const int32_t* col_indices32;
  const double* values; /* nnz */
} pdlp_csr;

/* GeneralFormLp (lp_model.hpp:24-43):  min c'x  s.t. Gx >= h, Ax = b, l <= x <= u. */
typedef struct {
  pdlp_csr inequality_matrix; /* G, m1 x n */
  pdlp_csr equality_matrix;   /* A, m2 x n */
  int64_t num_variables;      /* n */
  const double* objective;      /* c, n */
  const double* inequality_rhs; /* h, m1 */
  const double* equality_rhs;   /* b, m2 */
  const double* lower;          /* l, n, -inf allowed */
  const double* upper;          /* u, n, +inf allowed */
  double objective_constant;
} pdlp_lp;

/* SolverParams (solver.hpp:59-77), same fields and defaults, plus the B200
 * execution knobs at the end. Fill with pdlp_default_params first. */
typedef struct {
  double eps_optimal;          /* 1e-4 */
  double eps_infeasible;       /* 1e-8 */
  double time_limit_seconds;   /* 3600 */
  int64_t iteration_limit;     /* INT64_MAX */
  double beta_sufficient;      /* 0.2 */
  double beta_necessary;       /* 0.8 */
  double beta_artificial;      /* 0.36 */
  double theta_smoothing;      /* 0.5 */
  double eps_zero;             /* 1e-10 */
  int64_t evaluation_frequency; /* 64 */
  int32_t scaling;             /* PDLP_SCALING_RUIZ_PC */
  int32_t ruiz_iterations;     /* 10 */
  double pock_chambolle_alpha; /* 1.0 */
  double step_reduction_exponent; /* 0.3 */
  double step_growth_exponent;    /* 0.6 */
  double omega_min;            /* 1e-8 */
  double omega_max;            /* 1e8 */
  int32_t record_step_log;     /* 0 */
  /* ---- B200 extensions ---- */
  int32_t device;              /* CUDA ordinal, default 0 */
  int32_t mode;                /* PDLP_MODE_FAST */
  int32_t use_cuda_graph;      /* 1: replay each evaluation window as a CUDA graph */
  int32_t l2_persist;          /* 1: pin the gathered iterate in L2 (access-policy window); default 0 */
  int32_t engine;              /* PDLP_ENGINE_*: how a window of iterations is driven */
  /* Row sharding: this handle is rank `rank` of `world_size`
   * ranks (one per GPU), each running its contiguous share of the rows of K
   * and of K^T; peers are linked with pdlp_shard_link_local (ranks in one
   * process) or pdlp_shard_export / pdlp_shard_import (one process per GPU,
   * CUDA IPC over NVLink). Fast mode only. */
  int32_t world_size;          /* 1 */
  int32_t rank;                /* 0 */
  /* Tile breaks of a plan_world-way partition while running all rows on this
   * handle (verification: a world_size = 1 run with plan_world = P matches a
   * P-rank run bit for bit). 0 = world_size. */
  int32_t plan_world;
  int32_t reserved[3];
} pdlp_params;

/* ConvergenceInfo (solver.hpp:165-177) plus SolveResult scalars (:618-630). */
typedef struct {
  int32_t status;
  int32_t has_certificate;
  int64_t iterations;
  int64_t restarts;
  double solve_seconds;  /* loop time, excludes setup like the reference (:636-646,760) */
  double setup_seconds;  /* upload + K^T build + preconditioning (B200 extension) */
  double device_seconds; /* solve loop timed with CUDA events on the solver's stream */
  double window_seconds; /* time inside the iteration kernels (windows), CUDA events */
  double primal_objective;
  double dual_objective;
  double primal_objective_raw;
  double dual_objective_raw;
  double gap_abs;
  double primal_residual_norm;
  double dual_residual_norm;
  double relative_gap;
  double relative_primal_residual;
  double relative_dual_residual;
  double kkt_omega;
  int64_t step_log_size;
  int64_t restart_log_size;
  int64_t num_variables;
  int64_t num_constraints;
  int64_t trials;        /* total line-search trials (B200 extension) */
  int64_t evaluations;   /* evaluation blocks run (B200 extension) */
  int64_t gpu_launches;  /* kernels launched by the solve loop (B200 extension) */
  double eval_seconds;   /* time inside the evaluation kernels, CUDA events (B200 extension) */
  char message[256];
} pdlp_result_info;

/* StepLogEntry (solver.hpp:596-604) */
typedef struct {
  int64_t step_counter;
  double omega;
  double eta_accepted;
  double eta_bar;
  double eta_next;
  double movement_sq;
  double interaction;
} pdlp_step_log_entry;

/* RestartEvent (solver.hpp:606-616) */
typedef struct {
  int64_t total_iterations;
  int64_t epoch_length;
  int32_t criterion;
  int32_t candidate_is_average;
  double kkt_candidate;
  double kkt_previous_candidate;
  double kkt_epoch_start;
  double omega_before;
  double omega_after;
} pdlp_restart_event;

typedef struct pdlp_handle pdlp_handle;

/* Which operator pdlp_spmv applies. The scaled operator is the saddle
 * matrix K~ = D1 (G;A) D2 the loop iterates on (solver.hpp:644); the original
 * one is (G;A) as evaluate_point sees it (lp_model.hpp:184-187,205-207). */
enum {
  PDLP_OP_K_SCALED = 0,
  PDLP_OP_KT_SCALED = 1,
  PDLP_OP_K_ORIGINAL = 2,
  PDLP_OP_KT_ORIGINAL = 3
};

int pdlp_abi_version(void);

/* Number of visible CUDA devices (0 when the driver reports none); used by the
 * benchmark harness to spread worker threads over GPUs (bench.hpp:212-222). */
int pdlp_device_count(int32_t* count);
void pdlp_default_params(pdlp_params* params);

/* Validates (GeneralFormLp::validate lp_model.hpp:45-72, SolverParams::validate
 * solver.hpp:79-93), copies the instance to HBM, builds K^T on the device,
 * preconditions (Ruiz x ruiz_iterations then Pock-Chambolle) on the device. */
int pdlp_create(const pdlp_lp* lp, const pdlp_params* params, pdlp_handle** out);
void pdlp_destroy(pdlp_handle* h);

/* Runs restarted PDHG from z = 0 (solver.hpp:759-929). May be called again:
 * every call restarts from z = 0 on the resident, preconditioned instance. */
int pdlp_solve(pdlp_handle* h, pdlp_result_info* info);

/* Result vectors of the last solve (unscaled point or certificate ray, and
 * its reduced costs). Any pointer may be NULL. x, lambda*: n; y: m. */
int pdlp_get_solution(pdlp_handle* h, double* x, double* y, double* lambda,
                      double* lambda_pos, double* lambda_neg);
int pdlp_get_step_log(pdlp_handle* h, pdlp_step_log_entry* out, int64_t capacity);
int pdlp_get_restart_log(pdlp_handle* h, pdlp_restart_event* out, int64_t capacity);

/* D1 (m) and D2 (n) of the preconditioner. */
int pdlp_get_scaling(pdlp_handle* h, double* row_scale, double* col_scale);

/* out = op(in) with host buffers (kernel-level parity). */
int pdlp_spmv(pdlp_handle* h, int32_t op, const double* in, double* out);

/* Stepwise driving of the same loop pdlp_solve runs (for iterate parity):
 * begin = initialisation + initial evaluation (solver.hpp:764-792);
 * run = up to n more accepted iterations, with the evaluation/restart block
 * whenever the inner counter hits evaluation_frequency; *status receives
 * PDLP_STATUS_RUNNING or the terminal status. */
int pdlp_iterate_begin(pdlp_handle* h, int32_t* status);
int pdlp_iterate_run(pdlp_handle* h, int64_t n, int32_t* status);
/* Current scaled iterate and its product caches (any pointer may be NULL);
 * counters = {total k, inner t, outer n, trials}; scalars = {eta, eta_hat, omega,
 * weight_sum}. */
int pdlp_get_iterate(pdlp_handle* h, double* x, double* y, double* kx, double* kty,
                     int64_t* counters, double* scalars);

/* Times `reps` launches of one iteration kernel on the live solver state with
 * CUDA events on the launching stream (bench roofline). which: 0 = dual
 * (K x' fused update), 1 = primal (K^T y' fused update). Returns avg ms and the
 * algorithmic bytes one launch moves. */
int pdlp_time_kernel(pdlp_handle* h, int32_t which, int32_t reps, double* avg_ms,
                     double* bytes_per_launch);
/* One plain PDHG step with explicit extrapolation, pdhg_raw_step
 * (solver.hpp:335-358), on the handle's UNSCALED saddle problem
 * (to_saddle(lp), lp_model.hpp:88-98): x' = clamp(x - tau (c - K'y)),
 * y' = proj(y + sigma (q - K(2x' - x))). x, x_out: n; y, y_out: m (host).
 * Parity mode: bitwise equal to the reference; fast mode: the tiled engine's
 * row sums. Test-facing in the reference (test_solver.cpp:33-61); not used by
 * pdlp_solve. */
int pdlp_pdhg_raw_step(pdlp_handle* h, const double* x, const double* y, double tau, double sigma,
                       double* x_out, double* y_out);

/* Bytes of one launch of kernel `which` (0 dual, 1 primal, 2 SpMV K x, 3 SpMV
 * K^T y): out[0] = SURVEY.md §8(d)'s algorithmic bytes (what pdlp_time_kernel
 * reports), out[1] = the bytes the launched variant moves at one DRAM access
 * per element (bounds skipped when all [0, +inf), K'y' not stored under lazy
 * K'y, column panels' counts / block offsets / running sums), out[2] = the
 * operator's column-panel count (0: one tiled pass). (new; bench roofline) */
int pdlp_kernel_bytes(pdlp_handle* h, int32_t which, double* out);

/* Problem sizes after create: {n, m, m1, nnz}. */
int pdlp_get_sizes(pdlp_handle* h, int64_t* sizes);

/* ---- standard-form theory harness (standard_form.hpp:36-211) ------------- */

/* min c'x s.t. Ax = b, x >= 0 with A an m x n CSR (pdlp_csr), b (m), c (n).
 * parity = 1: sequential sums in the reference's order (bitwise with
 * restarted_pdhg_standard / kkt_error_standard / spectral_norm); 0: tiled,
 * tree-reduced (fast). */
typedef struct {
  double step_size;        /* s, both primal and dual step; must be > 0 */
  double restart_decay;    /* beta in (0, 1); default 0.5 */
  double convergence_tol;  /* stop once the epoch-start KKT error <= this; default 1e-9 */
  int64_t iteration_limit; /* default 1000000 */
  int32_t parity;
  int32_t device;
  int64_t reserved[4];
} pdlp_standard_options;

void pdlp_standard_default_options(pdlp_standard_options* options);

/* restarted_pdhg_standard (standard_form.hpp:131-211) on the GPU, from z = 0
 * or (x0, y0) when both are given. Per epoch (up to `cap`): its start KKT
 * error and length. counters[4] = {epochs, total_iterations, converged,
 * numerical_failure}. x_out (n) / y_out (m), optional: the last epoch's
 * start point. iter_x ([iter_cap][n]) /
 * iter_y ([iter_cap][m]), optional: record_iterates, the iterate after each of
 * the first iter_cap iterations (epoch by epoch, split by `lengths`). Invalid
 * options return PDLP_EINVAL with StandardPdhgOptions::validate's message. */
int pdlp_standard_pdhg(const pdlp_csr* a, const double* b, const double* c, const pdlp_standard_options* options,
                       const double* x0, const double* y0, double* start_kkt, int64_t* lengths, int64_t cap,
                       int64_t* counters, double* x_out, double* y_out, double* iter_x, double* iter_y,
                       int64_t iter_cap);

/* kkt_error_standard (standard_form.hpp:37-58):
 * ||(Ax - b; [-x]+; [A'y - c]+; [c'x - b'y]+)||_2 */
int pdlp_kkt_error_standard(const pdlp_csr* a, const double* b, const double* c, const double* x,
                            const double* y, int32_t parity, int32_t device, double* out);

/* spectral_norm (standard_form.hpp:63-89): largest singular value of A by
 * power iteration on A'A from the normalised all-ones vector. */
int pdlp_spectral_norm(const pdlp_csr* a, double tol, int32_t max_iterations, int32_t parity, int32_t device,
                       double* out);

/* p_s_norm_squared (standard_form.hpp:92-98): ||x||^2 + ||y||^2 + 2 s y'Ax. */
int pdlp_p_s_norm_squared(const pdlp_csr* a, const double* b, const double* c, double step, const double* x,
                          const double* y, int32_t parity, int32_t device, double* out);

/* ---- CSR construction on the GPU --------------------------------------- */

/* CsrMatrix::from_triplets (sparse_matrix.hpp:57-108) on device `device`:
 * sorted by (row, col), duplicates summed in input order, exact zeros dropped.
 * Outputs: row_offsets (rows + 1), col_indices / values (capacity nt);
 * *nnz_out = stored entries. An out-of-range triplet returns PDLP_EINVAL with
 * the reference's message naming the first one. Integer output is bit-exact
 * with the reference; values too wherever a (row, col) occurs at most twice. */
int pdlp_csr_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* r, const int64_t* c,
                           const double* v, int32_t device, int64_t* row_offsets, int64_t* col_indices,
                           double* values, int64_t* nnz_out);

/* ---- row sharding (B200 extension) ---------------------------------- */

/* Size of one rank's exported shard blob. */
int64_t pdlp_shard_blob_size(void);
/* Links the `world` ranks of one sharded solve that live in this process
 * (handles in rank order; typically all on one device: the loopback transport
 * used for verification). Their pdlp_solve calls must then run concurrently,
 * one host thread per rank. */
int pdlp_shard_link_local(pdlp_handle** handles, int32_t world);
/* One process per GPU: every rank exports its blob (CUDA IPC handles of the
 * buffers its peers write into), the caller all-gathers the blobs (e.g. over
 * torch.distributed), then every rank imports all of them in rank order. */
int pdlp_shard_export(pdlp_handle* h, void* blob, int64_t capacity);
int pdlp_shard_import(pdlp_handle* h, const void* blobs, int32_t world);
/* {world, rank, row0, row1, col0, col1, own K tiles, own K^T tiles, K tiles, K^T tiles} */
int pdlp_shard_info(pdlp_handle* h, int64_t* out);
/* Per-trial exchange and storage of this rank: out[0] = x' and y' values it
 * pushes to peers (only to the ranks whose rows gather each value, SURVEY
 * §8e's coupling-only exchange), out[1] = the values an all-to-all push would
 * send ((own columns + own rows) * (world - 1)), 8 bytes each; out[2], out[3]
 * = nonzeros of K and of K^T stored on this rank (a rank keeps only its own
 * rows after setup). `out` holds 4 values. (new) */
int pdlp_shard_exchange(pdlp_handle* h, int64_t* out);
/* Host-only: the row cuts (world + 1 each) of K = (G; A) and of K^T that a
 * world-way sharded solve of `lp` uses. No device work. */
int pdlp_plan_shards(const pdlp_lp* lp, int32_t world, int64_t* k_cuts, int64_t* kt_cuts);
/* Host-only: the gather masks of that partition (bit q of xmask[j]: a row of
 * K owned by rank q holds column j; bit q of ymask[i]: row i holds a column
 * owned by rank q; both optional, n and m entries) and, per rank, the x' / y'
 * values a trial pushes to peers with the masks (pushed[world]) and with an
 * all-to-all push (all_to_all[world]). No device work; the device builds the
 * same masks at pdlp_create (pdlp_shard_exchange). */
int pdlp_plan_exchange(const pdlp_lp* lp, int32_t world, int64_t* pushed, int64_t* all_to_all, uint32_t* xmask,
                       uint32_t* ymask);

/* ---- LP files (host I/O; no device work) ----------------------------- */

/* An LP read from MPS text, owning its arrays (64-bit indices). */
typedef struct pdlp_lp_file pdlp_lp_file;

/* read_mps_file (mps_io.hpp:582-585): format PDLP_MPS_*; a path ending in
 * ".gz" is inflated. Parse errors return PDLP_ERUNTIME with
 * "mps parse error at line N: ..." (MpsParseError, mps_io.hpp:26-36); crossing
 * bounds return PDLP_EINVAL (mps_io.hpp:536-546). */
int pdlp_read_mps(const char* path, int32_t format, pdlp_lp_file** out);
/* parse_mps + to_general_form (mps_io.hpp:163-554) on in-memory text. */
int pdlp_parse_mps(const char* text, int64_t length, int32_t format, pdlp_lp_file** out);
/* View of the GeneralFormLp (valid until pdlp_lp_file_free). */
const pdlp_lp* pdlp_lp_file_lp(const pdlp_lp_file* f);
/* NAME record and column names (index < num_variables). */
const char* pdlp_lp_file_name(const pdlp_lp_file* f);
const char* pdlp_lp_file_column_name(const pdlp_lp_file* f, int64_t index);
void pdlp_lp_file_free(pdlp_lp_file* f);

/* write_solution (solution_io.hpp:70-95): "format_version 1" key-value file with
 * status, objectives, relative gap, residual norms, iterations and
 * solve_seconds from *info; x (n) / y (m) blocks are written when non-NULL. */
int pdlp_write_solution(const char* path, const pdlp_result_info* info, const double* x,
                        int64_t n, const double* y, int64_t m);

/* Thread-local message of the last failing call (valid until the next call). */
const char* pdlp_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PDLP_B200_H_ */
