// kernels.cuh — declarations of the host-side launchers in kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <functional>

#include "device_state.h"

namespace pdlp {

// Host hook run after each launch whose outputs peers consume (sharded runs in
// one process order their ranks' streams through it; empty otherwise).
using PhaseFn = std::function<void()>;

// ---- setup -----------------------------------------------------------------
void launch_build_rowptr(const int64_t* g_off, const int64_t* a_off, int64_t m1, int64_t m2,
                         int64_t nnz_g, int* rp, cudaStream_t s);
void launch_narrow_cols(const int64_t* col64, int* col32, int64_t nnz, int n, int* err,
                        cudaStream_t s);
void launch_check_cols(const int* col32, int64_t nnz, int n, int* err, cudaStream_t s);
void launch_check_rows(const int* rp, const int* col, int rows, int* err, cudaStream_t s);
void launch_expand_rows(const int* rp, int rows, int* row_of, cudaStream_t s);
void launch_iota(int* p, int64_t n, cudaStream_t s);
void launch_count_cols(const int* col, int64_t nnz, int* counts, cudaStream_t s);
void launch_gather_transpose(const int* perm, const int* row_of, const double* val, int64_t nnz,
                             int* col_t, double* val_t, cudaStream_t s);
void launch_fill(double* p, int64_t n, double v, cudaStream_t s);
// out[i] = v4[4 i + slot] (one point of an interleaved evaluation array)
void launch_extract_slot(const double* v4, int slot, int64_t n, double* out, cudaStream_t s);
// Planner flags per row (more than min_len entries): 2 = first of four
// column-shifted rows; 1 = mostly consecutive columns (when want_contig); 0 = neither
void launch_row_contig(const int* rp, const int* col, int rows, int min_len, int want_contig,
                       unsigned char* out, cudaStream_t s);
void launch_fill_int(int* p, int64_t n, int v, cudaStream_t s);
// Ruiz (scaling.hpp:52-66): out[r] = max_k |v_k * (d_row[r] * d_col[col_k])|
void launch_row_absmax(const int* rp, const int* col, const double* val, int rows,
                       const double* d_self, const double* d_other, double* out, cudaStream_t s,
                       double avg_len = 1e9);
// Pock-Chambolle (scaling.hpp:72-94): out[r] = sequential sum_k |v*(d*d)|^p, then the
// row's pow(acc, 1/p) exactly as row_norms/col_norms (sparse_matrix.hpp:212-255)
void launch_row_pnorm(const int* rp, const int* col, const double* val, int rows,
                      const double* d_self, const double* d_other, double p, double* out,
                      cudaStream_t s);
void launch_ruiz_update(double* d, const double* norm, int n, cudaStream_t s);
void launch_pc_update(double* d, const double* sum, int n, double p, cudaStream_t s);
void launch_scale_values(const int* rp, const int* col, const double* val_orig, int rows,
                         const double* d_self, const double* d_other, double* val_out,
                         cudaStream_t s);
void launch_scale_vectors(const double* c, const double* l, const double* u, const double* q,
                          const double* d1, const double* d2, int n, int m, double* cs,
                          double* ls, double* us, double* qs, cudaStream_t s);
void launch_block_absmax(const double* v, int64_t n, double* partials, int nblocks,
                         cudaStream_t s);

// ---- iteration -------------------------------------------------------------
// out = A x with the tiled engine (parity: sequential rows, fast: tiled).
void launch_spmv(const DevCsr& a, bool orig_vals, const double* x, double* out, bool seq,
                 cudaStream_t s);
// Trial of adaptive_step_cached (solver.hpp:404-466) on the dual side, plus the
// step decision; sets the WHILE condition when `cond` != 0.
void launch_dual(const DevCsr& k, const DevIter& it, bool seq, unsigned long long cond,
                 int use_cond, cudaStream_t s);
// Separate step decision (it.decide_sep): sums the dual partials once.
void launch_decide(const DevIter& it, cudaStream_t s, unsigned long long cond = 0, int use_cond = 0);
// The evaluation block's decision on the device for chained windows: when the
// evaluation neither terminates, certifies infeasibility nor restarts, records
// kkt_last and starts the next window (outer / inner WHILE conditions);
// otherwise stops the chain for the host (Solver::evaluation_block).
void launch_chain_decide(DevState* st, const EvalOut* e, const ChainConsts& k, unsigned long long outer,
                         unsigned long long inner, cudaStream_t s);
// Primal side: K'y' + average + next trial x' (mode from state, or forced).
void launch_primal(const DevCsr& kt, const DevIter& it, bool seq, int mode_override,
                   cudaStream_t s, unsigned long long cond = 0, int use_cond = 0);
void launch_zero_iterate(const DevIter& it, cudaStream_t s);
void launch_restart_copy(const DevIter& it, int from_avg, cudaStream_t s);

// ---- pdhg_raw_step (solver.hpp:335-358) ---------------------------------------
void launch_raw_primal(const double* x, const double* kty, const double* c, const double* l, const double* u,
                       double tau, int64_t n, double* xo, double* ext, cudaStream_t s);
void launch_raw_dual(const double* y, const double* kext, const double* q, double sigma, int64_t m, int64_t m1,
                     double* yo, cudaStream_t s);

// ---- sharding ----------------------------------------------------------------
// Gather masks of x' (n) and y' (m): bit q = rank q reads the value (zeroed first).
void launch_shard_masks(const int* rp, const int* col, int rows, const int64_t* kc, const int64_t* ktc, int world,
                        unsigned* xmask, unsigned* ymask, cudaStream_t s);
void launch_shard_volume(const unsigned* xmask, const unsigned* ymask, int col0, int col1, int row0, int row1,
                         int world, int rank, unsigned long long* out, cudaStream_t s);

// ---- evaluation ------------------------------------------------------------
// Side stream + events for running EV1 and EV2 concurrently (single device).
struct EvalFork {
  cudaStream_t s2;
  cudaEvent_t e_fork, e_join;
};
void launch_eval(const DevCsr& k, const DevCsr& kt, const DevIter& it, const DevEval& ev,
                 bool seq, cudaStream_t s, const PhaseFn& phase = {}, const EvalFork* fork = nullptr);
int eval_grid0(int n, int m);
int eval_grid(int ntiles);
// Reduced costs of one evaluated point (slot 0..3) into lam[slot] (finish only).
void launch_eval_lambda(const DevCsr& kt, const DevIter& it, const DevEval& ev, bool seq, int slot,
                        cudaStream_t s, const PhaseFn& phase = {});
void launch_reduced_of_objective(const double* c, const double* l, const double* u, int n,
                                 double* lam, cudaStream_t s);

// ---- column panels (panels.cu) ---------------------------------------------
// Device view of one panelized operator (panel-major entries, per-panel row
// counts and block offsets, running row sums between passes).
struct PanelView {
  const int* col;
  const double* val;
  const unsigned char* cnt;  // [panels][rows_pad] entries of each row in each panel
  const int* boff;           // [panels][nblk + 1] first entry of each 1024-row block
  double* acc;               // [rows] running row sums between passes
  int rows, rows_pad, nblk, panels;
  int transposed;            // 1: the operator is K^T (its sweeps stage larger rounds)
};
void launch_panel_keys(const int* row_of, const int* col, int64_t nnz, int width, int rows, int* keys,
                       cudaStream_t s);
void launch_panel_gather(const int* perm, const int* col, const double* val, int64_t nnz, int* col_p,
                         double* val_p, cudaStream_t s);
void launch_panel_spread(const int* rp, const int* col, int rows, int width, unsigned long long* distinct,
                         cudaStream_t s);
void launch_panel_meta(const int* counts, const int* so, int rows, int rows_pad, int panels, int nblk,
                       unsigned char* cnt, int* boff, int* over, cudaStream_t s);
int panel_rows_pad(int rows);
int panel_blocks(int rows);  // 1024-row blocks = CTAs per pass = reduction partials of the last pass
void launch_panel_dual(const PanelView& kp, const DevIter& it, cudaStream_t s);
void launch_panel_primal(const PanelView& ktp, const DevIter& it, int mode_override, cudaStream_t s);
void launch_panel_spmv(const PanelView& pv, const double* v, double* out, cudaStream_t s);
void panel_kernel_attributes();  // dynamic shared memory of the sweep kernels (once per device)

void set_kernel_attributes();

}  // namespace pdlp
