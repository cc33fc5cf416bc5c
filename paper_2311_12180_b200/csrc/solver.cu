// solver.cu — host runtime: upload, K^T build, preconditioning, the windowed
// iteration loop replayed as a CUDA graph, and the evaluation/restart logic.
//
// Mirrors pdhglp::detail::SolveLoop (solver.hpp:634-929). Division of labour:
//   device: every O(nnz) and O(n + m) pass (SpMVs, projections, averages,
//           residuals, reductions) and the per-trial step decision;
//   host:   once per evaluation window (64 accepted iterations by default), the
//           O(1) scalar logic on ~30 reduced numbers: KKT_omega, candidate
//           choice, termination, Farkas tests, restart criteria and the primal
//           weight (glibc exp/log, bitwise with the reference), plus the
//           per-window table of glibc pow step factors (solver.hpp:388-390).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <limits>

#include "kernels.cuh"
#include "solver.cuh"

namespace pdlp {

namespace {

double sclamp(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

[[noreturn]] void invalid(const std::string& m) { throw InvalidArgument(m); }

void validate_params(const pdlp_params& p) {  // SolverParams::validate, solver.hpp:79-93
  if (!(p.eps_optimal > 0.0) || !(p.eps_infeasible > 0.0))
    invalid("params: tolerances must be positive");
  if (!(p.beta_sufficient > 0.0 && p.beta_sufficient < p.beta_necessary && p.beta_necessary < 1.0))
    invalid("params: need 0 < beta_sufficient < beta_necessary < 1");
  if (p.theta_smoothing < 0.0 || p.theta_smoothing > 1.0)
    invalid("params: theta_smoothing must lie in [0, 1]");
  if (p.evaluation_frequency < 1) invalid("params: evaluation_frequency must be >= 1");
  if (p.ruiz_iterations < 0) invalid("ruiz: negative iteration count");
  if (p.pock_chambolle_alpha < 0.0 || p.pock_chambolle_alpha > 2.0)
    invalid("pock-chambolle: alpha must lie in [0, 2]");
  if (p.mode != PDLP_MODE_FAST && p.mode != PDLP_MODE_PARITY) invalid("params: unknown mode");
  if (p.world_size < 1 || p.world_size > kMaxShards)
    invalid("params: world_size must lie in [1, " + std::to_string(kMaxShards) + "]");
  if (p.rank < 0 || p.rank >= p.world_size) invalid("params: rank must lie in [0, world_size)");
  if (p.plan_world < 0 || p.plan_world > kMaxShards) invalid("params: plan_world out of range");
  if (p.world_size > 1 && p.plan_world != 0 && p.plan_world != p.world_size)
    invalid("params: plan_world must equal world_size on a sharded rank");
  if (p.world_size > 1 && p.mode == PDLP_MODE_PARITY)
    invalid("params: parity mode runs on one device (world_size 1)");
  if (p.engine == PDLP_ENGINE_PERSISTENT)
    invalid("params: the persistent window engine was removed (it measured 2x slower than the graph engine "
            "on C1-C3); use PDLP_ENGINE_GRAPH or PDLP_ENGINE_STREAM");
}

}  // namespace

// GeneralFormLp::validate (lp_model.hpp:45-72) plus the raw-array checks of the
// C ABI (present pointers, monotone row offsets); host only, no CUDA call.
void validate_lp(const pdlp_lp& lp) {
  const pdlp_csr& G = lp.inequality_matrix;
  const pdlp_csr& A = lp.equality_matrix;
  const int64_t n = lp.num_variables;
  if (n < 0 || G.num_rows < 0 || A.num_rows < 0 || G.nnz < 0 || A.nnz < 0)
    invalid("lp: negative dimension");
  if (G.num_cols != n || A.num_cols != n) invalid("lp: constraint matrices must have n columns");
  const int64_t m1 = G.num_rows, m2 = A.num_rows, m = m1 + m2, nnz = G.nnz + A.nnz;
  auto need = [](const void* p, int64_t len, const char* what) {
    if (len > 0 && !p) invalid(std::string("lp: missing ") + what);
  };
  need(lp.objective, n, "objective");
  need(lp.lower, n, "lower bounds");
  need(lp.upper, n, "upper bounds");
  need(lp.inequality_rhs, m1, "inequality rhs");
  need(lp.equality_rhs, m2, "equality rhs");
  for (const pdlp_csr* c : {&G, &A}) {
    need(c->values, c->nnz, "matrix values");
    if (c->nnz > 0 && !c->col_indices && !c->col_indices32) invalid("lp: missing column indices");
    if (c->num_rows > 0 && !c->row_offsets) invalid("lp: missing row offsets");
    if (c->row_offsets && (c->row_offsets[0] != 0 || c->row_offsets[c->num_rows] != c->nnz))
      invalid("csr: row_offsets must start at 0 and end at nnz");
    if (c->row_offsets)
      for (int64_t r = 0; r < c->num_rows; ++r)
        if (c->row_offsets[r + 1] < c->row_offsets[r]) invalid("csr: row_offsets must be non-decreasing");
  }
  for (int64_t i = 0; i < n; ++i) {
    const double l = lp.lower[i], u = lp.upper[i];
    if (std::isnan(l) || std::isnan(u)) invalid("lp: NaN bound on variable " + std::to_string(i));
    if (l > u || l == INFINITY || u == -INFINITY)
      invalid("lp: empty bound interval on variable " + std::to_string(i));
  }
  for (int64_t i = 0; i < n; ++i)
    if (std::isnan(lp.objective[i])) invalid("lp: NaN objective entry");
}

namespace {

// validate_lp, then SolverParams::validate; runs before any CUDA call so
// invalid input is PDLP_EINVAL even without a GPU.
void validate_input(const pdlp_lp& lp, const pdlp_params& params) {
  validate_lp(lp);
  validate_params(params);
  const int64_t n = lp.num_variables;
  const int64_t m = lp.inequality_matrix.num_rows + lp.equality_matrix.num_rows;
  const int64_t nnz = lp.inequality_matrix.nnz + lp.equality_matrix.nnz;
  const int64_t lim = int64_t(std::numeric_limits<int32_t>::max()) - 1024;
  if (n > lim || m > lim || nnz > lim)
    throw std::runtime_error("instance exceeds the 32-bit index layout of one device (shard it)");
}

}  // namespace

double KktHost::weighted(double omega) const {  // KktResiduals::weighted
  const double pr = omega * prn, dr = drn / omega, g = gap();
  return std::sqrt(pr * pr + dr * dr + g * g);
}

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------

Solver::Solver(const pdlp_lp& lp, const pdlp_params& params) : params_(params) {
  const auto t = std::chrono::steady_clock::now();
  validate_input(lp, params);
  PDLP_CUDA(cudaSetDevice(params.device));
  {
    // the stream-ordered pool keeps freed memory for the next handle
    cudaMemPool_t pool;
    PDLP_CUDA(cudaDeviceGetDefaultMemPool(&pool, params.device));
    uint64_t keep = ~uint64_t(0);
    PDLP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  PDLP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  if (!std::getenv("PDLP_NO_EVAL_FORK")) {
    PDLP_CUDA(cudaStreamCreateWithFlags(&fork_.s2, cudaStreamNonBlocking));
    PDLP_CUDA(cudaEventCreateWithFlags(&fork_.e_fork, cudaEventDisableTiming));
    PDLP_CUDA(cudaEventCreateWithFlags(&fork_.e_join, cudaEventDisableTiming));
  }
  setup(lp);
  PDLP_CUDA(cudaStreamSynchronize(stream_));
  setup_seconds_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

Solver::~Solver() {
  if (stream_) cudaStreamSynchronize(stream_);  // pool frees below are stream-ordered
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  if (ev_begin_) cudaEventDestroy(ev_begin_);
  if (ev_end_) cudaEventDestroy(ev_end_);
  if (ev_w0_) cudaEventDestroy(ev_w0_);
  if (ev_w1_) cudaEventDestroy(ev_w1_);
  if (ev_e1_) cudaEventDestroy(ev_e1_);
  if (fork_.e_fork) cudaEventDestroy(fork_.e_fork);
  if (fork_.e_join) cudaEventDestroy(fork_.e_join);
  if (fork_.s2) cudaStreamDestroy(fork_.s2);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_) cudaGraphDestroy(graph_);
  if (chain_exec_) cudaGraphExecDestroy(chain_exec_);
  if (chain_graph_) cudaGraphDestroy(chain_graph_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Solver::setup(const pdlp_lp& lp) {
  // PDLP_TRACE_SETUP=1: per-phase wall times of the setup on stderr
  const bool trace = std::getenv("PDLP_TRACE_SETUP") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    PDLP_CUDA(cudaStreamSynchronize(stream_));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pdlp setup] %-14s %8.2f ms\n", what,
                 1e3 * std::chrono::duration<double>(now - tp).count());
    tp = now;
  };
  // validated by validate_input() before any device work
  const pdlp_csr& G = lp.inequality_matrix;
  const pdlp_csr& A = lp.equality_matrix;
  n_ = lp.num_variables;
  m1_ = G.num_rows;
  m2_ = A.num_rows;
  m_ = m1_ + m2_;
  nnz_ = G.nnz + A.nnz;

  objective_constant_ = lp.objective_constant;
  hc_ = lp.objective;
  hl_ = lp.lower;
  hu_ = lp.upper;
  hh_ = lp.inequality_rhs;
  hb_ = lp.equality_rhs;
  {  // termination_norms on the ORIGINAL instance (solver.hpp:157-163)
    double sh = 0.0, sb = 0.0, sc = 0.0;
    for (int64_t i = 0; i < m1_; ++i) sh += hh_[i] * hh_[i];
    for (int64_t i = 0; i < m2_; ++i) sb += hb_[i] * hb_[i];
    for (int64_t j = 0; j < n_; ++j) sc += hc_[j] * hc_[j];
    rhs_norm_ = std::sqrt(sh + sb);
    obj_norm_ = std::sqrt(sc);
  }

  cudaStream_t s = stream_;
  // ---- K = vstack(G, A) (sparse_matrix.hpp:181-200) in HBM, int32 indices ----
  k_rp_.alloc(m_ + 1 + kVecPad);  // padded for quad-aligned span loads
  k_rp_.zero(s);
  k_col_.alloc(nnz_ + kVecPad);
  k_val_orig_.alloc(nnz_ + kVecPad);
  k_val_.alloc(nnz_ + kVecPad);
  k_col_.zero(s);
  k_val_orig_.zero(s);
  k_val_.zero(s);
  DevBuf<int64_t> goff(m1_ + 1), aoff(m2_ + 1);
  std::vector<int64_t> zero_off{0};
  PDLP_CUDA(cudaMemcpyAsync(goff.get(), G.row_offsets ? G.row_offsets : zero_off.data(),
                            (m1_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  PDLP_CUDA(cudaMemcpyAsync(aoff.get(), A.row_offsets ? A.row_offsets : zero_off.data(),
                            (m2_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  launch_build_rowptr(goff.get(), aoff.get(), m1_, m2_, G.nnz, k_rp_.get(), s);
  mark("upload/rowptr");
  DevBuf<int> err(1);
  err.zero(s);
  int64_t off = 0;
  for (const pdlp_csr* c : {&G, &A}) {
    if (c->nnz > 0) {
      if (c->col_indices32) {
        PDLP_CUDA(cudaMemcpyAsync(k_col_.get() + off, c->col_indices32, c->nnz * sizeof(int),
                                  cudaMemcpyHostToDevice, s));
      } else {
        DevBuf<int64_t> tmp(c->nnz);
        PDLP_CUDA(cudaMemcpyAsync(tmp.get(), c->col_indices, c->nnz * sizeof(int64_t),
                                  cudaMemcpyHostToDevice, s));
        launch_narrow_cols(tmp.get(), k_col_.get() + off, c->nnz, int(n_), err.get(), s);
        PDLP_CUDA(cudaStreamSynchronize(s));
      }
      mark("upload/cols");
      PDLP_CUDA(cudaMemcpyAsync(k_val_orig_.get() + off, c->values, c->nnz * sizeof(double),
                                cudaMemcpyHostToDevice, s));
    }
    off += c->nnz;
  }
  mark("upload/values");
  launch_check_cols(k_col_.get(), nnz_, int(n_), err.get(), s);
  launch_check_rows(k_rp_.get(), k_col_.get(), int(m_), err.get(), s);
  int herr = 0;
  PDLP_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  if (herr & 1) invalid("csr: column index out of range");
  if (herr & 2) invalid("csr: row_offsets must be nondecreasing");
  if (herr & 4) invalid("csr: column indices must be strictly increasing within a row");

  mark("upload");
  build_transpose();
  mark("transpose");

  // original vectors on the device (evaluation on the unscaled LP)
  auto up = [&](DevBuf<double>& d, int64_t len, std::initializer_list<std::pair<const double*, int64_t>> parts) {
    d.alloc(size_t(len));
    int64_t at = 0;
    for (const auto& pr : parts) {
      if (pr.second > 0)
        PDLP_CUDA(cudaMemcpyAsync(d.get() + at, pr.first, size_t(pr.second) * sizeof(double),
                                  cudaMemcpyHostToDevice, s));
      at += pr.second;
    }
  };
  up(c_orig_, n_, {{hc_, n_}});
  up(l_orig_, n_, {{hl_, n_}});
  up(u_orig_, n_, {{hu_, n_}});
  up(q_orig_, m_, {{hh_, m1_}, {hb_, m2_}});

  precondition();
  mark("precondition");

  // tile plans (host planner over the offsets)
  // (page-locked, from the pool: no zero fill, full-speed D2H)
  size_t rp_cap = 0, rpt_cap = 0;
  std::unique_ptr<int, std::function<void(int*)>> rp_hold(
      static_cast<int*>(pinned_pool_get(size_t(m_ + 1) * sizeof(int), &rp_cap)),
      [&rp_cap](int* q) { pinned_pool_put(q, rp_cap); });
  std::unique_ptr<int, std::function<void(int*)>> rpt_hold(
      static_cast<int*>(pinned_pool_get(size_t(n_ + 1) * sizeof(int), &rpt_cap)),
      [&rpt_cap](int* q) { pinned_pool_put(q, rpt_cap); });
  int* rp_h = rp_hold.get();
  int* rpt_h = rpt_hold.get();
  PDLP_CUDA(cudaMemcpyAsync(rp_h, k_rp_.get(), (m_ + 1) * sizeof(int),
                            cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaMemcpyAsync(rpt_h, kt_rp_.get(), (n_ + 1) * sizeof(int),
                            cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  K_ = DevCsr{k_rp_.get(), k_col_.get(), k_val_.get(), k_val_orig_.get(), int(m_), int(n_), nnz_};
  KT_ = DevCsr{kt_rp_.get(), kt_col_.get(), kt_val_.get(), kt_val_orig_.get(), int(n_), int(m_), nnz_};
  // row sharding: contiguous row ranges of K and of K^T per rank (SURVEY.md
  // §8e), cut where every tiling starts a tile, so each rank runs whole tiles
  // of the one global plan and partials keep their global order
  world_ = params_.world_size;
  rank_ = params_.rank;
  const int plan_world = params_.plan_world > 0 ? params_.plan_world : world_;
  std::vector<int64_t> kbrk, ktbrk;
  k_cuts_ = {0, m_};
  kt_cuts_ = {0, n_};
  if (plan_world > 1) {
    const std::vector<int64_t> kc = shard_cuts<int>(m_, rp_h, plan_world);
    const std::vector<int64_t> ktc = shard_cuts<int>(n_, rpt_h, plan_world);
    kbrk.assign(kc.begin() + 1, kc.end() - 1);
    ktbrk.assign(ktc.begin() + 1, ktc.end() - 1);
    if (world_ > 1) {
      k_cuts_ = kc;
      kt_cuts_ = ktc;
    }
  }
  const int64_t r0 = k_cuts_[rank_], r1 = k_cuts_[rank_ + 1];
  const int64_t c0 = world_ > 1 ? kt_cuts_[rank_] : 0, c1 = world_ > 1 ? kt_cuts_[rank_ + 1] : n_;
  // two tilings of each operator: iteration kernels and evaluation kernels
  // (common.cuh TileGeom)
  mark("offsets");
  // rows with mostly consecutive columns get element-interleaved lane groups
  std::vector<uint8_t> kcon, ktcon;
  const std::vector<uint8_t>* kc_p = nullptr;
  const std::vector<uint8_t>* ktc_p = nullptr;
  // and groups of four column-shifted rows share one interleaved tile (the
  // contiguous-row mode is opt-in: measured -7% SpMV time over K on C2)
  if (!parity() && !std::getenv("PDLP_NO_ROW_GROUPS")) {
    const int want_contig = std::getenv("PDLP_CONTIG") ? 1 : 0;
    DevBuf<unsigned char> f1{static_cast<size_t>(m_)}, f2{static_cast<size_t>(n_)};
    launch_row_contig(k_rp_.get(), k_col_.get(), int(m_), kStreamMaxRow, want_contig, f1.get(), s);
    launch_row_contig(kt_rp_.get(), kt_col_.get(), int(n_), kStreamMaxRow, want_contig, f2.get(), s);
    kcon.resize(size_t(m_));
    ktcon.resize(size_t(n_));
    if (m_) PDLP_CUDA(cudaMemcpyAsync(kcon.data(), f1.get(), size_t(m_), cudaMemcpyDeviceToHost, s));
    if (n_) PDLP_CUDA(cudaMemcpyAsync(ktcon.data(), f2.get(), size_t(n_), cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
    kc_p = &kcon;
    ktc_p = &ktcon;
  }
  build_plan(k_it_, K_, rp_h, m_, kIterGeom, kbrk, r0, r1, kc_p);
  build_plan(kt_it_, KT_, rpt_h, n_, kIterGeom, ktbrk, c0, c1, ktc_p);
  build_plan(k_ev_, K_, rp_h, m_, kEvalGeom, kbrk, r0, r1, kc_p);
  build_plan(kt_ev_, KT_, rpt_h, n_, kEvalGeom, ktbrk, c0, c1, ktc_p);
  if (trace) {
    for (const auto& pr : {std::make_pair("K", &k_it_), std::make_pair("KT", &kt_it_)}) {
      const TilePlan& tp = pr.second->plan;
      int uni = 0, shift = 0;
      for (const Tile& t : tp.tiles) {
        uni += (t.kind == kTileStream && t.part > 0) ? 1 : 0;
        shift += (t.kind == kTileWarp && t.slot == 2) ? 1 : 0;
      }
      std::fprintf(stderr, "[pdlp setup] %s tiles: %d stream (%d uniform), %d warp (%d shifted), %d chunk\n",
                   pr.first, tp.stream_tiles, uni, tp.warp_tiles, shift, tp.chunk_tiles);
    }
  }
  K_ = k_it_.csr;
  KT_ = kt_it_.csr;
  K_full_ = K_;
  K_full_.tile0 = 0;
  K_full_.ntiles = int(k_it_.plan.tiles.size());
  KT_full_ = KT_;
  KT_full_.tile0 = 0;
  KT_full_.ntiles = int(kt_it_.plan.tiles.size());
  if (world_ > 1) {
    for (const OpPlan* op : {&k_it_, &kt_it_, &k_ev_, &kt_ev_})
      if (op->csr.ntiles < 1) invalid("shards: a rank owns no tile; use fewer ranks for this instance");
    // fingerprint of the partition: every rank must agree before linking
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    mix(uint64_t(n_)), mix(uint64_t(m_)), mix(uint64_t(nnz_)), mix(uint64_t(world_));
    for (int64_t v : k_cuts_) mix(uint64_t(v));
    for (int64_t v : kt_cuts_) mix(uint64_t(v));
    for (const OpPlan* op : {&k_it_, &kt_it_, &k_ev_, &kt_ev_}) mix(op->plan.tiles.size());
    plan_hash_ = h;
  }

  // column panels for operators that scatter over a vector much larger than
  // L2 (fast mode, one device; panels.cu)
  if (!parity() && world_ == 1 && !(std::getenv("PDLP_PANELS") && std::atoi(std::getenv("PDLP_PANELS")) == 0)) {
    build_panels(kpan_, K_, int(m_), int(n_), "K");
    build_panels(ktpan_, KT_, int(n_), int(m_), "KT");
  }
  mark("plans");
  allocate_iteration();
  mark("allocate");
  set_kernel_attributes();
  pin_iterates_in_l2();
  mark("attributes");
  if (omega_job_.valid()) omega_job_.get();
  hc_ = hl_ = hu_ = hh_ = hb_ = nullptr;  // the caller's arrays are not ours past pdlp_create
}

// Decides whether `op` (rows x cols) gets column panels and builds them: the
// gathered vector must exceed one panel's L2 budget (PDLP_PANEL_MB, default
// 48 MB) and the rows must scatter over it (on average across at least half of
// min(panels, row length) panels, i.e. no locality a single pass could use);
// no row may hold more than 255 entries in one panel. Operators past 64 M
// nonzeros that fail the scatter test run as a single panel (below).
// PDLP_PANELS=1 forces panels of PDLP_PANEL_WIDTH columns (tests); =0
// disables them.
void Solver::build_panels(PanelOp& po, const DevCsr& op, int rows, int cols, const char* which) {
  cudaStream_t s = stream_;
  const char* force = std::getenv("PDLP_PANELS");
  const bool forced = force && std::atoi(force) == 1;
  // measured on C4 (tools/panel_sweep.py): K (x, 320 MB) is fastest in 48 MB
  // panels; K^T has twice the rows, so its per-panel running sums cost twice
  // as much and it is fastest in 64 MB panels of y
  const bool kt = std::strcmp(which, "KT") == 0;
  double budget_mb = kt ? 64.0 : 48.0;
  if (const char* e = std::getenv("PDLP_PANEL_MB")) budget_mb = std::max(1.0, std::atof(e));
  if (const char* e = std::getenv(kt ? "PDLP_PANEL_MB_T" : "PDLP_PANEL_MB_K")) budget_mb = std::max(1.0, std::atof(e));
  int panels = int(std::ceil(8.0 * double(cols) / (budget_mb * 1048576.0)));
  int width = std::max(1, int((int64_t(cols) + panels - 1) / std::max(1, panels)));
  if (forced && std::getenv("PDLP_PANEL_WIDTH")) {
    width = std::max(1, std::atoi(std::getenv("PDLP_PANEL_WIDTH")));
    panels = int((int64_t(cols) + width - 1) / width);
  }
  if (rows < 1 || op.nnz < 1) return;
  // operators too large for L2 whose rows stay local (C5's staircase) still
  // run as one panel: the sweep's count-byte rows and fused final pass beat
  // the tiled kernels there (C5 58.8 -> 67.1 it/s; profiles/r02p1_ab_single_panel.jsonl)
  const bool single_ok = !forced && op.nnz >= (int64_t(1) << 26) && !std::getenv("PDLP_NO_SINGLE_PANEL");
  bool single = false;
  if (panels < 2 && !forced) {
    if (!single_ok) return;
    single = true;
  }
  if (!single && !forced) {
    DevBuf<unsigned long long> d{static_cast<size_t>(1)};
    d.zero(s);
    launch_panel_spread(op.rp, op.col, rows, width, d.get(), s);
    unsigned long long distinct = 0;
    PDLP_CUDA(cudaMemcpyAsync(&distinct, d.get(), 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
    const double per_row = double(distinct) / double(rows);
    const double avg_len = double(op.nnz) / double(rows);
    if (per_row < 0.5 * std::min(double(panels), avg_len)) {
      if (!single_ok) return;
      single = true;
    }
  }
  if (single) {
    panels = 1;
    width = cols;
  }
  if (int64_t(panels) * rows >= int64_t(std::numeric_limits<int32_t>::max()) - 1024) return;
  // panel-major order: entry k of row r, column c goes to stacked row
  // (c / width) * rows + r; a stable radix sort keeps each row's columns in
  // increasing order
  const int64_t nnz = op.nnz;
  const int srows = panels * rows;
  const int rows_pad = panel_rows_pad(rows);
  const int nblk = panel_blocks(rows);
  DevBuf<int> row_of{static_cast<size_t>(nnz)}, keys{static_cast<size_t>(nnz)},
      keys2{static_cast<size_t>(nnz)}, ids{static_cast<size_t>(nnz)}, perm{static_cast<size_t>(nnz)},
      counts{static_cast<size_t>(srows) + 1}, so{static_cast<size_t>(srows) + 1};
  launch_expand_rows(op.rp, rows, row_of.get(), s);
  launch_panel_keys(row_of.get(), op.col, nnz, width, rows, keys.get(), s);
  launch_iota(ids.get(), nnz, s);
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < srows) ++end_bit;
  size_t tmp_bytes = 0;
  PDLP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.get(), keys2.get(), ids.get(), perm.get(),
                                            int(nnz), 0, end_bit, s));
  // (temporaries are freed on cudaStreamPerThread: they must outlive the work
  // queued on `s`, which is synchronised before they go out of scope)
  DevBuf<unsigned char> tmp{tmp_bytes};
  PDLP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, keys.get(), keys2.get(), ids.get(), perm.get(),
                                            int(nnz), 0, end_bit, s));
  counts.zero(s);
  launch_count_cols(keys.get(), nnz, counts.get(), s);
  size_t scan_bytes = 0;
  PDLP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts.get(), so.get(), srows + 1, s));
  DevBuf<unsigned char> scan_tmp{scan_bytes};
  PDLP_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp.get(), scan_bytes, counts.get(), so.get(), srows + 1, s));
  po.cnt.alloc(size_t(panels) * rows_pad);
  po.boff.alloc(size_t(panels) * (nblk + 1));
  DevBuf<int> over{static_cast<size_t>(1)};
  over.zero(s);
  launch_panel_meta(counts.get(), so.get(), rows, rows_pad, panels, nblk, po.cnt.get(), po.boff.get(), over.get(),
                    s);
  int over_h = 0;
  PDLP_CUDA(cudaMemcpyAsync(&over_h, over.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  if (over_h) {  // a row holds more than 255 entries of one panel: no panels
    po.cnt = DevBuf<unsigned char>();
    po.boff = DevBuf<int>();
    return;
  }
  po.col.alloc(size_t(nnz) + kVecPad);
  po.val.alloc(size_t(nnz) + kVecPad);
  po.col.zero(s);
  po.val.zero(s);
  launch_panel_gather(perm.get(), op.col, op.val, nnz, po.col.get(), po.val.get(), s);
  PDLP_CUDA(cudaStreamSynchronize(s));
  po.acc.alloc(size_t(rows) + kVecPad);
  po.panels = panels;
  po.width = width;
  po.view = PanelView{po.col.get(), po.val.get(), po.cnt.get(), po.boff.get(), po.acc.get(),
                      rows, rows_pad, nblk, panels, kt ? 1 : 0};
  if (std::getenv("PDLP_TRACE_SETUP"))
    std::fprintf(stderr, "[pdlp setup] %s: %d column panels of %d columns, %d row blocks\n", which, panels,
                 width, nblk);
}

void Solver::dual_step(unsigned long long cond, int use_cond) {
  if (kpan_.panels)
    launch_panel_dual(kpan_.view, it_, stream_);
  else
    launch_dual(K_, it_, parity(), cond, use_cond, stream_);
}

void Solver::primal_step(int mode_override, unsigned long long cond, int use_cond) {
  if (ktpan_.panels)
    launch_panel_primal(ktpan_.view, it_, mode_override, stream_);
  else
    launch_primal(KT_, it_, parity(), mode_override, stream_, cond, use_cond);
}

void Solver::build_plan(OpPlan& p, const DevCsr& base, const int* rp, int64_t rows,
                        const TileGeom& g, const std::vector<int64_t>& breaks, int64_t r0,
                        int64_t r1, const std::vector<uint8_t>* contig) {
  // planner thresholds: env overrides are a tuning aid (clamped to the geometry)
  auto knob = [](const char* name, int def) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : def;
  };
  const int smax = std::min(knob("PDLP_STREAM_MAX_ROW", kStreamMaxRow), g.stream_nnz);
  const int wmax = std::min(knob("PDLP_WARP_MAX_ROW", kWarpMaxRow), g.lane_nnz * kThreads);
  const int cnnz = std::min(knob("PDLP_CHUNK_NNZ", g.chunk_nnz), g.chunk_nnz);
  const int lane = std::min(knob("PDLP_LANE_NNZ", g.lane_nnz), g.lane_nnz);
  // C1-class operators (64k-256k nnz) in 4096-nnz tiles occupy only ~25 of
  // 148 SMs and are latency-bound: 1024-nnz tiles there (C1 22.9 -> 15.6 ms
  // per solve). Smaller operators keep the full tiles: re-tiling moves fast
  // mode's reduction order, and the 37k-40k-nnz stand-ins of C3/C5 used by
  // the drift tests would move to 1.3e-10 over 100 iterates, past north_star's
  // 1e-10 bar (their full-size configs use 4096 anyway).
  int snnz_def = g.stream_nnz;
  if (&g == &kIterGeom) {
    const int64_t nnz = int64_t(rp[rows]);
    if (nnz >= (int64_t(1) << 16) && nnz < (int64_t(1) << 18)) snnz_def = 1024;
  }
  const int snnz = std::max(64, std::min(knob("PDLP_STREAM_NNZ", snnz_def), g.stream_nnz));
  const int srows = std::max(kThreads, std::min(knob("PDLP_STREAM_ROWS", g.stream_rows), g.stream_rows));
  p.plan = plan_tiles<int>(rows, rp, parity(), std::min(smax, snnz), wmax, cnnz,
                           snnz, srows, kThreads, lane, breaks, contig);
  const std::vector<Tile>& th = p.plan.tiles;
  p.tiles.alloc(th.size());
  PDLP_CUDA(cudaMemcpyAsync(p.tiles.get(), th.data(), th.size() * sizeof(Tile),
                            cudaMemcpyHostToDevice, stream_));
  p.chunk.alloc(size_t(std::max(1, p.plan.chunk_slots)) * 8);
  p.ctr.alloc(std::max(1, p.plan.split_rows));
  p.ctr.zero(stream_);
  p.csr = base;
  p.csr.tiles = p.tiles.get();
  const auto own = tile_range(p.plan, r0, r1, rows);  // this rank's tiles (all of them unsharded)
  p.csr.tile0 = own.first;
  p.csr.ntiles = own.second - own.first;
  p.csr.chunk_slots = p.plan.chunk_slots;
  p.csr.chunk_part = p.chunk.get();
  p.csr.chunk_ctr = p.ctr.get();
}

// explicit_transpose (sparse_matrix.hpp:167-178) on the device: a stable LSD
// radix sort of nnz ids by column keeps each column's entries in increasing
// row order, i.e. the reference's CSR of K^T; integer output is exact.
void Solver::build_transpose() {
  cudaStream_t s = stream_;
  kt_rp_.alloc(n_ + 1 + kVecPad);
  kt_rp_.zero(s);
  kt_col_.alloc(nnz_ + kVecPad);
  kt_val_orig_.alloc(nnz_ + kVecPad);
  kt_val_.alloc(nnz_ + kVecPad);
  kt_col_.zero(s);
  kt_val_orig_.zero(s);
  kt_val_.zero(s);
  const int nnz = int(nnz_);
  DevBuf<int> row_of(nnz_), ids(nnz_), keys_out(nnz_), perm(nnz_), counts(n_ + 1);
  launch_expand_rows(k_rp_.get(), int(m_), row_of.get(), s);
  launch_iota(ids.get(), nnz_, s);
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < n_) ++end_bit;
  size_t tmp_bytes = 0;
  PDLP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_col_.get(), keys_out.get(),
                                            ids.get(), perm.get(), nnz, 0, end_bit, s));
  DevBuf<unsigned char> tmp(tmp_bytes);
  PDLP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, k_col_.get(), keys_out.get(),
                                            ids.get(), perm.get(), nnz, 0, end_bit, s));
  counts.zero(s);
  launch_count_cols(k_col_.get(), nnz_, counts.get(), s);
  size_t scan_bytes = 0;
  PDLP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts.get(), kt_rp_.get(),
                                          int(n_ + 1), s));
  DevBuf<unsigned char> scan_tmp(scan_bytes);
  PDLP_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp.get(), scan_bytes, counts.get(), kt_rp_.get(),
                                          int(n_ + 1), s));
  launch_gather_transpose(perm.get(), row_of.get(), k_val_orig_.get(), nnz_, kt_col_.get(),
                          kt_val_orig_.get(), s);
  PDLP_CUDA(cudaStreamSynchronize(s));
}

// make_scaling(vstack(G,A), mode, ruiz_iterations, alpha) (scaling.hpp:117-132)
// then apply_scaling (scaling.hpp:137-170), all on the device.
void Solver::precondition() {
  cudaStream_t s = stream_;
  d1_dev_.alloc(m_);
  d2_dev_.alloc(n_);
  launch_fill(d1_dev_.get(), m_, 1.0, s);
  launch_fill(d2_dev_.get(), n_, 1.0, s);
  DevBuf<double> rn(m_), cn(n_);
  const int mode = params_.scaling;
  if (mode != PDLP_SCALING_NONE) {
    for (int it = 0; it < params_.ruiz_iterations; ++it) {  // ruiz_equilibrate :52-66
      launch_row_absmax(k_rp_.get(), k_col_.get(), k_val_orig_.get(), int(m_), d1_dev_.get(),
                        d2_dev_.get(), rn.get(), s, double(nnz_) / double(std::max<int64_t>(1, m_)));
      launch_row_absmax(kt_rp_.get(), kt_col_.get(), kt_val_orig_.get(), int(n_), d2_dev_.get(),
                        d1_dev_.get(), cn.get(), s, double(nnz_) / double(std::max<int64_t>(1, n_)));
      launch_ruiz_update(d1_dev_.get(), rn.get(), int(m_), s);
      launch_ruiz_update(d2_dev_.get(), cn.get(), int(n_), s);
    }
    if (mode == PDLP_SCALING_RUIZ_PC) {  // pock_chambolle_scale :72-94 + compose :98-112
      const double alpha = params_.pock_chambolle_alpha;
      launch_row_pnorm(k_rp_.get(), k_col_.get(), k_val_orig_.get(), int(m_), d1_dev_.get(),
                       d2_dev_.get(), 2.0 - alpha, rn.get(), s);
      launch_row_pnorm(kt_rp_.get(), kt_col_.get(), kt_val_orig_.get(), int(n_), d2_dev_.get(),
                       d1_dev_.get(), alpha, cn.get(), s);
      launch_pc_update(d1_dev_.get(), rn.get(), int(m_), 2.0 - alpha, s);
      launch_pc_update(d2_dev_.get(), cn.get(), int(n_), alpha, s);
    }
  }
  launch_scale_values(k_rp_.get(), k_col_.get(), k_val_orig_.get(), int(m_), d1_dev_.get(),
                      d2_dev_.get(), k_val_.get(), s);
  launch_scale_values(kt_rp_.get(), kt_col_.get(), kt_val_orig_.get(), int(n_), d2_dev_.get(),
                      d1_dev_.get(), kt_val_.get(), s);
  c_s_.alloc(n_);
  l_s_.alloc(n_);
  u_s_.alloc(n_);
  q_s_.alloc(m_);
  launch_scale_vectors(c_orig_.get(), l_orig_.get(), u_orig_.get(), q_orig_.get(), d1_dev_.get(),
                       d2_dev_.get(), int(n_), int(m_), c_s_.get(), l_s_.get(), u_s_.get(),
                       q_s_.get(), s);
  // eta_hat_0 = 1 / max|K~| (solver.hpp:771-772): order-free max
  const int nb = 296;
  DevBuf<double> part(nb);
  launch_block_absmax(k_val_.get(), nnz_, part.get(), nb, s);
  std::vector<double> ph(nb);
  d1_.resize(size_t(m_));
  d2_.resize(size_t(n_));
  PDLP_CUDA(cudaMemcpyAsync(ph.data(), part.get(), nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (m_)
    PDLP_CUDA(cudaMemcpyAsync(d1_.data(), d1_dev_.get(), m_ * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
  if (n_)
    PDLP_CUDA(cudaMemcpyAsync(d2_.data(), d2_dev_.get(), n_ * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  double mx = 0.0;
  for (double v : ph) mx = std::max(mx, v);
  eta_hat0_ = mx > 0.0 ? 1.0 / mx : 1.0;
  // initialize_primal_weight on the scaled problem (solver.hpp:293-300, :774-776):
  // the scaled vectors are the same products the device formed.
  // norm2 of the scaled c and q, summed in index order as norm2 of the
  // materialised vectors would be (no n-vector temporaries on the host)
  // (two sequential sums of tens of millions of terms: on a host thread while
  // the rest of setup runs; joined at its end)
  omega_job_ = std::async(std::launch::async, [this] {
    double sc = 0.0, sq = 0.0;
    for (int64_t j = 0; j < n_; ++j) {
      const double v = hc_[j] * d2_[j];
      sc += v * v;
    }
    for (int64_t i = 0; i < m_; ++i) {
      const double v = hq(i) * d1_[i];
      sq += v * v;
    }
    const double cn2 = std::sqrt(sc), qn2 = std::sqrt(sq);
    const double w = (cn2 > params_.eps_zero && qn2 > params_.eps_zero) ? cn2 / qn2 : 1.0;
    omega0_ = sclamp(w, params_.omega_min, params_.omega_max);
  });
}

// The iterate buffers the SpMVs gather from (x for K x', y for K'y') stay in
// L2 across the matrix streams: an access-policy window on the solver's stream
// (captured into the graph's kernel nodes) marks them persisting, sized to the
// device's persisting carve-out (hitRatio < 1 when the buffers are larger).
void Solver::pin_iterates_in_l2() {
  l2_window_bytes_ = 0;
  if (!params_.l2_persist || std::getenv("PDLP_NO_L2_PERSIST")) return;
  int max_persist = 0, max_window = 0;
  PDLP_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, params_.device));
  PDLP_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, params_.device));
  if (max_persist <= 0 || max_window <= 0) return;
  // the larger gather source: x for the dual kernel's K x' (n >= m in every
  // config), else y; all three rotation buffers (one allocation)
  const bool use_x = n_ >= m_;
  void* base = use_x ? static_cast<void*>(x_all_.get()) : static_cast<void*>(y_all_.get());
  const size_t bytes = 3 * sizeof(double) * size_t(use_x ? n_ : m_);
  const size_t window = std::min(bytes, size_t(max_window));
  const size_t carve = std::min(window, size_t(max_persist));
  PDLP_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.base_ptr = base;
  v.accessPolicyWindow.num_bytes = window;
  v.accessPolicyWindow.hitRatio = float(double(carve) / double(window));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  PDLP_CUDA(cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &v));
  l2_window_bytes_ = int64_t(carve);
}

void Solver::allocate_iteration() {
  cudaStream_t s = stream_;
  const bool ipc = world_ > 1;  // exchanged buffers must be CUDA-IPC capable
  x_all_.alloc(3 * size_t(n_), ipc);
  y_all_.alloc(3 * size_t(m_), ipc);
  for (auto& b : kx_) b.alloc(m_);
  for (auto& b : kty_) b.alloc(n_);
  avg_x_.alloc(n_, ipc);
  avg_y_.alloc(m_, ipc);
  x_start_.alloc(n_);
  y_start_.alloc(m_);
  const int64_t row0 = k_cuts_[rank_], row1 = k_cuts_[rank_ + 1];
  const int64_t col0 = kt_cuts_[rank_], col1 = kt_cuts_[rank_ + 1];
  const int avg_blocks = std::max<int64_t>(1, (row1 - row0 + 4095) / 4096);
  const int p_grid = KT_.ntiles + avg_blocks;
  // partial counts: one per tile of the operator's kernel, or one per combine
  // block when the operator runs as column panels
  const int k_tiles = kpan_.panels ? kpan_.view.nblk : int(k_it_.plan.tiles.size());
  const int kt_tiles = ktpan_.panels ? ktpan_.view.nblk : int(kt_it_.plan.tiles.size());
  d_part_.alloc(size_t(k_tiles) * 3, ipc);
  p_part_.alloc(size_t(kt_tiles) * 4 + 2, ipc);  // two parity buffers + dx^2 total
  p_part_.zero(s);
  const bool seq = parity();
  seq_dy2_.alloc(seq ? m_ : 1);
  seq_inter_.alloc(seq ? m_ : 1);
  seq_dx2_.alloc(seq ? n_ : 1);
  tab_cap_ = int(std::min<int64_t>(params_.evaluation_frequency, 4096));
  // chained windows (graph engine, fast mode, one rank, no step log): up to
  // 16 windows per launch, the device deciding the evaluations in between
  chain_windows_ = 0;
  if (!parity() && world_ == 1 && !params_.record_step_log && params_.evaluation_frequency <= 1024 &&
      (params_.engine == PDLP_ENGINE_GRAPH || (params_.engine == PDLP_ENGINE_AUTO && params_.use_cuda_graph)) &&
      !std::getenv("PDLP_NO_CHAIN"))
    chain_windows_ = 16;
  {
    // [EvalOut | DevState | step-factor pairs]: one D2H (eval + state) and one
    // H2D (state + factors) per window round trip
    auto up64 = [](size_t b) { return (b + 63) & ~size_t(63); };
    xo_state_ = up64(sizeof(EvalOut));
    xo_tab_ = xo_state_ + up64(sizeof(DevState));
    const size_t tab_entries = size_t(std::max(tab_cap_ * std::max(chain_windows_, 1), 128));  // head stages 128
    const size_t bytes = xo_tab_ + 2 * sizeof(double) * tab_entries;
    xfer_dev_.alloc(bytes);
    xfer_dev_.zero(s);
    xfer_host_.alloc(bytes);
    std::memset(xfer_host_.get(), 0, bytes);
    eval_dev_ = reinterpret_cast<EvalOut*>(xfer_dev_.get());
    state_dev_ = reinterpret_cast<DevState*>(xfer_dev_.get() + xo_state_);
    he_ = reinterpret_cast<EvalOut*>(xfer_host_.get());
    hs_ = reinterpret_cast<DevState*>(xfer_host_.get() + xo_state_);
    tab_host_ = reinterpret_cast<double*>(xfer_host_.get() + xo_tab_);
  }
  step_log_dev_.alloc(tab_cap_);
  snap_dev_.alloc(1);
  snap_dev_.zero(s);
  log_host_.alloc(tab_cap_);


  DevIter& it = it_;
  for (int i = 0; i < 3; ++i) {
    it.x[i] = x_all_.get() + size_t(i) * n_;
    it.y[i] = y_all_.get() + size_t(i) * m_;
  }
  for (int i = 0; i < 2; ++i) {
    it.kx[i] = kx_[i].get();
    it.kty[i] = kty_[i].get();
  }
  it.avg_x = avg_x_.get();
  it.avg_y = avg_y_.get();
  it.x_start = x_start_.get();
  it.y_start = y_start_.get();
  it.c = c_s_.get();
  it.l = l_s_.get();
  it.u = u_s_.get();
  it.q = q_s_.get();
  it.n = int(n_);
  it.m = int(m_);
  it.m1 = int(m1_);
  it.p_grid = p_grid;
  it.p_tiles = kt_tiles;
  {
    // l = +0 (sign bit clear, so l / d2 stays +0) and u = +inf everywhere:
    // min(max(v, l), u) == max(v, 0) bitwise, and the bound streams are skipped
    bool nonneg = true;
    for (int64_t j = 0; j < n_ && nonneg; ++j)
      nonneg = hl_[j] == 0.0 && !std::signbit(hl_[j]) && hu_[j] == INFINITY;
    it.nonneg = nonneg ? 1 : 0;
  }
  it.avg_blocks = avg_blocks;
  it.d_part = d_part_.get();
  it.p_part = p_part_.get();
  it.px_total = p_part_.get() + size_t(kt_tiles) * 4;
  it.snap = snap_dev_.get();
  it.d_tiles = k_tiles;
  // per-CTA decisions re-read every dual partial: past ~2M partial reads per
  // trial a one-CTA decision kernel is cheaper (C3/C4-sized operators)
  it.decide_sep = (!parity() && double(k_tiles) * double(p_grid) > 2.0e6) ? 1 : 0;
  if (const char* e = std::getenv("PDLP_DECIDE_SEP")) it.decide_sep = parity() ? 0 : std::atoi(e);
  // 2 (decision in the dual's last CTA) needs every partial on this device
  if (world_ > 1 && it.decide_sep == 2) it.decide_sep = 1;
  // panel kernels read the committed decision
  if (kpan_.panels || ktpan_.panels) it.decide_sep = 1;
  it.seq_dy2 = seq_dy2_.get();
  it.seq_inter = seq_inter_.get();
  it.seq_dx2 = seq_dx2_.get();
  it.red_tab = reinterpret_cast<const double*>(xfer_dev_.get() + xo_tab_);
  it.step_log = step_log_dev_.get();
  // iteration engine
  engine_ = params_.engine;
  if (engine_ == PDLP_ENGINE_AUTO)
    engine_ = params_.use_cuda_graph ? PDLP_ENGINE_GRAPH : PDLP_ENGINE_STREAM;
  // fast per-trial kernels skip storing K'y' on accepted steps (8n bytes per
  // iteration)
  it.kty_lazy = (!parity() && !std::getenv("PDLP_NO_LAZY_KTY")) ? 1 : 0;
  // L2 prefetch of the tiles before griddepcontrol.wait (overlapping the
  // previous kernel's tail) pays where the operators are mid-sized and mostly
  // L2-resident: C2 123.9 -> 119.3 ms per solve. Tiny operators only pay the
  // extra prologue (C1 20.2 -> 20.9 ms) and ones far beyond L2 lose the
  // gathered vector to the prefetched lines (C3 200.5 -> 207.4 ms).
  it.prefetch = (nnz_ >= (int64_t(1) << 20) && nnz_ <= (int64_t(8) << 20)) ? 1 : 0;
  if (const char* e = std::getenv("PDLP_PREFETCH")) it.prefetch = std::atoi(e) != 0;
  it.st = state_dev_;

  X4_.alloc(size_t(n_) * 4);
  Y4_.alloc(size_t(m_) * 4);
  lam_.alloc(size_t(n_) * 4, world_ > 1);
  scratch_n_.alloc(n_);
  scratch_m_.alloc(m_);
  const int grid0 = eval_grid0(int(n_), int(m_));
  part0_.alloc(size_t(std::max(1, grid0)) * 4);
  const int ev1_tiles = int(k_ev_.plan.tiles.size()), ev2_tiles = int(kt_ev_.plan.tiles.size());
  part1_.alloc(size_t(ev1_tiles) * 14, world_ > 1);
  part2_.alloc(size_t(ev2_tiles) * 18, world_ > 1);
  seq_r_.alloc(seq ? size_t(m_) * 4 : 1);
  seq_d_.alloc(seq ? size_t(n_) * 4 : 1);

  DevEval& ev = ev_;
  ev.X4 = X4_.get();
  ev.Y4 = Y4_.get();
  ev.lam = lam_.get();
  ev.c = c_orig_.get();
  ev.l = l_orig_.get();
  ev.u = u_orig_.get();
  ev.q = q_orig_.get();
  ev.d1 = d1_dev_.get();
  ev.d2 = d2_dev_.get();
  ev.objective_constant = objective_constant_;
  ev.part0 = part0_.get();
  ev.part1 = part1_.get();
  ev.part2 = part2_.get();
  ev.grid0 = grid0;
  ev.seq_r = seq_r_.get();
  ev.seq_d = seq_d_.get();
  ev.out = eval_dev_;
  ev.ev1_tiles = ev1_tiles;
  ev.ev2_tiles = ev2_tiles;
  eval_stage_.alloc(36 * size_t(kEvalReduceCtas));
  ev.stage = eval_stage_.get();

  // sharding: own slices, sync block, peer table (own entries until linked)
  sync_.alloc(1, world_ > 1);
  sync_.zero(s);
  shv_dev_.alloc(1);
  it.world = world_, it.rank = rank_;
  it.row0 = int(row0), it.row1 = int(row1), it.col0 = int(col0), it.col1 = int(col1);
  it.sync = sync_.get();
  it.shv = shv_dev_.get();
  ev.world = world_, ev.rank = rank_;
  ev.sync = sync_.get();
  ev.shv = shv_dev_.get();
  // trials push x' / y' only to the peers whose rows gather them (a banded or
  // staircase operator exchanges its coupling values only); PDLP_SHARD_FULL=1
  // pushes every value to every peer
  it.xmask = it.ymask = nullptr;
  if (world_ > 1 && !std::getenv("PDLP_SHARD_FULL")) {
    DevBuf<int64_t> kc{k_cuts_.size()}, ktc{kt_cuts_.size()};
    PDLP_CUDA(cudaMemcpyAsync(kc.get(), k_cuts_.data(), k_cuts_.size() * 8, cudaMemcpyHostToDevice, s));
    PDLP_CUDA(cudaMemcpyAsync(ktc.get(), kt_cuts_.data(), kt_cuts_.size() * 8, cudaMemcpyHostToDevice, s));
    xmask_.alloc(n_);
    ymask_.alloc(m_);
    xmask_.zero(s);
    launch_shard_masks(k_rp_.get(), k_col_.get(), int(m_), kc.get(), ktc.get(), world_, xmask_.get(), ymask_.get(), s);
    DevBuf<unsigned long long> vol{static_cast<size_t>(2)};
    vol.zero(s);
    launch_shard_volume(xmask_.get(), ymask_.get(), int(col0), int(col1), int(row0), int(row1), world_, rank_,
                        vol.get(), s);
    unsigned long long vh[2] = {0, 0};
    PDLP_CUDA(cudaMemcpyAsync(vh, vol.get(), sizeof vh, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
    push_values_ = int64_t(vh[0]);
    push_values_full_ = int64_t(vh[1]);
    it.xmask = xmask_.get();
    it.ymask = ymask_.get();
  } else if (world_ > 1) {
    push_values_ = push_values_full_ = ((col1 - col0) + (row1 - row0)) * int64_t(world_ - 1);
  }
  // a rank keeps only its own rows of K and K^T from here on (the setup above
  // needed all of them: scaling, plans, gather masks)
  if (world_ > 1 && !std::getenv("PDLP_SHARD_KEEP_ALL")) compact_own_rows();
  for (int q = 0; q < kMaxShards; ++q) {
    shv_.x_all[q] = x_all_.get();
    shv_.y_all[q] = y_all_.get();
    shv_.d_part[q] = d_part_.get();
    shv_.p_part[q] = p_part_.get();
    shv_.avg_x[q] = avg_x_.get();
    shv_.avg_y[q] = avg_y_.get();
    shv_.part1[q] = part1_.get();
    shv_.part2[q] = part2_.get();
    shv_.lam[q] = lam_.get();
    shv_.sync[q] = sync_.get();
  }
  shard_view_upload();
  linked_ = world_ == 1;
}

void Solver::shard_view_upload() {
  PDLP_CUDA(cudaMemcpyAsync(shv_dev_.get(), &shv_, sizeof(ShardView), cudaMemcpyHostToDevice, stream_));
  PDLP_CUDA(cudaStreamSynchronize(stream_));
}

void Solver::require_linked() const {
  if (!linked_) throw std::logic_error("sharded rank: peers not linked (pdlp_shard_link_local / import)");
}

// The evaluation window as one CUDA graph: WHILE(cond) { dual; primal }, the
// condition being cleared by the dual kernel's last CTA once the window's
// accepted-step target is met (or the step failed).
void Solver::capture_window_graph() {
  PDLP_CUDA(cudaGraphCreate(&graph_, 0));
  cudaGraphConditionalHandle h;
  PDLP_CUDA(cudaGraphConditionalHandleCreate(&h, graph_, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  PDLP_CUDA(cudaGraphAddNode(&node, graph_, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  PDLP_CUDA(cudaStreamBeginCaptureToGraph(stream_, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
  const unsigned long long ch = static_cast<unsigned long long>(h);
  // whichever kernel takes the step decision sets the WHILE condition
  const int ds = it_.decide_sep;
  dual_step(ch, (parity() || ds == 2) ? 1 : 0);
  if (ds == 1) launch_decide(it_, stream_, ch, 1);
  primal_step(-1, ch, (!parity() && ds == 0) ? 1 : 0);
  PDLP_CUDA(cudaStreamEndCapture(stream_, &body));
  PDLP_CUDA(cudaGraphInstantiate(&graph_exec_, graph_, 0));
  cond_handle_ = static_cast<unsigned long long>(h);
}

// WHILE(chain) { WHILE(window) { dual; primal }; evaluation; chain decision }.
// The inner body is the same capture as capture_window_graph; the outer body
// adds the evaluation block of launch_eval and chain_decide_kernel, which
// either re-arms both conditions for the next window or ends the chain.
void Solver::capture_chain_graph() {
  PDLP_CUDA(cudaGraphCreate(&chain_graph_, 0));
  cudaGraphConditionalHandle ho, hi;
  PDLP_CUDA(cudaGraphConditionalHandleCreate(&ho, chain_graph_, 1, cudaGraphCondAssignDefault));
  PDLP_CUDA(cudaGraphConditionalHandleCreate(&hi, chain_graph_, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams op = {};
  op.type = cudaGraphNodeTypeConditional;
  op.conditional.handle = ho;
  op.conditional.type = cudaGraphCondTypeWhile;
  op.conditional.size = 1;
  cudaGraphNode_t onode;
  PDLP_CUDA(cudaGraphAddNode(&onode, chain_graph_, nullptr, 0, &op));
  cudaGraph_t obody = op.conditional.phGraph_out[0];
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hi;
  ip.conditional.type = cudaGraphCondTypeWhile;
  ip.conditional.size = 1;
  cudaGraphNode_t inode;
  PDLP_CUDA(cudaGraphAddNode(&inode, obody, nullptr, 0, &ip));
  cudaGraph_t ibody = ip.conditional.phGraph_out[0];
  const unsigned long long ci = static_cast<unsigned long long>(hi), co = static_cast<unsigned long long>(ho);
  // inner body: one trial (as capture_window_graph)
  PDLP_CUDA(cudaStreamBeginCaptureToGraph(stream_, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  const int ds = it_.decide_sep;
  dual_step(ci, ds == 2 ? 1 : 0);
  if (ds == 1) launch_decide(it_, stream_, ci, 1);
  primal_step(-1, ci, ds == 0 ? 1 : 0);
  PDLP_CUDA(cudaStreamEndCapture(stream_, &ibody));
  // outer body after the inner loop: evaluation + decision
  PDLP_CUDA(cudaStreamBeginCaptureToGraph(stream_, obody, &inode, nullptr, 1, cudaStreamCaptureModeThreadLocal));
  launch_eval(k_ev_.csr, kt_ev_.csr, it_, ev_, false, stream_, phase_, fork_.s2 ? &fork_ : nullptr);
  ChainConsts k{};
  k.eps_optimal = params_.eps_optimal;
  k.eps_infeasible = params_.eps_infeasible;
  k.eps_zero = params_.eps_zero;
  k.beta_sufficient = params_.beta_sufficient;
  k.beta_necessary = params_.beta_necessary;
  k.beta_artificial = params_.beta_artificial;
  k.rhs_norm = rhs_norm_;
  k.obj_norm = obj_norm_;
  k.iteration_limit = params_.iteration_limit;
  k.freq = int32_t(params_.evaluation_frequency);
  launch_chain_decide(state_dev_, eval_dev_, k, co, ci, stream_);
  PDLP_CUDA(cudaStreamEndCapture(stream_, &obody));
  PDLP_CUDA(cudaGraphInstantiate(&chain_exec_, chain_graph_, 0));
}

bool Solver::chain_enabled() const {
  return chain_windows_ > 1 && engine_ == PDLP_ENGINE_GRAPH;
}

// Up to `windows` full windows with the evaluations between them decided on
// the device. Returns true when the chain ended on a device-decided
// evaluation (nothing left for evaluation_block), false when the last
// evaluation needs the host (termination, infeasibility, restart) or a window
// failed.
bool Solver::run_chain(int windows) {
  DevState& st = *hs_;
  const int freq = int(params_.evaluation_frequency);
  double* tab = tab_host_;
  const int steps = windows * freq;
  for (int i = 0; i < steps; ++i) {
    const double kp1 = double(st.total + 1 + i) + 1.0;
    tab[2 * i] = 1.0 - std::pow(kp1, -params_.step_reduction_exponent);
    tab[2 * i + 1] = 1.0 + std::pow(kp1, -params_.step_growth_exponent);
  }
  st.window_target = freq;
  st.window_accepts = 0;
  st.table_base = st.total;
  st.failure = 0;
  st.kkt_epoch_start = kkt_epoch_start_;
  st.kkt_last = kkt_last_;
  st.chain_left = windows - 1;
  st.chain_stop = 0;
  st.chain_evals = 0;
  const int64_t trials_before = st.trials_total;
  PDLP_CUDA(cudaMemcpyAsync(state_dev_, hs_, xo_tab_ - xo_state_ + 2 * sizeof(double) * size_t(steps),
                            cudaMemcpyHostToDevice, stream_));
  eval_fresh_ = false;
  PDLP_CUDA(cudaEventRecord(ev_w0_, stream_));
  if (!chain_exec_) capture_chain_graph();
  PDLP_CUDA(cudaGraphLaunch(chain_exec_, stream_));
  PDLP_CUDA(cudaEventRecord(ev_w1_, stream_));
  PDLP_CUDA(cudaEventRecord(ev_e1_, stream_));
  PDLP_CUDA(cudaMemcpyAsync(he_, eval_dev_, xo_state_ + sizeof(DevState), cudaMemcpyDeviceToHost, stream_));
  spin_sync();
  eval_fresh_ = true;
  {
    float ms = 0.f;
    PDLP_CUDA(cudaEventElapsedTime(&ms, ev_w0_, ev_w1_));
    window_seconds_ += 1e-3 * double(ms);  // windows and their evaluations
    const int ran = windows - st.chain_left;
    if (ran > 0) window_time_est_ = 1e-3 * double(ms) / double(ran);
  }
  const int evals = st.chain_evals + (st.chain_stop == 1 ? 1 : 0);
  evaluations_ += evals;
  launches_ += int64_t(evals) * 6 + (it_.decide_sep == 1 ? 3 : 2) * (st.trials_total - trials_before);
  kkt_last_ = st.kkt_last;
  return st.chain_stop == 2;
}

void Solver::upload_state() {
  PDLP_CUDA(cudaMemcpyAsync(state_dev_, hs_, sizeof(DevState), cudaMemcpyHostToDevice,
                            stream_));
}

void Solver::download_state() {
  PDLP_CUDA(cudaMemcpyAsync(hs_, state_dev_, sizeof(DevState), cudaMemcpyDeviceToHost,
                            stream_));
  spin_sync();
}

// The per-window round trip waits by polling the stream: the host resumes as
// soon as the device finishes instead of after a blocking-sync wake-up.
void Solver::spin_sync() {
  for (;;) {
    const cudaError_t e = cudaStreamQuery(stream_);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) PDLP_CUDA(e);
  }
}

double Solver::elapsed() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
}

// ---------------------------------------------------------------------------
// the loop
// ---------------------------------------------------------------------------

void Solver::iterate_begin(int32_t* status) {
  PDLP_CUDA(cudaSetDevice(params_.device));
  require_linked();
  // graphs are captured and instantiated once per handle, before the solve's
  // clocks start (the first instantiation in a process also loads the modules)
  if (engine_ == PDLP_ENGINE_GRAPH && !graph_exec_) capture_window_graph();
  if (chain_enabled() && !chain_exec_) capture_chain_graph();
  t0_ = std::chrono::steady_clock::now();
  DevState& st = *hs_;
  std::memset(&st, 0, sizeof st);
  st.eta = eta_hat0_;
  st.eta_acc = eta_hat0_;
  st.omega = omega0_;
  st.ix_cur = 0, st.ix_prev = 1, st.ix_trial = 2;
  st.iy_cur = 0, st.iy_prev = 1, st.iy_trial = 2;
  st.ikx_cur = 0, st.ikty_cur = 0;
  st.record_log = params_.record_step_log ? 1 : 0;
  outer_ = 0;
  launches_ = 0;
  evaluations_ = 0;
  step_log_.clear();
  restart_log_.clear();
  finished_ = false;
  begun_ = true;
  state_valid_ = true;
  std::memset(&info_, 0, sizeof info_);
  if (!ev_begin_) {
    PDLP_CUDA(cudaEventCreate(&ev_begin_));
    PDLP_CUDA(cudaEventCreate(&ev_end_));
    PDLP_CUDA(cudaEventCreate(&ev_w0_));
    PDLP_CUDA(cudaEventCreate(&ev_w1_));
    PDLP_CUDA(cudaEventCreate(&ev_e1_));
  }
  window_seconds_ = 0.0;
  eval_seconds_ = 0.0;
  PDLP_CUDA(cudaEventRecord(ev_begin_, stream_));
  upload_state();
  eval_fresh_ = false;
  launch_zero_iterate(it_, stream_);  // z = 0, Kx = K 0 = 0, K'y = 0 (solver.hpp:764-769)
  ++launches_;
  // initial evaluation on the unscaled zero point (solver.hpp:784-792)
  evaluate();
  const KktHost r0 = kkt(0);
  kkt_epoch_start_ = r0.weighted(st.omega);
  kkt_last_ = kkt_epoch_start_;
  if (terminated(r0)) {
    finish(PDLP_STATUS_OPTIMAL, 0, 0, 0, r0);
  } else {
    // first trial x' = proj(x - tau (c - K'y)) at z = 0
    upload_state();
    primal_step(kPRetry);
    phase();
    ++launches_;
  }
  if (status) *status = finished_ ? info_.status : PDLP_STATUS_RUNNING;
}

void Solver::iterate_run(int64_t count, int32_t* status) {
  if (!begun_ || !state_valid_) throw std::logic_error("iterate_run before iterate_begin");
  PDLP_CUDA(cudaSetDevice(params_.device));
  DevState& st = *hs_;
  const int64_t freq = params_.evaluation_frequency;
  int64_t done = 0;
  while (!finished_ && done < count) {
    // limits at the loop top (solver.hpp:795-804); the time limit is checked
    // once per window
    if (st.total >= params_.iteration_limit) {
      evaluate();
      finish_candidate(PDLP_STATUS_ITERATION_LIMIT);
      break;
    }
    if (elapsed() >= params_.time_limit_seconds) {
      evaluate();
      finish_candidate(PDLP_STATUS_TIME_LIMIT);
      break;
    }
    int64_t target = freq - st.inner % freq;
    target = std::min<int64_t>(target, params_.iteration_limit - st.total);
    target = std::min<int64_t>(target, count - done);
    target = std::min<int64_t>(target, tab_cap_);
    const int64_t before = st.total;
    // a chain may use half of the remaining time limit, at the measured window rate
    const double left = params_.time_limit_seconds - elapsed();
    const int64_t by_time = window_time_est_ > 0.0 ? int64_t(0.5 * left / window_time_est_) : 0;
    if (chain_enabled() && target == freq && st.inner % freq == 0 &&
        count - done >= int64_t(freq) * chain_windows_ && by_time >= 2) {
      // whole windows back to back on the device; the host sees only the
      // evaluation that needs it (or the chain's end)
      const int64_t fit = (params_.iteration_limit - st.total) / freq;
      const int w = int(std::min<int64_t>(std::min<int64_t>(chain_windows_, fit), by_time));
      const bool handled = run_chain(w);
      done += st.total - before;
      if (st.failure) {
        evaluate();
        finish_candidate(PDLP_STATUS_NUMERICAL_ERROR,
                         "non-finite iterate in adaptive step at iteration " + std::to_string(st.total));
        break;
      }
      if (!handled) evaluation_block();
      continue;
    }
    run_window(int(target));
    done += st.total - before;
    if (st.failure) {
      evaluate();
      finish_candidate(PDLP_STATUS_NUMERICAL_ERROR,
                       "non-finite iterate in adaptive step at iteration " + std::to_string(st.total));
      break;
    }
    if (st.inner % freq != 0) continue;
    evaluate();
    evaluation_block();
  }
  if (status) *status = finished_ ? info_.status : PDLP_STATUS_RUNNING;
}

void Solver::run_window(int target) {
  DevState& st = *hs_;
  double* tab = tab_host_;
  for (int i = 0; i < target; ++i) {
    // factors of adaptive_step_cached for step counter k = total + 1 (solver.hpp:388-390)
    const double kp1 = double(st.total + 1 + i) + 1.0;
    tab[2 * i] = 1.0 - std::pow(kp1, -params_.step_reduction_exponent);
    tab[2 * i + 1] = 1.0 + std::pow(kp1, -params_.step_growth_exponent);
  }
  st.window_target = target;
  st.window_accepts = 0;
  st.table_base = st.total;
  st.failure = 0;
  const int64_t trials_before = st.trials_total;
  // state + the window's factor pairs in one H2D copy
  PDLP_CUDA(cudaMemcpyAsync(state_dev_, hs_, xo_tab_ - xo_state_ + 2 * sizeof(double) * size_t(target),
                            cudaMemcpyHostToDevice, stream_));
  eval_fresh_ = false;
  PDLP_CUDA(cudaEventRecord(ev_w0_, stream_));
  if (engine_ == PDLP_ENGINE_GRAPH) {
    if (!graph_exec_) capture_window_graph();
    PDLP_CUDA(cudaGraphLaunch(graph_exec_, stream_));
  } else {
    int remaining = target;
    while (true) {
      for (int i = 0; i < remaining; ++i) {
        dual_step(0, 0);
        phase();
        if (it_.decide_sep == 1) launch_decide(it_, stream_);
        primal_step(-1);
        phase();
      }
      download_state();
      if (st.failure || st.window_accepts >= target) break;
      remaining = target - st.window_accepts;
    }
  }
  PDLP_CUDA(cudaEventRecord(ev_w1_, stream_));
  // the evaluation block is enqueued behind the window (it reads the device
  // state), so one host round trip per window brings back state, scalars, log
  launch_eval(k_ev_.csr, kt_ev_.csr, it_, ev_, parity(), stream_, phase_, fork_.s2 ? &fork_ : nullptr);
  PDLP_CUDA(cudaEventRecord(ev_e1_, stream_));
  launches_ += parity() ? 6 : 5;  // prep, rows, cols, reduce, final (+ parity displacement)
  ++evaluations_;
  // evaluation results + state in one D2H copy
  PDLP_CUDA(cudaMemcpyAsync(he_, eval_dev_, xo_state_ + sizeof(DevState), cudaMemcpyDeviceToHost,
                            stream_));
  if (st.record_log)
    PDLP_CUDA(cudaMemcpyAsync(log_host_.get(), step_log_dev_.get(),
                              size_t(target) * sizeof(pdlp_step_log_entry), cudaMemcpyDeviceToHost,
                              stream_));
  spin_sync();
  eval_fresh_ = true;
  {
    float ms = 0.f;
    PDLP_CUDA(cudaEventElapsedTime(&ms, ev_w0_, ev_w1_));
    window_seconds_ += 1e-3 * double(ms);
    float ems = 0.f;
    PDLP_CUDA(cudaEventElapsedTime(&ems, ev_w1_, ev_e1_));
    eval_seconds_ += 1e-3 * double(ems);
    if (target == int(params_.evaluation_frequency)) window_time_est_ = 1e-3 * double(ms + ems);
  }
  launches_ += (it_.decide_sep == 1 ? 3 : 2) * (st.trials_total - trials_before);
  if (st.record_log && st.window_accepts > 0)
    step_log_.insert(step_log_.end(), log_host_.get(), log_host_.get() + st.window_accepts);
}

void Solver::evaluate() {
  if (eval_fresh_) return;  // nothing changed since the window's own evaluation
  upload_state();
  launch_eval(k_ev_.csr, kt_ev_.csr, it_, ev_, parity(), stream_, phase_, fork_.s2 ? &fork_ : nullptr);
  launches_ += parity() ? 6 : 5;  // prep, rows, cols, reduce, final (+ parity displacement)
  ++evaluations_;
  PDLP_CUDA(cudaMemcpyAsync(he_, eval_dev_, sizeof(EvalOut), cudaMemcpyDeviceToHost,
                            stream_));
  spin_sync();
  eval_fresh_ = true;
}

KktHost Solver::kkt(int slot) const {
  const EvalOut& e = *he_;
  return KktHost{e.prn[slot], e.drn[slot], e.pobj[slot], e.dobj[slot]};
}

// termination_criteria_met (solver.hpp:204-222)
bool Solver::terminated(const KktHost& r) const {
  if (!std::isfinite(r.prn) || !std::isfinite(r.drn) || !std::isfinite(r.pobj) ||
      !std::isfinite(r.dobj))
    return false;
  const double eps = params_.eps_optimal;
  const bool gap_ok = std::abs(r.gap()) <= eps * (1.0 + std::abs(r.dobj) + std::abs(r.pobj));
  const bool p_ok = r.prn <= eps * (1.0 + rhs_norm_);
  const bool d_ok = r.drn <= eps * (1.0 + obj_norm_);
  return gap_ok && p_ok && d_ok;
}

// The evaluation block of SolveLoop::run (solver.hpp:843-927).
void Solver::evaluation_block() {
  DevState& st = *hs_;
  const EvalOut& e = *he_;
  const KktHost cur = kkt(0), avg = kkt(1);
  const double kc = cur.weighted(st.omega), ka = avg.weighted(st.omega);
  const int cand = !(kc < ka) ? 1 : 0;  // ties go to the average (:718)
  const KktHost rc = cand ? avg : cur, ro = cand ? cur : avg;
  const double kkt_cand = cand ? ka : kc;
  if (terminated(rc)) return finish(PDLP_STATUS_OPTIMAL, cand, cand, cand, rc);
  if (terminated(ro)) return finish(PDLP_STATUS_OPTIMAL, 1 - cand, 1 - cand, 1 - cand, ro);

  // check_infeasibility: delta ray, then normalized ray (solver.hpp:581-590)
  const double eps_inf = params_.eps_infeasible, eps_zero = params_.eps_zero;
  for (int r = 0; r < 2; ++r) {
    const double yn = e.y_norm[r];
    if (yn > eps_zero && e.kty_resid[r] <= eps_inf * yn && e.ray_dobj[r] > eps_inf * yn) {
      finish(PDLP_STATUS_PRIMAL_INFEASIBLE, -1, 2 + r, 2 + r, rc);
      info_.has_certificate = 1;
      return;
    }
    const double xn = e.x_norm[r];
    if (xn > eps_zero) {
      const double tol = eps_inf * xn;
      const bool ok = e.ax_norm[r] <= tol && !(e.gx_negmax[r] > tol) && !(e.xl_negmax[r] > tol) &&
                      !(e.xu_max[r] > tol) && e.cx[r] < -tol;
      if (ok) {
        finish(PDLP_STATUS_DUAL_INFEASIBLE, 2 + r, -1, -2, rc);
        info_.has_certificate = 1;
        return;
      }
    }
  }

  // should_restart (solver.hpp:270-286, :887-892)
  const double prev = kkt_last_;
  int crit = PDLP_RESTART_NONE;
  if (kkt_cand <= params_.beta_sufficient * kkt_epoch_start_)
    crit = PDLP_RESTART_SUFFICIENT_DECAY;
  else if (kkt_cand <= params_.beta_necessary * kkt_epoch_start_ && kkt_cand > prev)
    crit = PDLP_RESTART_NECESSARY_DECAY;
  else if (double(st.inner) >= params_.beta_artificial * double(st.total))
    crit = PDLP_RESTART_LONG_INNER_LOOP;
  kkt_last_ = kkt_cand;
  if (crit == PDLP_RESTART_NONE) return;

  pdlp_restart_event ev{};
  ev.total_iterations = st.total;
  ev.epoch_length = st.inner;
  ev.criterion = crit;
  ev.candidate_is_average = cand;
  ev.kkt_candidate = kkt_cand;
  ev.kkt_previous_candidate = prev;
  ev.kkt_epoch_start = kkt_epoch_start_;
  ev.omega_before = st.omega;

  // restart (solver.hpp:907-927): z_start = z = candidate, fresh products,
  // averages reset, primal weight update (:305-325) with host glibc exp/log
  const double dx = std::sqrt(e.dx2[cand]), dy = std::sqrt(e.dy2[cand]);
  double omega = st.omega;
  if (dx > eps_zero && dy > eps_zero)
    omega = std::exp(params_.theta_smoothing * std::log(dy / dx) +
                     (1.0 - params_.theta_smoothing) * std::log(st.omega));
  const bool from_avg = cand == 1 && st.wsum != 0.0;
  upload_state();
  launch_restart_copy(it_, from_avg ? 1 : 0, stream_);
  st.omega = sclamp(omega, params_.omega_min, params_.omega_max);
  st.wsum = 0.0;
  st.inner = 0;
  outer_ += 1;
  upload_state();
  launch_spmv(K_, false, it_.x[st.ix_cur], it_.kx[st.ikx_cur], parity(), stream_);
  primal_step(kPRestart);
  phase();
  launches_ += 3;
  eval_fresh_ = false;
  ev.omega_after = st.omega;
  restart_log_.push_back(ev);
  kkt_epoch_start_ = rc.weighted(st.omega);
  kkt_last_ = kkt_epoch_start_;
}

namespace {
std::mutex& pinned_pool_mu() {
  static std::mutex mu;
  return mu;
}
// blocks are kept for the life of the process (bounded by peak concurrent use)
std::multimap<size_t, void*>& pinned_pool() {
  static auto* pool = new std::multimap<size_t, void*>();
  return *pool;
}
}  // namespace

void* pinned_pool_get(size_t bytes, size_t* capacity) {
  std::lock_guard<std::mutex> g(pinned_pool_mu());
  auto& pool = pinned_pool();
  // smallest free block that fits, if it is not wastefully large
  auto it = pool.lower_bound(bytes);
  if (it != pool.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
    void* p = it->second;
    *capacity = it->first;
    pool.erase(it);
    return p;
  }
  void* p = nullptr;
  const size_t cap = std::max<size_t>(bytes, 64);
  PDLP_CUDA(cudaMallocHost(&p, cap));
  *capacity = cap;
  return p;
}

void pinned_pool_put(void* p, size_t capacity) {
  std::lock_guard<std::mutex> g(pinned_pool_mu());
  pinned_pool().emplace(capacity, p);
}

void Solver::finish_candidate(int status, const std::string& msg) {
  const DevState& st = *hs_;
  const KktHost cur = kkt(0), avg = kkt(1);
  const int cand = !(cur.weighted(st.omega) < avg.weighted(st.omega)) ? 1 : 0;
  finish(status, cand, cand, cand, cand ? avg : cur, msg);
}

// SolveLoop::finish (solver.hpp:741-757). slot_x/slot_y: which of the four
// evaluated points supplies x / y (-1 = zero vector); slot_lam: reduced costs
// of that slot, or -2 for reduced_costs(lp, 0) of a dual-infeasibility exit.
void Solver::finish(int status, int slot_x, int slot_y, int slot_lam, const KktHost& r,
                    const std::string& msg) {
  const DevState& st = *hs_;
  cudaStream_t s = stream_;
  // overwritten below by the D2H copies; zero vectors where no slot supplies one
  if (slot_x >= 0) rx_.resize(size_t(n_)); else rx_.assign(size_t(n_), 0.0);
  if (slot_y >= 0) ry_.resize(size_t(m_)); else ry_.assign(size_t(m_), 0.0);
  rlam_.resize(size_t(n_));
  // the returned point is one slot of the interleaved [.][4] evaluation
  // arrays: extract it on the device (a pitched 8-byte-wide D2H copy costs
  // milliseconds at n = 1e6), then contiguous copies after the device clock
  // stops (the solve's device time excludes the PCIe download)
  const double* lam_src = nullptr;
  if (slot_x >= 0 && n_) launch_extract_slot(X4_.get(), slot_x, n_, scratch_n_.get(), s);
  if (slot_y >= 0 && m_) launch_extract_slot(Y4_.get(), slot_y, m_, scratch_m_.get(), s);
  if (n_) {
    if (slot_lam >= 0) {
      launch_eval_lambda(kt_ev_.csr, it_, ev_, parity(), slot_lam, s, phase_);
      lam_src = lam_.get() + size_t(slot_lam) * n_;
    } else {  // reduced_costs(lp, 0) of a dual-infeasibility exit, into lam_'s slot 0
      launch_reduced_of_objective(c_orig_.get(), l_orig_.get(), u_orig_.get(), int(n_), lam_.get(), s);
      lam_src = lam_.get();
    }
  }
  PDLP_CUDA(cudaEventRecord(ev_end_, s));
  if (slot_x >= 0 && n_)
    PDLP_CUDA(cudaMemcpyAsync(rx_.data(), scratch_n_.get(), n_ * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (slot_y >= 0 && m_)
    PDLP_CUDA(cudaMemcpyAsync(ry_.data(), scratch_m_.get(), m_ * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (lam_src)
    PDLP_CUDA(cudaMemcpyAsync(rlam_.data(), lam_src, n_ * sizeof(double), cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  pdlp_result_info& in = info_;
  std::memset(&in, 0, sizeof in);
  in.status = status;
  in.primal_objective_raw = r.pobj;
  in.dual_objective_raw = r.dobj;
  in.primal_objective = r.pobj + objective_constant_;
  in.dual_objective = r.dobj + objective_constant_;
  in.gap_abs = std::abs(r.gap());
  in.primal_residual_norm = r.prn;
  in.dual_residual_norm = r.drn;
  in.relative_gap = in.gap_abs / (1.0 + std::abs(r.dobj) + std::abs(r.pobj));
  in.relative_primal_residual = r.prn / (1.0 + rhs_norm_);
  in.relative_dual_residual = r.drn / (1.0 + obj_norm_);
  in.kkt_omega = r.weighted(st.omega);
  in.iterations = st.total;
  in.restarts = outer_;
  in.solve_seconds = elapsed();
  in.setup_seconds = setup_seconds_;
  {
    float ms = 0.f;
    PDLP_CUDA(cudaEventElapsedTime(&ms, ev_begin_, ev_end_));
    in.device_seconds = 1e-3 * double(ms);
    in.window_seconds = window_seconds_;
    in.eval_seconds = eval_seconds_;
  }
  in.step_log_size = int64_t(step_log_.size());
  in.restart_log_size = int64_t(restart_log_.size());
  in.num_variables = n_;
  in.num_constraints = m_;
  in.trials = st.trials_total;
  in.evaluations = evaluations_;
  in.gpu_launches = launches_;
  std::snprintf(in.message, sizeof in.message, "%s", msg.c_str());
  finished_ = true;
}

void Solver::solve(pdlp_result_info* info) {
  int32_t status;
  iterate_begin(&status);
  while (!finished_) iterate_run(std::numeric_limits<int64_t>::max(), &status);
  if (info) *info = info_;
}

// ---------------------------------------------------------------------------
// accessors
// ---------------------------------------------------------------------------

void Solver::get_iterate(double* x, double* y, double* kx, double* kty, int64_t* counters,
                         double* scalars) {
  if (!state_valid_) throw std::logic_error("no live iterate (call iterate_begin)");
  const DevState& st = *hs_;
  cudaStream_t s = stream_;
  if (x && n_) PDLP_CUDA(cudaMemcpyAsync(x, it_.x[st.ix_cur], n_ * 8, cudaMemcpyDeviceToHost, s));
  if (y && m_) PDLP_CUDA(cudaMemcpyAsync(y, it_.y[st.iy_cur], m_ * 8, cudaMemcpyDeviceToHost, s));
  if (kx && m_)
    PDLP_CUDA(cudaMemcpyAsync(kx, kx_[st.ikx_cur].get(), m_ * 8, cudaMemcpyDeviceToHost, s));
  if (kty && n_) {
    // lazily kept K'y': recompute it for the current y (same tiles and order
    // as the primal kernel, so bitwise what it would have stored)
    if (it_.kty_lazy)
      launch_spmv(compacted_ ? KT_ : KT_full_, false, it_.y[st.iy_cur], it_.kty[st.ikty_cur], parity(), s);
    PDLP_CUDA(cudaMemcpyAsync(kty, kty_[st.ikty_cur].get(), n_ * 8, cudaMemcpyDeviceToHost, s));
  }
  PDLP_CUDA(cudaStreamSynchronize(s));
  if (counters) {
    counters[0] = st.total;
    counters[1] = st.inner;
    counters[2] = outer_;
    counters[3] = st.trials_total;
  }
  if (scalars) {
    scalars[0] = st.eta_acc;
    scalars[1] = st.eta;
    scalars[2] = st.omega;
    scalars[3] = st.wsum;
  }
}

void Solver::get_solution(double* x, double* y, double* lambda, double* lambda_pos,
                          double* lambda_neg) {
  if (!finished_) throw std::logic_error("no solution: solve has not finished");
  if (x) std::copy(rx_.begin(), rx_.end(), x);
  if (y) std::copy(ry_.begin(), ry_.end(), y);
  for (int64_t j = 0; j < n_; ++j) {
    const double v = rlam_[j];
    if (lambda) lambda[j] = v;
    if (lambda_pos) lambda_pos[j] = v > 0.0 ? v : 0.0;
    if (lambda_neg) lambda_neg[j] = v < 0.0 ? -v : 0.0;
  }
}

int64_t Solver::get_step_log(pdlp_step_log_entry* out, int64_t cap) const {
  const int64_t k = std::min<int64_t>(cap, int64_t(step_log_.size()));
  if (out) std::copy(step_log_.begin(), step_log_.begin() + k, out);
  return k;
}

int64_t Solver::get_restart_log(pdlp_restart_event* out, int64_t cap) const {
  const int64_t k = std::min<int64_t>(cap, int64_t(restart_log_.size()));
  if (out) std::copy(restart_log_.begin(), restart_log_.begin() + k, out);
  return k;
}

void Solver::get_scaling(double* row_scale, double* col_scale) const {
  if (row_scale) std::copy(d1_.begin(), d1_.end(), row_scale);
  if (col_scale) std::copy(d2_.begin(), d2_.end(), col_scale);
}

void Solver::spmv(int op, const double* in, double* out) {
  if (compacted_) throw std::logic_error("spmv: a sharded rank keeps only its own rows of the operators");
  const bool transpose = op == PDLP_OP_KT_SCALED || op == PDLP_OP_KT_ORIGINAL;
  const bool orig = op == PDLP_OP_K_ORIGINAL || op == PDLP_OP_KT_ORIGINAL;
  if (op < 0 || op > 3) invalid("spmv: unknown operator");
  const int64_t nin = transpose ? m_ : n_, nout = transpose ? n_ : m_;
  DevBuf<double> din(nin), dout(nout);
  if (nin) PDLP_CUDA(cudaMemcpyAsync(din.get(), in, nin * 8, cudaMemcpyHostToDevice, stream_));
  // the scaled operator through the engine the iteration uses (column panels
  // when the operator is panelized)
  const PanelOp& po = transpose ? ktpan_ : kpan_;
  if (!orig && po.panels)
    launch_panel_spmv(po.view, din.get(), dout.get(), stream_);
  else
    launch_spmv(transpose ? KT_full_ : K_full_, orig, din.get(), dout.get(), parity(), stream_);
  if (nout) PDLP_CUDA(cudaMemcpyAsync(out, dout.get(), nout * 8, cudaMemcpyDeviceToHost, stream_));
  PDLP_CUDA(cudaStreamSynchronize(stream_));
}

// Times the fused iteration kernels on a live window (after a solve). Each
// repetition runs a real trial (dual then primal); the events bracket only the
// kernel being timed. Leaves the iterate state invalid.
void Solver::time_kernel(int which, int reps, double* avg_ms, double* bytes) {
  if (world_ > 1) throw std::logic_error("time_kernel: single-device handles only");
  if (!begun_) {
    int32_t s;
    iterate_begin(&s);
  }
  if (which == 2 || which == 3) {
    // plain SpMV microbenchmark on device-resident vectors: 2 = K x, 3 = K^T y
    const DevState& st = *hs_;
    cudaEvent_t e0, e1;
    PDLP_CUDA(cudaEventCreate(&e0));
    PDLP_CUDA(cudaEventCreate(&e1));
    // the operator as the iteration runs it: panel sweeps when panelized
    auto run = [&]() {
      if (which == 2) {
        if (kpan_.panels)
          launch_panel_spmv(kpan_.view, it_.x[st.ix_cur], it_.kx[1 - st.ikx_cur], stream_);
        else
          launch_spmv(K_, false, it_.x[st.ix_cur], it_.kx[1 - st.ikx_cur], parity(), stream_);
      } else {
        if (ktpan_.panels)
          launch_panel_spmv(ktpan_.view, it_.y[st.iy_cur], it_.kty[1 - st.ikty_cur], stream_);
        else
          launch_spmv(KT_, false, it_.y[st.iy_cur], it_.kty[1 - st.ikty_cur], parity(), stream_);
      }
    };
    run();
    PDLP_CUDA(cudaEventRecord(e0, stream_));
    for (int r = 0; r < reps; ++r) run();
    PDLP_CUDA(cudaEventRecord(e1, stream_));
    PDLP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PDLP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (avg_ms) *avg_ms = ms / reps;
    if (bytes) kernel_bytes(which, bytes, nullptr);
    state_valid_ = false;
    return;
  }
  reps = std::max(1, std::min(reps, tab_cap_));
  DevState& st = *hs_;
  st.failure = 0;
  st.window_accepts = 0;
  st.window_target = 1 << 30;
  st.table_base = st.total;
  st.record_log = 0;
  double* tab = tab_host_;
  for (int i = 0; i < reps; ++i) {
    const double kp1 = double(st.total + 1 + i) + 1.0;
    tab[2 * i] = 1.0 - std::pow(kp1, -params_.step_reduction_exponent);
    tab[2 * i + 1] = 1.0 + std::pow(kp1, -params_.step_growth_exponent);
  }
  PDLP_CUDA(cudaMemcpyAsync(state_dev_, hs_, xo_tab_ - xo_state_ + 2 * sizeof(double) * size_t(reps),
                            cudaMemcpyHostToDevice, stream_));
  // a trial needs a fresh x'; recompute it from the current point
  primal_step(kPRetry);
  std::vector<cudaEvent_t> ev(2 * reps);
  for (auto& e : ev) PDLP_CUDA(cudaEventCreate(&e));
  for (int r = 0; r < reps; ++r) {
    if (which == 0) PDLP_CUDA(cudaEventRecord(ev[2 * r], stream_));
    dual_step(0, 0);
    if (it_.decide_sep == 1) launch_decide(it_, stream_);
    if (which == 0) PDLP_CUDA(cudaEventRecord(ev[2 * r + 1], stream_));
    if (which == 1) PDLP_CUDA(cudaEventRecord(ev[2 * r], stream_));
    primal_step(-1);
    if (which == 1) PDLP_CUDA(cudaEventRecord(ev[2 * r + 1], stream_));
  }
  PDLP_CUDA(cudaStreamSynchronize(stream_));
  double total = 0.0;
  for (int r = 0; r < reps; ++r) {
    float ms = 0.f;
    PDLP_CUDA(cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]));
    total += ms;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  download_state();
  state_valid_ = false;
  if (avg_ms) *avg_ms = total / reps;
  if (bytes) kernel_bytes(which, bytes, nullptr);
}

// Bytes of one launch of kernel `which` (0 dual, 1 primal accept, 2 SpMV K x,
// 3 SpMV K^T y). `alg`: SURVEY.md §8(d)'s algorithmic figure (int32 index +
// fp64 value per nonzero, int32 row offsets, the gathered vector once, every
// dense stream once). `moved`: what the variant the iteration launches moves
// when each access reaches DRAM once: bounds only when not all [0, +inf),
// K'y' only when stored (not kty_lazy), and for column panels the per-panel
// row counts and block offsets instead of row offsets plus the running row
// sums (written by the first pass, read and written by the middle ones, read
// by the last).
void Solver::kernel_bytes(int which, double* alg, double* moved) const {
  const double nnz = double(nnz_), n = double(n_), m = double(m_);
  const bool dual_side = which == 0 || which == 2;
  const double rows = dual_side ? m : n, cols = dual_side ? n : m;
  const PanelOp& po = dual_side ? kpan_ : ktpan_;
  double a = 12.0 * nnz + 4.0 * (rows + 1) + 8.0 * cols;
  double mv = 12.0 * nnz + 8.0 * cols;
  if (po.panels) {
    const double P = po.panels;
    mv += P * double(po.view.rows_pad) + 4.0 * P * (po.view.nblk + 1) + 16.0 * rows * (P - 1.0);
  } else {
    mv += 4.0 * (rows + 1);
  }
  double dense_a = 0.0, dense_mv = 0.0;
  if (which == 0) {  // y, q, Kx read; y', Kx' write
    dense_a = dense_mv = 8.0 * 5.0 * m;
  } else if (which == 1) {  // x, c, l, u read; K'y', x' write; avg_x r+w; avg_y r+w, y read
    dense_a = 8.0 * 8.0 * n + 8.0 * 3.0 * m;
    const double nstreams = 5.0 + (it_.nonneg ? 0.0 : 2.0) + (it_.kty_lazy ? 0.0 : 1.0);
    dense_mv = 8.0 * nstreams * n + 8.0 * 3.0 * m;
  } else {  // plain SpMV: the output once
    dense_a = dense_mv = 8.0 * rows;
  }
  if (alg) *alg = a + dense_a;
  if (moved) *moved = mv + dense_mv;
}

void Solver::sizes(int64_t* out) const {
  out[0] = n_;
  out[1] = m_;
  out[2] = m1_;
  out[3] = nnz_;
}

// ---------------------------------------------------------------------------
// sharding: linking the ranks
// ---------------------------------------------------------------------------

LocalGroup::LocalGroup(int world) : world_(world), ev_(size_t(world), nullptr) {
  for (auto& e : ev_) PDLP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

LocalGroup::~LocalGroup() {
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
}

void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  const unsigned long long gen = gen_;
  if (++arrived_ == world_) {
    arrived_ = 0;
    ++gen_;
    cv_.notify_all();
    return;
  }
  if (!cv_.wait_for(lk, std::chrono::seconds(120), [&] { return gen_ != gen; }))
    throw std::runtime_error("shard group: a rank did not reach the barrier within 120 s");
}

void LocalGroup::phase(int rank, cudaStream_t s) {
  PDLP_CUDA(cudaEventRecord(ev_[size_t(rank)], s));
  barrier();
  for (int q = 0; q < world_; ++q)
    if (q != rank) PDLP_CUDA(cudaStreamWaitEvent(s, ev_[size_t(q)], 0));
  barrier();  // nobody records its next event before every peer enqueued its waits
}

void Solver::link_local(const std::vector<Solver*>& ranks) {
  const int world = int(ranks.size());
  if (world < 2) invalid("shard link: need at least two ranks");
  for (int q = 0; q < world; ++q) {
    const Solver* r = ranks[size_t(q)];
    if (!r) invalid("shard link: null handle");
    if (r->world_ != world || r->rank_ != q) invalid("shard link: handles must be ranks 0..world-1 in order");
    if (r->plan_hash_ != ranks[0]->plan_hash_) invalid("shard link: ranks were built from different instances");
  }
  auto group = std::make_shared<LocalGroup>(world);
  ShardView v{};
  for (int q = 0; q < world; ++q) {
    const Solver* r = ranks[size_t(q)];
    v.x_all[q] = r->x_all_.get();
    v.y_all[q] = r->y_all_.get();
    v.d_part[q] = r->d_part_.get();
    v.p_part[q] = r->p_part_.get();
    v.avg_x[q] = r->avg_x_.get();
    v.avg_y[q] = r->avg_y_.get();
    v.part1[q] = r->part1_.get();
    v.part2[q] = r->part2_.get();
    v.lam[q] = r->lam_.get();
    v.sync[q] = r->sync_.get();
  }
  for (int q = 0; q < world; ++q) {
    Solver* r = ranks[size_t(q)];
    PDLP_CUDA(cudaSetDevice(r->params_.device));
    r->shv_ = v;
    r->shard_view_upload();
    r->group_ = group;
    cudaStream_t st = r->stream_;
    LocalGroup* g = group.get();
    r->phase_ = [g, q, st] { g->phase(q, st); };
    // host-ordered launches: the per-launch phases need the stream engine
    r->engine_ = PDLP_ENGINE_STREAM;
    r->linked_ = true;
  }
}

void Solver::export_shard(ShardBlob* out) const {
  if (world_ < 2) invalid("shard export: not a sharded handle (world_size 1)");
  ShardBlob b{};
  b.magic = 0x50444c50u;  // "PDLP"
  b.rank = rank_;
  b.world = world_;
  b.device = params_.device;
  b.n = n_, b.m = m_, b.nnz = nnz_;
  b.plan_hash = plan_hash_;
  const void* bufs[10] = {x_all_.get(), y_all_.get(), d_part_.get(), p_part_.get(), avg_x_.get(),
                          avg_y_.get(), part1_.get(), part2_.get(), lam_.get(), sync_.get()};
  PDLP_CUDA(cudaSetDevice(params_.device));
  for (int i = 0; i < 10; ++i) PDLP_CUDA(cudaIpcGetMemHandle(&b.h[i], const_cast<void*>(bufs[i])));
  *out = b;
}

void Solver::import_shards(const ShardBlob* blobs, int world) {
  if (world != world_) invalid("shard import: world size differs from this handle's");
  PDLP_CUDA(cudaSetDevice(params_.device));
  ShardView v = shv_;
  for (int q = 0; q < world; ++q) {
    const ShardBlob& b = blobs[q];
    if (b.magic != 0x50444c50u || b.rank != q || b.world != world)
      invalid("shard import: blobs must be every rank's export, in rank order");
    if (b.plan_hash != plan_hash_ || b.n != n_ || b.m != m_ || b.nnz != nnz_)
      invalid("shard import: ranks were built from different instances or partitions");
    if (q == rank_) continue;
    void* p[10];
    for (int i = 0; i < 10; ++i) {
      PDLP_CUDA(cudaIpcOpenMemHandle(&p[i], b.h[i], cudaIpcMemLazyEnablePeerAccess));
      ipc_opened_.push_back(p[i]);
    }
    v.x_all[q] = static_cast<double*>(p[0]);
    v.y_all[q] = static_cast<double*>(p[1]);
    v.d_part[q] = static_cast<double*>(p[2]);
    v.p_part[q] = static_cast<double*>(p[3]);
    v.avg_x[q] = static_cast<double*>(p[4]);
    v.avg_y[q] = static_cast<double*>(p[5]);
    v.part1[q] = static_cast<double*>(p[6]);
    v.part2[q] = static_cast<double*>(p[7]);
    v.lam[q] = static_cast<double*>(p[8]);
    v.sync[q] = static_cast<ShardSync*>(p[9]);
  }
  shv_ = v;
  shard_view_upload();
  linked_ = true;  // in-kernel flag barriers order the ranks
}

// Per-rank operator storage: copies this rank's rows of K (rows [k_cuts_[r],
// k_cuts_[r+1])) and of K^T (rows [kt_cuts_[r], kt_cuts_[r+1])) into compact
// arrays and frees the full ones. The device views keep global row and entry
// indices (the tiles store them): their pointers are the compact arrays offset
// by the first own row / entry, so every kernel runs unchanged on own tiles.
void Solver::compact_own_rows() {
  cudaStream_t s = stream_;
  auto compact = [&](DevBuf<int>& rp, DevBuf<int>& col, DevBuf<double>& val, DevBuf<double>& val_orig,
                     int64_t r0, int64_t r1, std::initializer_list<DevCsr*> views) {
    // the kernels' vector loads need the global alignment: starts rounded
    // down to a multiple of 8 rows / entries
    int k01[3] = {0, 0, 0};
    PDLP_CUDA(cudaMemcpyAsync(&k01[2], rp.get() + r0, sizeof(int), cudaMemcpyDeviceToHost, s));
    r0 &= ~int64_t(7);
    PDLP_CUDA(cudaMemcpyAsync(&k01[0], rp.get() + r0, sizeof(int), cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaMemcpyAsync(&k01[1], rp.get() + r1, sizeof(int), cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
    const int64_t k0 = int64_t(k01[0]) & ~int64_t(7), k1 = k01[1], rows = r1 - r0, nz = k1 - k0;
    const int64_t own = k1 - k01[2];  // entries of the own rows (the copy starts a few earlier)
    DevBuf<int> rp_o(size_t(rows + 1) + kVecPad), col_o(size_t(nz) + kVecPad);
    DevBuf<double> val_o(size_t(nz) + kVecPad), vor_o(size_t(nz) + kVecPad);
    rp_o.zero(s);
    col_o.zero(s);
    val_o.zero(s);
    vor_o.zero(s);
    PDLP_CUDA(cudaMemcpyAsync(rp_o.get(), rp.get() + r0, size_t(rows + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (nz) {
      PDLP_CUDA(cudaMemcpyAsync(col_o.get(), col.get() + k0, size_t(nz) * sizeof(int), cudaMemcpyDeviceToDevice, s));
      PDLP_CUDA(cudaMemcpyAsync(val_o.get(), val.get() + k0, size_t(nz) * sizeof(double), cudaMemcpyDeviceToDevice, s));
      PDLP_CUDA(cudaMemcpyAsync(vor_o.get(), val_orig.get() + k0, size_t(nz) * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    }
    PDLP_CUDA(cudaStreamSynchronize(s));
    rp = std::move(rp_o);
    col = std::move(col_o);
    val = std::move(val_o);
    val_orig = std::move(vor_o);
    for (DevCsr* v : views) {
      v->rp = rp.get() - r0;
      v->col = col.get() - k0;
      v->val = val.get() - k0;
      v->val_orig = val_orig.get() - k0;
    }
    return own;
  };
  const int64_t own_k = compact(k_rp_, k_col_, k_val_, k_val_orig_, k_cuts_[rank_], k_cuts_[rank_ + 1],
                                {&K_, &K_full_, &k_it_.csr, &k_ev_.csr});
  const int64_t own_kt = compact(kt_rp_, kt_col_, kt_val_, kt_val_orig_, kt_cuts_[rank_], kt_cuts_[rank_ + 1],
                                 {&KT_, &KT_full_, &kt_it_.csr, &kt_ev_.csr});
  own_nnz_[0] = own_k;
  own_nnz_[1] = own_kt;
  compacted_ = true;
}

void Solver::shard_info(int64_t* out) const {
  out[0] = world_;
  out[1] = rank_;
  out[2] = k_cuts_[size_t(rank_)];
  out[3] = k_cuts_[size_t(rank_) + 1];
  out[4] = kt_cuts_[size_t(rank_)];
  out[5] = kt_cuts_[size_t(rank_) + 1];
  out[6] = K_.ntiles;
  out[7] = KT_.ntiles;
  out[8] = int64_t(k_it_.plan.tiles.size());
  out[9] = int64_t(kt_it_.plan.tiles.size());
}

// pdhg_raw_step (solver.hpp:335-358) from (x, y) on the unscaled saddle
// problem to_saddle(lp) (original values of K, c, l, u, q): K'y, the primal
// half with the extrapolation, K ext, the dual half. Parity mode sums every
// row sequentially (bitwise with the reference); fast mode uses the tiled
// engine's reduction order.
void Solver::pdhg_raw_step(const double* x, const double* y, double tau, double sigma, double* xo, double* yo) {
  if (world_ > 1) throw std::logic_error("pdhg_raw_step: single-device handles only");
  if (!(tau > 0.0) || !(sigma > 0.0) || !std::isfinite(tau) || !std::isfinite(sigma))
    invalid("pdhg_raw_step: tau and sigma must be positive and finite");
  PDLP_CUDA(cudaSetDevice(params_.device));
  cudaStream_t s = stream_;
  DevBuf<double> dx(n_), dy(m_), kty(n_), ext(n_), kext(m_), dxo(n_), dyo(m_);
  if (n_) PDLP_CUDA(cudaMemcpyAsync(dx.get(), x, n_ * sizeof(double), cudaMemcpyHostToDevice, s));
  if (m_) PDLP_CUDA(cudaMemcpyAsync(dy.get(), y, m_ * sizeof(double), cudaMemcpyHostToDevice, s));
  if (n_) launch_fill(kty.get(), n_, 0.0, s);
  launch_spmv(KT_, true, dy.get(), kty.get(), parity(), s);  // spmv_transpose, solver.hpp:341
  launch_raw_primal(dx.get(), kty.get(), c_orig_.get(), l_orig_.get(), u_orig_.get(), tau, n_, dxo.get(), ext.get(),
                    s);
  if (m_) launch_fill(kext.get(), m_, 0.0, s);
  launch_spmv(K_, true, ext.get(), kext.get(), parity(), s);  // spmv, solver.hpp:352
  launch_raw_dual(dy.get(), kext.get(), q_orig_.get(), sigma, m_, m1_, dyo.get(), s);
  if (n_) PDLP_CUDA(cudaMemcpyAsync(xo, dxo.get(), n_ * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (m_) PDLP_CUDA(cudaMemcpyAsync(yo, dyo.get(), m_ * sizeof(double), cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  launches_ += 4;
}

void Solver::shard_exchange(int64_t* out) const {
  out[0] = push_values_;
  out[1] = push_values_full_;
  out[2] = compacted_ ? own_nnz_[0] : nnz_;  // stored nonzeros of K on this rank
  out[3] = compacted_ ? own_nnz_[1] : nnz_;  // ... and of K^T
}

}  // namespace pdlp
