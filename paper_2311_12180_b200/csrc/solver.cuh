// solver.cuh — host runtime of the B200 restarted-PDHG solver (one handle).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <future>
#include <vector>

#include "../../include/pdlp_b200.h"
#include "common.cuh"
#include "device_state.h"
#include "kernels.cuh"
#include "tiles.h"

namespace pdlp {

// GeneralFormLp::validate plus the C ABI's raw-array checks (host only).
void validate_lp(const pdlp_lp& lp);


template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), ipc_(o.ipc_) { o.p_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      ipc_ = o.ipc_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  // Device memory comes from the device's stream-ordered pool (kept across
  // handles: creating and destroying a solver does not round-trip through the
  // driver's allocator); `ipc` buffers (exported to peer processes) use
  // cudaMalloc, which CUDA IPC requires.
  void alloc(size_t n, bool ipc = false) {
    release();
    n_ = n;
    ipc_ = ipc;
    const size_t bytes = (n ? n : 1) * sizeof(T);
    if (ipc) {
      PDLP_CUDA(cudaMalloc(&p_, bytes));
    } else {
      PDLP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), bytes, cudaStreamPerThread));
      PDLP_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
    }
  }
  void zero(cudaStream_t s) { PDLP_CUDA(cudaMemsetAsync(p_, 0, (n_ ? n_ : 1) * sizeof(T), s)); }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  void release() {
    if (p_) {
      if (ipc_)
        cudaFree(p_);
      else
        cudaFreeAsync(p_, cudaStreamPerThread);
    }
    p_ = nullptr;
  }
  T* p_ = nullptr;
  size_t n_ = 0;
  bool ipc_ = false;
};

// Page-locked host memory from a process-wide pool: cudaMallocHost costs
// milliseconds per call, so result buffers are recycled across solver handles.
void* pinned_pool_get(size_t bytes, size_t* capacity);
void pinned_pool_put(void* p, size_t capacity);

// A resizable page-locked double array (the solve's result vectors: the D2H of
// x, y and lambda at full PCIe rate instead of the pageable staging path).
class PinnedVec {
 public:
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  ~PinnedVec() {
    if (p_) pinned_pool_put(p_, cap_);
  }
  void resize(size_t n) {  // contents unspecified (the caller overwrites them)
    if (n * sizeof(double) > cap_ || !p_) {
      if (p_) pinned_pool_put(p_, cap_);
      p_ = static_cast<double*>(pinned_pool_get(std::max<size_t>(n, 1) * sizeof(double), &cap_));
    }
    n_ = n;
  }
  void assign(size_t n, double v) {
    resize(n);
    std::fill(p_, p_ + n, v);
  }
  double* data() const { return p_; }
  size_t size() const { return n_; }
  double* begin() const { return p_; }
  double* end() const { return p_ + n_; }
  double& operator[](size_t i) const { return p_[i]; }

 private:
  double* p_ = nullptr;
  size_t n_ = 0, cap_ = 0;
};

template <class T>
class PinnedBuf {
 public:
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p_) cudaFreeHost(p_);
  }
  void alloc(size_t n) {
    if (p_) cudaFreeHost(p_);
    PDLP_CUDA(cudaMallocHost(&p_, (n ? n : 1) * sizeof(T)));
    n_ = n;
  }
  T* get() const { return p_; }
  T& operator[](size_t i) const { return p_[i]; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

struct KktHost {  // KktResiduals (solver.hpp:109-123)
  double prn, drn, pobj, dobj;
  double gap() const { return dobj - pobj; }
  double weighted(double omega) const;
};

// Ranks of one sharded solve living in ONE process (the loopback transport:
// every rank on its own stream, usually the same device). After each launch
// whose outputs peers consume, every rank records an event, meets the others
// at a host barrier and makes its stream wait on every peer's event, so no
// consumer kernel ever starts (and spins) before its producers finished.
class LocalGroup {
 public:
  explicit LocalGroup(int world);
  ~LocalGroup();
  void phase(int rank, cudaStream_t s);
  int world() const { return world_; }

 private:
  void barrier();
  int world_;
  std::vector<cudaEvent_t> ev_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  unsigned long long gen_ = 0;
};

// Exported view of one rank's exchanged buffers (CUDA IPC handles).
struct ShardBlob {
  uint32_t magic;
  int32_t rank, world;
  int32_t device;
  int64_t n, m, nnz;
  uint64_t plan_hash;
  cudaIpcMemHandle_t h[10];  // x_all y_all d_part p_part avg_x avg_y part1 part2 lam sync
};

class Solver {
 public:
  Solver(const pdlp_lp& lp, const pdlp_params& params);
  ~Solver();

  void solve(pdlp_result_info* info);
  void iterate_begin(int32_t* status);
  void iterate_run(int64_t n, int32_t* status);
  void get_iterate(double* x, double* y, double* kx, double* kty, int64_t* counters,
                   double* scalars);
  void get_solution(double* x, double* y, double* lambda, double* lambda_pos, double* lambda_neg);
  int64_t get_step_log(pdlp_step_log_entry* out, int64_t cap) const;
  int64_t get_restart_log(pdlp_restart_event* out, int64_t cap) const;
  void get_scaling(double* row_scale, double* col_scale) const;
  void spmv(int op, const double* in, double* out);
  void time_kernel(int which, int reps, double* avg_ms, double* bytes);
  void kernel_bytes(int which, double* alg, double* moved) const;
  int panels(int op) const { return op == 0 ? kpan_.panels : ktpan_.panels; }
  void sizes(int64_t* out) const;
  void shard_exchange(int64_t* out) const;
  void pdhg_raw_step(const double* x, const double* y, double tau, double sigma, double* xo, double* yo);
  // ---- sharding ----
  static void link_local(const std::vector<Solver*>& ranks);
  void export_shard(ShardBlob* out) const;
  void import_shards(const ShardBlob* blobs, int world);
  void shard_info(int64_t* out) const;
  const pdlp_result_info& info() const { return info_; }

 private:
  void setup(const pdlp_lp& lp);
  void build_transpose();
  void precondition();
  struct OpPlan {
    TilePlan plan;
    DevBuf<Tile> tiles;
    DevBuf<double> chunk;
    DevBuf<unsigned> ctr;
    DevCsr csr{};
  };
  // rp: host copy of the operator's rows + 1 row offsets
  void build_plan(OpPlan& p, const DevCsr& base, const int* rp, int64_t rows, const TileGeom& g,
                  const std::vector<int64_t>& breaks, int64_t r0, int64_t r1,
                  const std::vector<uint8_t>* contig = nullptr);
  void shard_view_upload();
  // column panels of one operator (panels.cu): panel-major entries, per-panel
  // row counts and block offsets, running row sums
  struct PanelOp {
    int panels = 0;  // 0: not panelized
    int width = 0;
    DevBuf<int> col, boff;
    DevBuf<double> val, acc;
    DevBuf<unsigned char> cnt;
    PanelView view{};
  };
  void build_panels(PanelOp& po, const DevCsr& op, int rows, int cols, const char* which);
  void dual_step(unsigned long long cond, int use_cond);
  void primal_step(int mode_override, unsigned long long cond = 0, int use_cond = 0);
  void phase() {
    if (phase_) phase_();
  }
  void require_linked() const;
  void allocate_iteration();
  void pin_iterates_in_l2();
  void capture_window_graph();
  void capture_chain_graph();
  bool chain_enabled() const;
  bool run_chain(int windows);  // true: the last evaluation was decided on the device
  void upload_state();
  void download_state();
  void spin_sync();
  void run_window(int target);
  void evaluate();
  KktHost kkt(int slot) const;
  bool terminated(const KktHost& r) const;
  void evaluation_block();
  void finish(int status, int slot_x, int slot_y, int slot_lam, const KktHost& r,
              const std::string& msg = {});
  void finish_candidate(int status, const std::string& msg = {});
  double elapsed() const;
  bool parity() const { return params_.mode == PDLP_MODE_PARITY; }

  pdlp_params params_;
  cudaStream_t stream_ = nullptr;
  int64_t n_ = 0, m_ = 0, m1_ = 0, m2_ = 0, nnz_ = 0;
  double objective_constant_ = 0.0;

  // host copies of the original vectors (evaluation bookkeeping is host-side)
  // the caller's objective, bounds and right-hand sides: read during
  // pdlp_create only (setup), never kept
  const double *hc_ = nullptr, *hl_ = nullptr, *hu_ = nullptr, *hh_ = nullptr, *hb_ = nullptr;
  double hq(int64_t i) const { return i < m1_ ? hh_[i] : hb_[i - m1_]; }
  PinnedVec d1_, d2_;  // the scaling, downloaded once at setup
  double rhs_norm_ = 0.0, obj_norm_ = 0.0;  // termination_norms (solver.hpp:157-163)
  double eta_hat0_ = 1.0, omega0_ = 1.0;

  // operator storage: K = (G; A) and its separately stored transpose
  DevBuf<int> k_rp_, k_col_, kt_rp_, kt_col_;
  DevBuf<double> k_val_, k_val_orig_, kt_val_, kt_val_orig_;
  OpPlan k_it_, kt_it_, k_ev_, kt_ev_;
  PanelOp kpan_, ktpan_;
  DevCsr K_{}, KT_{};  // the iteration-kernel tilings (this rank's tiles)
  DevCsr K_full_{}, KT_full_{};  // every tile (kernel-level API on a sharded rank)

  // vectors
  DevBuf<double> c_orig_, l_orig_, u_orig_, q_orig_, d1_dev_, d2_dev_;
  DevBuf<double> c_s_, l_s_, u_s_, q_s_;
  DevBuf<double> x_all_, y_all_;  // the three x (3 n) and y (3 m) rotation buffers
  DevBuf<double> kx_[2], kty_[2], avg_x_, avg_y_, x_start_, y_start_;
  DevBuf<double> d_part_, p_part_, seq_dy2_, seq_inter_, seq_dx2_;
  // one transfer block per window round trip: [EvalOut | DevState | factor pairs]
  DevBuf<unsigned char> xfer_dev_;
  PinnedBuf<unsigned char> xfer_host_;
  size_t xo_state_ = 0, xo_tab_ = 0;
  DevBuf<pdlp_step_log_entry> step_log_dev_;
  DevState* state_dev_ = nullptr;  // inside xfer_dev_
  DevBuf<DevState> snap_dev_;
  DevBuf<double> eval_stage_;
  DevBuf<double> X4_, Y4_, lam_, part0_, part1_, part2_, seq_r_, seq_d_, scratch_n_, scratch_m_;
  EvalOut* eval_dev_ = nullptr;  // inside xfer_dev_
  DevIter it_{};
  DevEval ev_{};
  int tab_cap_ = 0;

  DevState* hs_ = nullptr;   // pinned, inside xfer_host_
  EvalOut* he_ = nullptr;
  double* tab_host_ = nullptr;
  PinnedBuf<pdlp_step_log_entry> log_host_;

  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  unsigned long long cond_handle_ = 0;
  // chained windows: WHILE(chain) { WHILE(window) { dual; primal }; evaluation; decision }
  cudaGraph_t chain_graph_ = nullptr;
  cudaGraphExec_t chain_exec_ = nullptr;
  int chain_windows_ = 0;  // windows per chain launch (0: chaining off)
  double window_time_est_ = 0.0;  // measured seconds per window (bounds a chain by the time limit)

  // host-side loop state (solver.hpp:683-698)
  int64_t outer_ = 0;
  double kkt_epoch_start_ = 0.0, kkt_last_ = 0.0;
  std::chrono::steady_clock::time_point t0_;
  bool begun_ = false, finished_ = false, state_valid_ = false;
  int64_t launches_ = 0, evaluations_ = 0;
  double setup_seconds_ = 0.0;
  cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr, ev_w0_ = nullptr, ev_w1_ = nullptr;
  double window_seconds_ = 0.0, eval_seconds_ = 0.0;
  cudaEvent_t ev_e1_ = nullptr;
  EvalFork fork_{};  // side stream for the concurrent evaluation passes
  int engine_ = PDLP_ENGINE_GRAPH;
  bool eval_fresh_ = false;  // EvalOut on the host matches the device state
  std::vector<pdlp_step_log_entry> step_log_;
  std::vector<pdlp_restart_event> restart_log_;
  pdlp_result_info info_{};
  PinnedVec rx_, ry_, rlam_;

  // ---- sharding (world_ == 1: a single device) ----
  int64_t l2_window_bytes_ = 0;  // persisting L2 carve-out for the gathered iterate
  int world_ = 1, rank_ = 0;
  std::vector<int64_t> k_cuts_, kt_cuts_;  // world + 1 row boundaries of K and K^T
  DevBuf<unsigned> xmask_, ymask_;          // gather masks of x' / y' (sharded)
  int64_t push_values_ = 0, push_values_full_ = 0;  // values pushed per trial: masked / every peer
  bool compacted_ = false;                          // sharded rank holding only its own operator rows
  int64_t own_nnz_[2] = {0, 0};
  void compact_own_rows();
  uint64_t plan_hash_ = 0;
  DevBuf<ShardSync> sync_;
  DevBuf<ShardView> shv_dev_;
  ShardView shv_{};
  bool linked_ = false;
  std::shared_ptr<LocalGroup> group_;
  PhaseFn phase_;
  std::vector<void*> ipc_opened_;
  // initialize_primal_weight's host sums (setup); declared last so that it
  // is destroyed (joined) before the members it reads
  std::future<void> omega_job_;
};

}  // namespace pdlp
