// standard_form.cu — the standard-form theory harness on the GPU
// (standard_form.hpp:36-211): fixed-step
// restarted PDHG with uniform averaging for min c'x s.t. Ax = b, x >= 0,
// restarting to the average once KKT(avg) <= beta * KKT(epoch start), plus
// the KKT error, the spectral norm by power iteration and the P_s norm.
//
// A and A' are resident with tile plans and run through the same tiled SpMV
// engine as the solver (launch_spmv). Every iteration is five kernels plus the
// two SpMVs of the average's KKT error; the restart / convergence / limit
// decision is taken on the device by a one-CTA kernel, so the host only polls
// a small state block every kPoll iterations (launches after a stop are
// no-ops).
//
// Parity mode (pdlp_standard_options::parity): sequential row sums and
// sequential scalar sums in the reference's order, built with --fmad=false,
// so the trace (epoch KKT values, lengths) and the final point are bitwise
// those of restarted_pdhg_standard. Fast mode: tiled rows and tree sums.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pdlp_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "spmv_engine.cuh"
#include "tiles.h"

namespace pdlp {
void set_last_error(const std::string& msg);  // capi.cu

namespace {

constexpr int kPoll = 32;          // iterations between host polls
constexpr int kRedBlocks = 148;    // fast-mode reduction blocks (one wave)

template <class T>
struct Buf {
  T* p = nullptr;
  size_t n = 0;
  Buf() = default;
  explicit Buf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    n = count;
    PDLP_CUDA(cudaMalloc(&p, (count ? count : 1) * sizeof(T)));
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

// One operator (A or A') with its tile plan, ready for launch_spmv.
struct Op {
  Buf<int> rp, col;
  Buf<double> val;
  Buf<Tile> tiles;
  Buf<double> chunk;
  Buf<unsigned> ctr;
  DevCsr d{};

  void upload(int rows, int cols, const std::vector<int>& hrp, const std::vector<int>& hcol,
              const std::vector<double>& hval, bool parity, cudaStream_t s) {
    const int64_t nnz = hrp.back();
    rp.alloc(hrp.size() + kVecPad);
    col.alloc(size_t(nnz) + kVecPad);
    val.alloc(size_t(nnz) + kVecPad);
    PDLP_CUDA(cudaMemsetAsync(col.p, 0, (size_t(nnz) + kVecPad) * sizeof(int), s));
    PDLP_CUDA(cudaMemsetAsync(val.p, 0, (size_t(nnz) + kVecPad) * sizeof(double), s));
    PDLP_CUDA(cudaMemcpyAsync(rp.p, hrp.data(), hrp.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    if (nnz) {
      PDLP_CUDA(cudaMemcpyAsync(col.p, hcol.data(), size_t(nnz) * sizeof(int), cudaMemcpyHostToDevice, s));
      PDLP_CUDA(cudaMemcpyAsync(val.p, hval.data(), size_t(nnz) * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    const TileGeom g = kIterGeom;
    const TilePlan plan = plan_tiles<int>(rows, hrp.data(), parity, std::min(kStreamMaxRow, g.stream_nnz),
                                          std::min(kWarpMaxRow, g.lane_nnz * kThreads), g.chunk_nnz, g.stream_nnz,
                                          g.stream_rows, kThreads, g.lane_nnz);
    tiles.alloc(plan.tiles.size());
    if (!plan.tiles.empty())
      PDLP_CUDA(cudaMemcpyAsync(tiles.p, plan.tiles.data(), plan.tiles.size() * sizeof(Tile),
                                cudaMemcpyHostToDevice, s));
    chunk.alloc(size_t(std::max(1, plan.chunk_slots)) * 8);
    ctr.alloc(size_t(std::max(1, plan.split_rows)));
    PDLP_CUDA(cudaMemsetAsync(ctr.p, 0, ctr.n * sizeof(unsigned), s));
    d.rp = rp.p;
    d.col = col.p;
    d.val = val.p;
    d.val_orig = val.p;
    d.rows = rows;
    d.cols = cols;
    d.nnz = nnz;
    d.tiles = tiles.p;
    d.ntiles = int(plan.tiles.size());
    d.tile0 = 0;
    d.chunk_slots = plan.chunk_slots;
    d.chunk_part = chunk.p;
    d.chunk_ctr = ctr.p;
  }
};

// A (int64 CSR from the caller) and its transpose, built on the host by a
// stable counting sort (row order inside each column, i.e. the summation order
// of spmv_transpose's scatter, sparse_matrix.hpp:142-158).
struct Operators {
  Op a, at;
  int m = 0, n = 0;
  Operators(const pdlp_csr& A, bool parity, cudaStream_t s) {
    if (A.num_rows < 0 || A.num_cols < 0 || A.num_rows > INT32_MAX || A.num_cols > INT32_MAX ||
        A.nnz > INT32_MAX)
      throw std::invalid_argument("standard-form lp: matrix too large for 32-bit indices");
    m = int(A.num_rows);
    n = int(A.num_cols);
    std::vector<int> rp(size_t(m) + 1), col(size_t(A.nnz)), trp(size_t(n) + 1, 0), tcol(size_t(A.nnz));
    std::vector<double> val(A.values, A.values + A.nnz), tval(size_t(A.nnz));
    for (int64_t i = 0; i <= m; ++i) rp[size_t(i)] = int(A.row_offsets[i]);
    if (rp[0] != 0 || rp[size_t(m)] != A.nnz) throw std::invalid_argument("standard-form lp: bad row offsets");
    for (int64_t k = 0; k < A.nnz; ++k) {
      const int64_t c = A.col_indices ? A.col_indices[k] : int64_t(A.col_indices32[k]);
      if (c < 0 || c >= n) throw std::invalid_argument("standard-form lp: column index out of range");
      col[size_t(k)] = int(c);
      ++trp[size_t(c) + 1];
    }
    for (int j = 0; j < n; ++j) trp[size_t(j) + 1] += trp[size_t(j)];
    std::vector<int> fill(trp.begin(), trp.end() - 1);
    for (int r = 0; r < m; ++r)
      for (int k = rp[size_t(r)]; k < rp[size_t(r) + 1]; ++k) {
        const int dst = fill[size_t(col[size_t(k)])]++;
        tcol[size_t(dst)] = r;
        tval[size_t(dst)] = val[size_t(k)];
      }
    a.upload(m, n, rp, col, val, parity, s);
    at.upload(n, m, trp, tcol, tval, parity, s);
  }
};

// Device-side state of the restarted loop (one block, host-polled).
struct SfState {
  int64_t total;       // total inner iterations
  int64_t inner;       // iterations of the current epoch
  int64_t epochs;      // epochs opened so far
  int64_t limit;
  int32_t stop;        // 1 = converged / limit / failure: later launches are no-ops
  int32_t converged;
  int32_t failure;
  int32_t bad;         // non-finite flag of the current trial (integer OR: order-free)
  double start_kkt;    // KKT of the current epoch's start
  double decay, tol, step;
};

// ---------------------------------------------------------------------------
// Reductions: parity = one thread, reference order; fast = fixed tree.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum1(double v) {
  __shared__ double sh[kWarps];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kWarps; ++w) t += sh[w];
  return t;  // valid in thread 0
}

// KKT terms of (x, y) given Ax and A'y: the five sums of kkt_error_standard
// (standard_form.hpp:37-58): sum (Ax-b)^2, sum max(-x,0)^2, sum max(A'y-c,0)^2,
// c'x, b'y. Fast mode: per-block partials [5][kRedBlocks].
__global__ void kkt_partials_kernel(const double* ax, const double* b, const double* x, const double* aty,
                                    const double* c, const double* y, int m, int n, double* part) {
  double t[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const double r = ax[i] - b[i];
    t[0] += r * r;
    t[4] += b[i] * y[i];
  }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const double r1 = smax(-x[j], 0.0);
    t[1] += r1 * r1;
    const double r2 = smax(aty[j] - c[j], 0.0);
    t[2] += r2 * r2;
    t[3] += c[j] * x[j];
  }
  for (int k = 0; k < 5; ++k) {
    const double s = block_sum1(t[k]);
    if (threadIdx.x == 0) part[k * gridDim.x + blockIdx.x] = s;
  }
}

__device__ double kkt_from_partials(const double* part, int nb) {
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < 5; ++k)
    for (int i = 0; i < nb; ++i) s[k] += part[k * nb + i];
  const double gap = smax(s[3] - s[4], 0.0);
  double sum = s[0] + s[1];
  sum += s[2];
  sum += gap * gap;
  return sqrt(sum);
}

// the reference's exact order: one running sum over the m, n, n terms, then gap^2
__device__ double kkt_sequential(const double* ax, const double* b, const double* x, const double* aty,
                                 const double* c, const double* y, int m, int n) {
  double sum = 0.0;
  for (int i = 0; i < m; ++i) {
    const double r = ax[i] - b[i];
    sum += r * r;
  }
  for (int j = 0; j < n; ++j) {
    const double r = smax(-x[j], 0.0);
    sum += r * r;
  }
  for (int j = 0; j < n; ++j) {
    const double r = smax(aty[j] - c[j], 0.0);
    sum += r * r;
  }
  double cx = 0.0, by = 0.0;
  for (int j = 0; j < n; ++j) cx += c[j] * x[j];
  for (int i = 0; i < m; ++i) by += b[i] * y[i];
  const double gap = smax(cx - by, 0.0);
  sum += gap * gap;
  return sqrt(sum);
}

// ---------------------------------------------------------------------------
// The inner iteration (standard_form.hpp:163-186)
// ---------------------------------------------------------------------------
// x+ = max(x - s (c - A'y), 0), extrapolated = 2 x+ - x
__global__ void sf_primal_kernel(SfState* st, const double* x, const double* c, const double* aty, double* xn,
                                 double* ext, int n) {
  if (st->stop) return;
  const double s = st->step;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double v = smax(x[j] - s * (c[j] - aty[j]), 0.0);
    xn[j] = v;
    ext[j] = 2.0 * v - x[j];
    if (!isfinite(v)) st->bad = 1;
  }
}

// y+ = y + s (b - A ext)
__global__ void sf_dual_kernel(SfState* st, const double* y, const double* b, const double* aext, double* yn,
                               int m) {
  if (st->stop) return;
  const double s = st->step;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const double v = y[i] + s * (b[i] - aext[i]);
    yn[i] = v;
    if (!isfinite(v)) st->bad = 1;
  }
}

// z = z+ and the uniform running averages (w = 1 / inner), or a numerical
// failure when any entry of z+ is not finite (all_finite, vector_ops.hpp:74-79)
// (record_iterates: z+ also into row `total` of the iterate log)
__global__ void sf_commit_kernel(SfState* st, double* x, double* y, const double* xn, const double* yn,
                                 double* xa, double* ya, int n, int m, double* log_x, double* log_y,
                                 int64_t log_cap) {
  if (st->stop || st->bad) return;
  const double w = 1.0 / double(st->inner + 1);
  const int64_t k = st->total;
  double* lx = k < log_cap ? log_x + k * n : nullptr;
  double* ly = k < log_cap ? log_y + k * m : nullptr;
  const int stride = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    x[j] = xn[j];
    xa[j] += w * (xn[j] - xa[j]);
    if (lx) lx[j] = xn[j];
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    y[i] = yn[i];
    ya[i] += w * (yn[i] - ya[i]);
    if (ly) ly[i] = yn[i];
  }
}

// Restart test on the average (standard_form.hpp:191-199) by one CTA; the
// epoch log gets (start KKT, length).
__global__ void sf_decide_kernel(SfState* st, const double* part, int nb, const double* ax, const double* b,
                                 const double* xa, const double* aty, const double* c, const double* ya, int m,
                                 int n, int seq, double* ep_kkt, int64_t* ep_len, int64_t cap, int* restart) {
  if (st->stop) {
    if (threadIdx.x == 0) *restart = 0;
    return;
  }
  double kkt = 0.0;
  if (seq) {
    if (threadIdx.x == 0 && !st->bad) kkt = kkt_sequential(ax, b, xa, aty, c, ya, m, n);
  } else if (threadIdx.x == 0 && !st->bad) {
    kkt = kkt_from_partials(part, nb);
  }
  if (threadIdx.x != 0) return;
  *restart = 0;
  if (st->bad) {  // numerical failure: the trial is dropped, the loop ends
    st->failure = 1;
    st->stop = 1;
    return;
  }
  st->inner += 1;
  st->total += 1;
  if (kkt <= st->decay * st->start_kkt) {
    const int64_t e = st->epochs - 1;
    if (e >= 0 && e < cap) ep_len[e] = st->inner;
    // open_epoch(avg): its KKT is the one just computed from the same vectors
    if (st->epochs < cap) ep_kkt[st->epochs] = kkt;
    st->epochs += 1;
    st->start_kkt = kkt;
    st->inner = 0;
    *restart = 1;
  }
  // the loop head: the limit first, then the epoch-start KKT (standard_form.hpp:157-162)
  if (st->total >= st->limit) {
    st->stop = 1;
  } else if (st->start_kkt <= st->tol) {
    st->converged = 1;
    st->stop = 1;
  }
}

// on restart: z = epoch start = avg, averages zeroed
__global__ void sf_restart_kernel(const int* restart, double* x, double* y, double* xs, double* ys, double* xa,
                                  double* ya, int n, int m) {
  if (!*restart) return;
  const int stride = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    x[j] = xa[j];
    xs[j] = xa[j];
    xa[j] = 0.0;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    y[i] = ya[i];
    ys[i] = ya[i];
    ya[i] = 0.0;
  }
}

// KKT of the starting point (open_epoch(z) at the top of the loop)
__global__ void sf_open_kernel(SfState* st, const double* part, int nb, const double* ax, const double* b,
                               const double* x, const double* aty, const double* c, const double* y, int m, int n,
                               int seq, double* ep_kkt, int64_t cap) {
  if (threadIdx.x != 0) return;
  const double kkt = seq ? kkt_sequential(ax, b, x, aty, c, y, m, n) : kkt_from_partials(part, nb);
  st->start_kkt = kkt;
  if (cap > 0) ep_kkt[0] = kkt;
  st->epochs = 1;
  if (st->total >= st->limit) {
    st->stop = 1;
  } else if (kkt <= st->tol) {
    st->converged = 1;
    st->stop = 1;
  }
}

__global__ void zero_int_kernel(int32_t* p) { *p = 0; }

// ---- spectral_norm (standard_form.hpp:63-89): power iteration on A'A ----
struct PowerState {
  double lambda;
  double next;
  int64_t it;
  int64_t max_it;
  double tol;
  int32_t stop;
};

// sum of squares of v: one thread in order (parity) or a fixed tree (fast)
__device__ double sum_squares(const double* v, int n, bool seq) {
  if (seq) {
    double s = 0.0;
    if (threadIdx.x == 0)
      for (int i = 0; i < n; ++i) s += v[i] * v[i];
    return s;
  }
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += v[i] * v[i];
  return block_sum1(t);
}

// next = norm2(A'A v); v = A'A v / next, or a basis kick when it vanished
__global__ void power_step_kernel(PowerState* ps, const double* atav, double* v, int n, int seq) {
  __shared__ double s_next;
  __shared__ int s_act;  // 0 = stopped, 1 = scale, 2 = kick
  if (threadIdx.x == 0) s_act = ps->stop ? 0 : 1;
  __syncthreads();
  if (!s_act) return;
  const double sq = sum_squares(atav, n, seq != 0);
  if (threadIdx.x == 0) {
    const double next = sqrt(sq);
    s_next = next;
    s_act = next == 0.0 ? 2 : 1;
  }
  __syncthreads();
  const double next = s_next;
  const int64_t it = ps->it;
  if (s_act == 2) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = i == int(it % n) ? 1.0 : 0.0;
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = atav[i] / next;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (s_act == 1) {
    if (fabs(next - ps->lambda) <= ps->tol * smax(1.0, next)) {
      ps->lambda = next;
      ps->stop = 1;
    } else {
      ps->lambda = next;
    }
  }
  ps->it = it + 1;
  if (ps->it >= ps->max_it) ps->stop = 1;
}

__global__ void power_init_kernel(double* v, int n, int seq) {
  // v = ones / norm2(ones)
  __shared__ double s_nv;
  double sq = 0.0;
  if (seq) {
    if (threadIdx.x == 0)
      for (int i = 0; i < n; ++i) sq += 1.0 * 1.0;
  } else {
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += 1.0;
    sq = block_sum1(t);
  }
  if (threadIdx.x == 0) s_nv = sqrt(sq);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = 1.0 / s_nv;
}

// squared_norm(x) + squared_norm(y) + 2 s y'(Ax) (standard_form.hpp:93-98)
__global__ void ps_norm_kernel(const double* x, const double* y, const double* ax, int n, int m, double s, int seq,
                               double* out) {
  double a = 0.0, b = 0.0, d = 0.0;
  if (seq) {
    if (threadIdx.x == 0) {
      for (int j = 0; j < n; ++j) a += x[j] * x[j];
      for (int i = 0; i < m; ++i) b += y[i] * y[i];
      for (int i = 0; i < m; ++i) d += y[i] * ax[i];
    }
  } else {
    double ta = 0.0, tb = 0.0, td = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) ta += x[j] * x[j];
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      tb += y[i] * y[i];
      td += y[i] * ax[i];
    }
    a = block_sum1(ta);
    b = block_sum1(tb);
    d = block_sum1(td);
  }
  if (threadIdx.x == 0) *out = a + b + 2.0 * s * d;
}

int vec_grid(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return int(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 8)));
}

struct Vec {
  Buf<double> b;
  explicit Vec(int64_t n, cudaStream_t s) : b(size_t(n)) {
    PDLP_CUDA(cudaMemsetAsync(b.p, 0, size_t(std::max<int64_t>(n, 1)) * 8, s));
  }
  double* p() const { return b.p; }
};

void upload(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (n) PDLP_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * 8, cudaMemcpyHostToDevice, s));
}

// the five KKT sums of (x, y) on the device, into `part` (fast) or left to the
// sequential consumer (parity): Ax -> ax, A'y -> aty first
void kkt_prepare(const Operators& ops, const double* x, const double* y, double* ax, double* aty, const double* b,
                 const double* c, double* part, bool seq, cudaStream_t s) {
  launch_spmv(ops.a.d, false, x, ax, seq, s);
  launch_spmv(ops.at.d, false, y, aty, seq, s);
  if (!seq)
    kkt_partials_kernel<<<kRedBlocks, kThreads, 0, s>>>(ax, b, x, aty, c, y, ops.m, ops.n, part);
}

struct Stream {
  cudaStream_t s;
  Stream() { PDLP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() { cudaStreamDestroy(s); }
};

int check_args(const pdlp_csr* A, const double* b, const double* c) {
  if (!A || !b || !c || (A->nnz > 0 && ((!A->col_indices && !A->col_indices32) || !A->values)) ||
      !A->row_offsets) {
    set_last_error("null argument");
    return PDLP_EINVAL;
  }
  return PDLP_OK;
}

template <class F>
int guarded(int32_t device, F&& f) {
  try {
    PDLP_CUDA(cudaSetDevice(device));
    set_kernel_attributes();
    f();
    set_last_error("");
    return PDLP_OK;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return PDLP_ECUDA;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return PDLP_EINVAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PDLP_ERUNTIME;
  }
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" void pdlp_standard_default_options(pdlp_standard_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->step_size = 0.0;
  o->restart_decay = 0.5;
  o->convergence_tol = 1e-9;
  o->iteration_limit = 1000000;
  o->parity = 0;
  o->device = 0;
}

extern "C" int pdlp_standard_pdhg(const pdlp_csr* A, const double* b, const double* c,
                                  const pdlp_standard_options* o, const double* x0, const double* y0,
                                  double* start_kkt, int64_t* lengths, int64_t cap, int64_t* counters,
                                  double* x_out, double* y_out, double* iter_x, double* iter_y,
                                  int64_t iter_cap) {
  if (int rc = check_args(A, b, c)) return rc;
  if (!o || !counters || (cap > 0 && (!start_kkt || !lengths))) {
    set_last_error("null argument");
    return PDLP_EINVAL;
  }
  // StandardPdhgOptions::validate (standard_form.hpp:107-112)
  if (!(o->step_size > 0.0)) {
    set_last_error("step_size must be positive");
    return PDLP_EINVAL;
  }
  if (!(o->restart_decay > 0.0 && o->restart_decay < 1.0)) {
    set_last_error("restart_decay must lie in (0, 1)");
    return PDLP_EINVAL;
  }
  return guarded(o->device, [&]() {
    Stream st_;
    cudaStream_t s = st_.s;
    const bool seq = o->parity != 0;
    Operators ops(*A, seq, s);
    const int m = ops.m, n = ops.n;
    Vec x(n, s), y(m, s), xn(n, s), yn(m, s), ext(n, s), aty(n, s), aext(m, s), xa(n, s), ya(m, s), ax(m, s),
        atya(n, s), bv(m, s), cv(n, s), part(5 * kRedBlocks, s), xs(n, s), ys(m, s);
    upload(bv.p(), b, m, s);
    upload(cv.p(), c, n, s);
    if (x0 && y0) {
      upload(x.p(), x0, n, s);
      upload(y.p(), y0, m, s);
      upload(xs.p(), x0, n, s);
      upload(ys.p(), y0, m, s);
    }
    const int64_t ecap = std::max<int64_t>(cap, 1);
    Buf<double> ep_kkt{size_t(ecap)};
    Buf<int64_t> ep_len{size_t(ecap)};
    PDLP_CUDA(cudaMemsetAsync(ep_len.p, 0, size_t(ecap) * 8, s));
    const int64_t lcap = (iter_x && iter_y) ? std::max<int64_t>(0, iter_cap) : 0;
    Buf<double> log_x{size_t(std::max<int64_t>(1, lcap * n))}, log_y{size_t(std::max<int64_t>(1, lcap * m))};
    Buf<SfState> state(1);
    Buf<int> restart(1);
    SfState h{};
    h.limit = o->iteration_limit;
    h.decay = o->restart_decay;
    h.tol = o->convergence_tol;
    h.step = o->step_size;
    PDLP_CUDA(cudaMemcpyAsync(state.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    // open_epoch(z0)
    kkt_prepare(ops, x.p(), y.p(), ax.p(), atya.p(), bv.p(), cv.p(), part.p(), seq, s);
    sf_open_kernel<<<1, 32, 0, s>>>(state.p, part.p(), kRedBlocks, ax.p(), bv.p(), x.p(), atya.p(), cv.p(), y.p(),
                                    m, n, seq, ep_kkt.p, cap);
    const int gn = vec_grid(n), gm = vec_grid(m), gnm = vec_grid(std::max(n, m));
    for (;;) {
      PDLP_CUDA(cudaMemcpyAsync(&h, state.p, sizeof(h), cudaMemcpyDeviceToHost, s));
      PDLP_CUDA(cudaStreamSynchronize(s));
      if (h.stop) break;
      for (int k = 0; k < kPoll; ++k) {
        zero_int_kernel<<<1, 1, 0, s>>>(&state.p->bad);
        launch_spmv(ops.at.d, false, y.p(), aty.p(), seq, s);
        sf_primal_kernel<<<gn, kThreads, 0, s>>>(state.p, x.p(), cv.p(), aty.p(), xn.p(), ext.p(), n);
        launch_spmv(ops.a.d, false, ext.p(), aext.p(), seq, s);
        sf_dual_kernel<<<gm, kThreads, 0, s>>>(state.p, y.p(), bv.p(), aext.p(), yn.p(), m);
        sf_commit_kernel<<<gnm, kThreads, 0, s>>>(state.p, x.p(), y.p(), xn.p(), yn.p(), xa.p(), ya.p(), n, m,
                                                  log_x.p, log_y.p, lcap);
        kkt_prepare(ops, xa.p(), ya.p(), ax.p(), atya.p(), bv.p(), cv.p(), part.p(), seq, s);
        sf_decide_kernel<<<1, 32, 0, s>>>(state.p, part.p(), kRedBlocks, ax.p(), bv.p(), xa.p(), atya.p(), cv.p(),
                                          ya.p(), m, n, seq, ep_kkt.p, ep_len.p, cap, restart.p);
        sf_restart_kernel<<<gnm, kThreads, 0, s>>>(restart.p, x.p(), y.p(), xs.p(), ys.p(), xa.p(), ya.p(), n,
                                                   m);
      }
      PDLP_CUDA(cudaGetLastError());
    }
    // the in-progress epoch's length (standard_form.hpp:207-209)
    std::vector<int64_t> hlen(static_cast<size_t>(ecap));
    std::vector<double> hkkt(static_cast<size_t>(ecap));
    PDLP_CUDA(cudaMemcpyAsync(hlen.data(), ep_len.p, size_t(ecap) * 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaMemcpyAsync(hkkt.data(), ep_kkt.p, size_t(ecap) * 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
    const int64_t ne = h.epochs;
    if (ne > 0 && ne - 1 < cap && hlen[size_t(ne - 1)] == 0) hlen[size_t(ne - 1)] = h.inner;
    for (int64_t e = 0; e < std::min(ne, cap); ++e) {
      start_kkt[e] = hkkt[size_t(e)];
      lengths[e] = hlen[size_t(e)];
    }
    counters[0] = ne;
    counters[1] = h.total;
    counters[2] = h.converged;
    counters[3] = h.failure;
    // the last epoch's start point (trace.epochs.back().start)
    if (x_out) PDLP_CUDA(cudaMemcpyAsync(x_out, xs.p(), size_t(n) * 8, cudaMemcpyDeviceToHost, s));
    if (y_out) PDLP_CUDA(cudaMemcpyAsync(y_out, ys.p(), size_t(m) * 8, cudaMemcpyDeviceToHost, s));
    const int64_t logged = std::min<int64_t>(lcap, h.total);
    if (logged > 0) {
      if (n) PDLP_CUDA(cudaMemcpyAsync(iter_x, log_x.p, size_t(logged * n) * 8, cudaMemcpyDeviceToHost, s));
      if (m) PDLP_CUDA(cudaMemcpyAsync(iter_y, log_y.p, size_t(logged * m) * 8, cudaMemcpyDeviceToHost, s));
    }
    PDLP_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int pdlp_spectral_norm(const pdlp_csr* A, double tol, int32_t max_iterations, int32_t parity,
                                  int32_t device, double* out) {
  if (!A || !A->row_offsets || (A->nnz > 0 && ((!A->col_indices && !A->col_indices32) || !A->values)) || !out) {
    set_last_error("null argument");
    return PDLP_EINVAL;
  }
  if (A->num_rows == 0 || A->num_cols == 0 || A->nnz == 0) {
    *out = 0.0;
    return PDLP_OK;
  }
  return guarded(device, [&]() {
    Stream st_;
    cudaStream_t s = st_.s;
    const bool seq = parity != 0;
    Operators ops(*A, seq, s);
    const int m = ops.m, n = ops.n;
    Vec v(n, s), av(m, s), atav(n, s);
    Buf<PowerState> ps(1);
    PowerState h{};
    h.max_it = max_iterations;
    h.tol = tol;
    h.stop = max_iterations <= 0;
    PDLP_CUDA(cudaMemcpyAsync(ps.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    power_init_kernel<<<1, kThreads, 0, s>>>(v.p(), n, seq);
    for (;;) {
      PDLP_CUDA(cudaMemcpyAsync(&h, ps.p, sizeof(h), cudaMemcpyDeviceToHost, s));
      PDLP_CUDA(cudaStreamSynchronize(s));
      if (h.stop) break;
      for (int k = 0; k < kPoll; ++k) {
        launch_spmv(ops.a.d, false, v.p(), av.p(), seq, s);
        launch_spmv(ops.at.d, false, av.p(), atav.p(), seq, s);
        power_step_kernel<<<1, kThreads, 0, s>>>(ps.p, atav.p(), v.p(), n, seq);
      }
      PDLP_CUDA(cudaGetLastError());
    }
    *out = std::sqrt(h.lambda);
  });
}

extern "C" int pdlp_p_s_norm_squared(const pdlp_csr* A, const double* b, const double* c, double step,
                                     const double* x, const double* y, int32_t parity, int32_t device,
                                     double* out) {
  if (int rc = check_args(A, b, c)) return rc;
  if (!x || !y || !out) {
    set_last_error("null argument");
    return PDLP_EINVAL;
  }
  return guarded(device, [&]() {
    Stream st_;
    cudaStream_t s = st_.s;
    const bool seq = parity != 0;
    Operators ops(*A, seq, s);
    const int m = ops.m, n = ops.n;
    Vec xv(n, s), yv(m, s), ax(m, s);
    upload(xv.p(), x, n, s);
    upload(yv.p(), y, m, s);
    launch_spmv(ops.a.d, false, xv.p(), ax.p(), seq, s);
    Buf<double> r(1);
    ps_norm_kernel<<<1, kThreads, 0, s>>>(xv.p(), yv.p(), ax.p(), n, m, step, seq, r.p);
    PDLP_CUDA(cudaMemcpyAsync(out, r.p, 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int pdlp_kkt_error_standard(const pdlp_csr* A, const double* b, const double* c, const double* x,
                                       const double* y, int32_t parity, int32_t device, double* out) {
  if (int rc = check_args(A, b, c)) return rc;
  if (!x || !y || !out) {
    set_last_error("null argument");
    return PDLP_EINVAL;
  }
  return guarded(device, [&]() {
    Stream st_;
    cudaStream_t s = st_.s;
    const bool seq = parity != 0;
    Operators ops(*A, seq, s);
    const int m = ops.m, n = ops.n;
    Vec xv(n, s), yv(m, s), ax(m, s), aty(n, s), bv(m, s), cv(n, s), part(5 * kRedBlocks, s);
    upload(xv.p(), x, n, s);
    upload(yv.p(), y, m, s);
    upload(bv.p(), b, m, s);
    upload(cv.p(), c, n, s);
    kkt_prepare(ops, xv.p(), yv.p(), ax.p(), aty.p(), bv.p(), cv.p(), part.p(), seq, s);
    Buf<SfState> state(1);
    SfState h{};
    h.limit = INT64_MAX;
    h.tol = -1.0;
    PDLP_CUDA(cudaMemcpyAsync(state.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    Buf<double> k(1);
    sf_open_kernel<<<1, 32, 0, s>>>(state.p, part.p(), kRedBlocks, ax.p(), bv.p(), xv.p(), aty.p(), cv.p(), yv.p(),
                                    m, n, seq, k.p, 1);
    PDLP_CUDA(cudaMemcpyAsync(out, k.p, 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
  });
}
