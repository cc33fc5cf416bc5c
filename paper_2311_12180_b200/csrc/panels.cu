// panels.cu — column-panel sweeps for operators whose gathered vector is far
// larger than L2 and whose rows scatter over it (C4: random columns over a
// 320 MB x and a 160 MB y; a direct gather pulls a 32-byte DRAM sector per
// nonzero). Reference: spmv (sparse_matrix.hpp:117-132) and spmv_transpose
// (:142-158, as a gather over the stored K^T), inside adaptive_step_cached
// (solver.hpp:409,456).
//
// Layout. The entries are re-ordered panel-major: panel p holds the entries
// whose column lies in [p w, (p+1) w), row by row, each row's entries in
// column order. Per panel, a byte per row gives the row's entry count in that
// panel (`cnt`), and one int per warp block of 128 rows gives the block's
// first entry (`boff`); no per-(panel, row) offsets are stored.
//
// Iteration. Pass p (one launch per panel) walks every block of 1024 rows
// (one CTA, 4 rows per thread). Every load a CTA needs is issued up front and
// only the true dependences wait: the block's first entry (`boff`, L2) ->
// its indices (HBM) -> the gathers of v[col] (the L2-resident panel slice),
// with the values, the count bytes and the running sums arriving meanwhile;
// the products are staged in shared memory and each thread continues its
// rows' running sums over them in entry order. The running sums live in `acc`
// between passes (16 B per row per pass); the last pass applies the fused
// update of the dual or primal kernel (DualEpi / PrimalEpi) instead, with one
// reduction partial per block. Measured slower on C4 and not kept (DESIGN.md
// §3): TMA bulk copies of the blocks (per CTA with a 2-3 stage ring, per warp;
// 1.7-2.3x); row bands whose running sums stay L2-resident beside 16-32 MB
// panels, as one launch per (band, panel) (K 2.3-3.6 ms vs 1.7), as a
// persistent CTA or warp sweep with cp.async double buffering (3.4-6.9 ms);
// 2048-row blocks (K 1.9-2.5 ms); an L2 prefetch of the block one wave ahead
// (K 1.74-1.92 ms vs 1.70). The pass is latency-bound at 4 CTAs of 64
// registers per SM (ncu: long-scoreboard 44% of stall samples, 48% warps
// active, ~3.2 TB/s of DRAM traffic).
//
// Every row is summed by one thread, starting from 0.0, in increasing column
// order: exactly the reference's `out[r] += val * x[col]` sequence. The panel
// sweep is therefore bitwise equal to the sequential SpMV (and to the tiled
// engine's STREAM rows), whatever the panel count.
#include "epilogues.cuh"
#include "kernels.cuh"
#include "spmv_engine.cuh"

namespace pdlp {

namespace {
int grid_n(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return int(g);
}

__device__ __forceinline__ unsigned ld_stream_u32_ef(const unsigned char* p, uint64_t pol) {
  unsigned r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_stream_i1_ef(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_stream_d1_ef(const double* p, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_acc(const double* p) {
  double r;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_acc(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

}  // namespace

using SweepOp = PanelView;

#ifndef PDLP_SWEEP_ROWS
#define PDLP_SWEEP_ROWS 1024
#endif
constexpr int kSweepRows = PDLP_SWEEP_ROWS;  // rows per CTA: 4 or 8 per thread, stride kThreads
constexpr int kSweepRPT = kSweepRows / kThreads;
// 1536 staged entries (6 per thread) and 6 resident CTAs per SM for the SpMV
// passes, 5 / 4 for the dual / primal final passes (C4: K 1.70 -> 1.44 ms,
// whole iteration 234 -> 250 it/s; the passes are latency-bound, so resident
// CTAs matter more than loads in flight per thread)
#ifndef PDLP_SWEEP_CHUNK_K
#define PDLP_SWEEP_CHUNK_K 1536
#endif
// K^T blocks hold ~1.7 k entries on C4 (5 per row over 3 panels): a 1792-entry
// stage keeps them in one round (K^T 1.45 -> 1.31 ms), while K's ~1.46 k
// entries per block run faster in 1536
#ifndef PDLP_SWEEP_CHUNK_T
#define PDLP_SWEEP_CHUNK_T 1792
#endif
#ifndef PDLP_SWEEP_CTAS
#define PDLP_SWEEP_CTAS 6
#endif
// resident CTAs per SM of the final passes (their fused updates need more
// registers than the SpMV passes)
#ifndef PDLP_SWEEP_CTAS_DUALF
#define PDLP_SWEEP_CTAS_DUALF 5
#endif
#ifndef PDLP_SWEEP_CTAS_PRIMALF
#define PDLP_SWEEP_CTAS_PRIMALF 4
#endif
// the final passes stream their dense update operands (.cs) past the L2-resident panel slice
#ifndef PDLP_SWEEP_STREAM_IO
#define PDLP_SWEEP_STREAM_IO 1
#endif
constexpr bool kSweepStreamIO = PDLP_SWEEP_STREAM_IO != 0;
constexpr int kChunkK = PDLP_SWEEP_CHUNK_K;  // products staged per round: sweeps over K
constexpr int kChunkT = PDLP_SWEEP_CHUNK_T;  // ... over K^T
constexpr int kSweepCtasPerSm = PDLP_SWEEP_CTAS;

static_assert(kSweepRPT == 4 || kSweepRPT == 8, "four or eight count bytes and rows per thread");

template <int CH>
struct SweepSmem {
  int off[kSweepRows + 1];
  int warp[kWarps + 1];
  double prod[CH];
};

// ---- setup -----------------------------------------------------------------

__global__ void panel_keys_kernel(const int* row_of, const int* col, int64_t nnz, int width, int rows,
                                  int* keys) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x)
    keys[k] = (col[k] / width) * rows + row_of[k];
}

__global__ void panel_gather_kernel(const int* perm, const int* col, const double* val, int64_t nnz,
                                    int* col_p, double* val_p) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x) {
    const int p = perm[k];
    col_p[k] = col[p];
    val_p[k] = val[p];
  }
}

// rows whose entries fall into more than one panel, summed over rows (the
// planner's "does this operator scatter over its vector" test)
__global__ void panel_spread_kernel(const int* rp, const int* col, int rows, int width,
                                    unsigned long long* distinct) {
  unsigned long long local = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    int last = -1;
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const int p = col[k] / width;
      if (p != last) ++local, last = p;
    }
  }
  atomicAdd(distinct, local);  // integer: order-free
}

// cnt[p][r] (bytes) and boff[p][b] from the per-(panel, row) counts and their
// exclusive scan `so` over the stacked rows (p, r); `over` flags a count > 255.
__global__ void panel_meta_kernel(const int* counts, const int* so, int rows, int rows_pad, int panels, int nblk,
                                  unsigned char* cnt, int* boff, int* over) {
  const int64_t total = int64_t(panels) * rows_pad;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int p = int(i / rows_pad), r = int(i % rows_pad);
    int cv = 0;
    if (r < rows) cv = counts[int64_t(p) * rows + r];
    if (cv > 255) atomicOr(over, 1);
    cnt[i] = (unsigned char)(cv > 255 ? 255 : cv);
  }
  const int64_t nb = int64_t(panels) * (nblk + 1);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nb; i += int64_t(gridDim.x) * blockDim.x) {
    const int p = int(i / (nblk + 1)), b = int(i % (nblk + 1));
    const int64_t r = int64_t(b) * kSweepRows < rows ? int64_t(b) * kSweepRows : int64_t(rows);
    boff[i] = so[int64_t(p) * rows + r];
  }
}

void launch_panel_keys(const int* row_of, const int* col, int64_t nnz, int width, int rows, int* keys,
                       cudaStream_t s) {
  panel_keys_kernel<<<grid_n(nnz), kThreads, 0, s>>>(row_of, col, nnz, width, rows, keys);
  PDLP_CUDA(cudaGetLastError());
}
void launch_panel_gather(const int* perm, const int* col, const double* val, int64_t nnz, int* col_p,
                         double* val_p, cudaStream_t s) {
  panel_gather_kernel<<<grid_n(nnz), kThreads, 0, s>>>(perm, col, val, nnz, col_p, val_p);
  PDLP_CUDA(cudaGetLastError());
}
void launch_panel_spread(const int* rp, const int* col, int rows, int width, unsigned long long* distinct,
                         cudaStream_t s) {
  panel_spread_kernel<<<grid_n(rows), kThreads, 0, s>>>(rp, col, rows, width, distinct);
  PDLP_CUDA(cudaGetLastError());
}
void launch_panel_meta(const int* counts, const int* so, int rows, int rows_pad, int panels, int nblk,
                       unsigned char* cnt, int* boff, int* over, cudaStream_t s) {
  panel_meta_kernel<<<grid_n(int64_t(panels) * rows_pad), kThreads, 0, s>>>(counts, so, rows, rows_pad, panels,
                                                                            nblk, cnt, boff, over);
  PDLP_CUDA(cudaGetLastError());
}
int panel_rows_pad(int rows) { return (rows + kSweepRows - 1) / kSweepRows * kSweepRows; }
int panel_blocks(int rows) { return (rows + kSweepRows - 1) / kSweepRows; }

// ---- iteration ---------------------------------------------------------------

namespace {

// Exclusive block scan of one int per thread (fixed order; integers).
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp /* kWarps + 1 */, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int t = lane < kWarps ? s_warp[lane] : 0;
    int ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += u;
    }
    if (lane < kWarps) s_warp[lane] = ti - t;
    if (lane == kWarps - 1) s_warp[kWarps] = ti;
  }
  __syncthreads();
  *total = s_warp[kWarps];
  return s_warp[warp] + incl - v;
}

// Continues the running sums acc[i] of this thread's rows b R + tid + i kThreads
// over panel p of v (acc[] = 0.0 at p = 0, else the sums loaded from `acc`);
// returns a bit per row with entries in this panel.
template <int CH>
__device__ __forceinline__ unsigned sweep_block(const SweepOp& op, int p, int b, const double* __restrict__ v,
                                                double (&acc)[kSweepRPT], SweepSmem<CH>& sm) {
  constexpr int kSweepChunk = CH;                    // entries staged per round
  constexpr int kSweepPer = CH / kThreads;           // entries per thread per round, all in flight
  const int tid = threadIdx.x;
  const uint64_t ef = l2_evict_first_policy();
  // independent loads first: the block's entry range, its count bytes, the sums
  const int* bo = op.boff + size_t(p) * (op.nblk + 1) + b;
  const int e0 = __ldg(bo), e1 = __ldg(bo + 1);
  uint2 cw;
  {
    const unsigned char* cp = op.cnt + size_t(p) * op.rows_pad + size_t(b) * kSweepRows + kSweepRPT * tid;
    cw.x = ld_stream_u32_ef(cp, ef);
    cw.y = kSweepRPT == 8 ? ld_stream_u32_ef(cp + 4, ef) : 0u;
  }
  const int r0 = b * kSweepRows + tid;
#pragma unroll
  for (int q = 0; q < kSweepRPT; ++q) acc[q] = p > 0 ? ld_acc(op.acc + r0 + q * kThreads) : 0.0;
  const int E = e1 - e0;
  const int* __restrict__ col = op.col + e0;
  const double* __restrict__ val = op.val + e0;
  // the first round's products need only the entry range: staged before the scan
  auto stage = [&](int c0, int c1) {
    int cc[kSweepPer];
#pragma unroll
    for (int j = 0; j < kSweepPer; ++j) {
      const int k = c0 + tid + j * kThreads;
      cc[j] = k < c1 ? ld_stream_i1_ef(col + k, ef) : 0;
    }
    double g[kSweepPer];
#pragma unroll
    for (int j = 0; j < kSweepPer; ++j) {
      const int k = c0 + tid + j * kThreads;
      if (k < c1) g[j] = __ldg(v + cc[j]);
    }
#pragma unroll
    for (int j = 0; j < kSweepPer; ++j) {
      const int k = c0 + tid + j * kThreads;
      if (k < c1) sm.prod[k - c0] = ld_stream_d1_ef(val + k, ef) * g[j];  // rounded product, as val * x
    }
  };
  stage(0, min(E, kSweepChunk));
  // row offsets inside the block (the thread's rows' count bytes, block scan)
  int tot = 0;
#pragma unroll
  for (int i = 0; i < kSweepRPT; ++i) tot += int(((i < 4 ? cw.x : cw.y) >> (8 * (i & 3))) & 255u);
  int Et;
  const int ex = block_excl_scan(tot, sm.warp, &Et);  // (its barriers also publish the staged products)
  {
    int o = ex;
#pragma unroll
    for (int i = 0; i < kSweepRPT; ++i) {
      sm.off[kSweepRPT * tid + i] = o;
      o += int(((i < 4 ? cw.x : cw.y) >> (8 * (i & 3))) & 255u);
    }
  }
  if (tid == kThreads - 1) sm.off[kSweepRows] = Et;
  __syncthreads();
  unsigned has = 0;
  for (int c0 = 0; c0 < E; c0 += kSweepChunk) {
    const int c1 = min(E, c0 + kSweepChunk);
    if (c0 > 0) {  // a further round of an oversized block
      __syncthreads();
      stage(c0, c1);
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kSweepRPT; ++q) {
      const int r = tid + q * kThreads;
      const int o = sm.off[r], e = sm.off[r + 1];
      if (c0 == 0) has |= (e > o ? 1u : 0u) << q;
      const int k0 = max(o, c0), k1 = min(e, c1);
      for (int k = k0; k < k1; ++k) acc[q] = acc[q] + sm.prod[k - c0];  // sparse_matrix.hpp:128-130
    }
  }
  return has;
}

}  // namespace

// Passes 0 .. P-2: the dual gathers x' (the trial primal); the primal gathers
// the current y after the decision (decide_kernel committed it) and skips when
// the branch needs no K'y.
template <bool kPrimal>
__global__ void __launch_bounds__(kThreads, kSweepCtasPerSm) sweep_pass_kernel(SweepOp op, DevIter it, int p,
                                                                             int mode_override) {
  __shared__ SweepSmem<kPrimal ? kChunkT : kChunkK> sm;
  griddep_wait();
  const DevState* st = it.st;
  const double* src;
  if (!kPrimal) {
    if (st->failure || st->window_accepts >= st->window_target) return;
    src = it.x[st->ix_trial];
  } else {
    const int mode = mode_override >= 0 ? mode_override : st->p_mode;
    const bool lazy_retry = it.kty_lazy && mode == kPRetry && mode_override < 0;
    if (!(mode == kPAccept || mode == kPRestart || lazy_retry)) return;
    src = it.y[st->iy_cur];
  }
  const int b = blockIdx.x;
  double acc[kSweepRPT];
  const unsigned has = sweep_block(op, p, b, src, acc, sm);
  griddep_launch_dependents();
  const int r0 = b * kSweepRows + threadIdx.x;
#pragma unroll
  for (int q = 0; q < kSweepRPT; ++q) {
    const int r = r0 + q * kThreads;
    if (r < op.rows && (p == 0 || ((has >> q) & 1u))) st_acc(op.acc + r, acc[q]);
  }
}

// Last pass of the dual: CTA 0 is the helper (state snapshot, dx^2 of x'); CTA
// b >= 1 finishes rows [(b-1) R, b R) and applies the dual update (DualEpi)
// with its partials at slot b-1.
__global__ void __launch_bounds__(kThreads, PDLP_SWEEP_CTAS_DUALF) sweep_dual_final_kernel(SweepOp op, DevIter it) {
  __shared__ SweepSmem<kChunkK> sm;
  griddep_wait();
  DevState* st = it.st;
  const bool parked = st->failure || st->window_accepts >= st->window_target;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) *it.snap = *st;
    double pp[2];
    sum_partials<2, 0>(it.p_part + size_t(st->trials_total & 1) * it.p_tiles * 2, it.p_tiles, pp);
    if (threadIdx.x == 0) {
      it.px_total[0] = pp[0];
      it.px_total[1] = pp[1];
    }
    return;
  }
  if (parked) return;
  const int b = blockIdx.x - 1;
  const int r0 = b * kSweepRows + threadIdx.x;
  double acc[kSweepRPT];
  sweep_block(op, op.panels - 1, b, it.x[st->ix_trial], acc, sm);
  int nvalid = 0;
#pragma unroll
  for (int q = 0; q < kSweepRPT; ++q)
    if (r0 + q * kThreads < op.rows) nvalid = q + 1;
  DualEpi<false> epi;
  epi.xg = nullptr;
  epi.y = it.y[st->iy_cur];
  epi.kx = it.kx[st->ikx_cur];
  epi.q = it.q;
  epi.yt = it.y[st->iy_trial];
  epi.kxt = it.kx[1 - st->ikx_cur];
  epi.sigma = st->eta * st->omega;  // sigma = eta * omega, solver.hpp:402
  epi.m1 = it.m1;
  double a2[kSweepRPT][1];
#pragma unroll
  for (int q = 0; q < kSweepRPT; ++q) a2[q][0] = acc[q];
  double red[3] = {0.0, 0.0, 0.0};
  epi.rows_strided<kSweepRPT, 1, 3, kSweepStreamIO>(r0, kThreads, nvalid, a2, red);
  griddep_launch_dependents();
  store_partial<3, 0>(red, it.d_part, b, it.d_tiles);
}

// Last pass of the primal (decision already committed by decide_kernel): CTAs
// b < nblk finish columns [b R, (b+1) R) and apply PrimalEpi (accept: with the
// averages; restart / lazy retry: without), or recompute x' from the kept K'y
// (retry); the trailing CTAs update avg_y on accepted steps.
template <bool kNonneg>
__global__ void __launch_bounds__(kThreads, PDLP_SWEEP_CTAS_PRIMALF) sweep_primal_final_kernel(SweepOp op, DevIter it,
                                                                                     int mode_override) {
  __shared__ SweepSmem<kChunkT> sm;
  griddep_wait();
  DevState* st = it.st;
  const DevState& s = *st;
  const int mode = mode_override >= 0 ? mode_override : s.p_mode;
  if (mode == kPNone) return;
  const double tau = s.eta / s.omega;  // tau = eta / omega, solver.hpp:401
  const int bid = blockIdx.x;
  const int nblk = op.nblk;
  if (bid >= nblk) {  // avg_y .add (solver.hpp:839)
    if (mode == kPAccept) {
      const int nb = gridDim.x - nblk, b = bid - nblk;
      const int per = (it.m + nb - 1) / nb;
      const int i0 = b * per, i1 = min(it.m, i0 + per);
      const double* yc = it.y[s.iy_cur];
      for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
        const double yv = ld_io_plain<kSweepStreamIO>(yc + i);
        const double av = s.avg_first ? 0.0 : ld_io_plain<kSweepStreamIO>(it.avg_y + i);
        st_io<kSweepStreamIO>(it.avg_y + i, s.avg_first ? yv : av + s.avg_ratio * (yv - av));
      }
    }
    return;
  }
  const int j0 = bid * kSweepRows + threadIdx.x;
  const bool lazy_retry = it.kty_lazy && mode == kPRetry && mode_override < 0;
  double red[2] = {0.0, 0.0};
  if (mode == kPAccept || mode == kPRestart || lazy_retry) {
    double acc[kSweepRPT];
    sweep_block(op, op.panels - 1, bid, it.y[s.iy_cur], acc, sm);
    int nvalid = 0;
#pragma unroll
    for (int q = 0; q < kSweepRPT; ++q)
      if (j0 + q * kThreads < op.rows) nvalid = q + 1;
    const bool acc_step = mode == kPAccept;
    PrimalEpi<false, kNonneg> epi;
    epi.yg = nullptr;
    epi.xc = it.x[s.ix_cur];
    epi.c = it.c;
    epi.l = it.l;
    epi.u = it.u;
    epi.kty_out = it.kty[s.ikty_cur];
    epi.xt = it.x[s.ix_trial];
    epi.avg_x = it.avg_x;
    epi.seq_dx2 = nullptr;
    epi.tau = tau;
    epi.ratio = s.avg_ratio;
    epi.do_avg = acc_step;
    epi.avg_first = s.avg_first;
    epi.store_kty = (acc_step && it.kty_lazy) ? 0 : 1;
    double a2[kSweepRPT][1];
#pragma unroll
    for (int q = 0; q < kSweepRPT; ++q) a2[q][0] = acc[q];
    epi.template rows_strided<kSweepRPT, 1, 2, kSweepStreamIO>(j0, kThreads, nvalid, a2, red);
  } else if (mode == kPRetry) {
    const double* xc = it.x[s.ix_cur];
    const double* kty = it.kty[s.ikty_cur];
    double* xt = it.x[s.ix_trial];
#pragma unroll
    for (int q = 0; q < kSweepRPT; ++q) {
      const int j = j0 + q * kThreads;
      if (j < it.n) {
        const double xa = xc[j];
        const double v = xa - tau * (it.c[j] - kty[j]);
        const double xn = kNonneg ? smax(v, 0.0) : clamp_box(v, it.l[j], it.u[j]);
        xt[j] = xn;
        red[0] += (xn - xa) * (xn - xa);
        red[1] += isfinite(xn) ? 0.0 : 1.0;
      }
    }
  }
  griddep_launch_dependents();
  const size_t half = size_t(s.trials_total & 1) * it.p_tiles * 2;
  store_partial<2, 0>(red, it.p_part + half, bid, it.p_tiles);
}

// Plain SpMV through the panel sweep (bench / kernel parity): out = A v, the
// last pass storing the sums.
template <int CH>
__global__ void __launch_bounds__(kThreads, kSweepCtasPerSm) sweep_spmv_kernel(SweepOp op, const double* v, int p,
                                                                             double* out) {
  __shared__ SweepSmem<CH> sm;
  const int b = blockIdx.x;
  const int r0 = b * kSweepRows + threadIdx.x;
  double acc[kSweepRPT];
  const unsigned has = sweep_block(op, p, b, v, acc, sm);
  const bool last = p == op.panels - 1;
#pragma unroll
  for (int q = 0; q < kSweepRPT; ++q) {
    const int r = r0 + q * kThreads;
    if (r >= op.rows) continue;
    if (last)
      out[r] = acc[q];
    else if (p == 0 || ((has >> q) & 1u))
      st_acc(op.acc + r, acc[q]);
  }
}

void panel_kernel_attributes() {}

namespace {
template <class... P, class... A>
void launch_pdl2(void (*kern)(P...), int grid, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PDLP_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}
}  // namespace

void launch_panel_dual(const PanelView& kp, const DevIter& it, cudaStream_t s) {
  const SweepOp& op = kp;
  for (int p = 0; p + 1 < op.panels; ++p) launch_pdl2(sweep_pass_kernel<false>, op.nblk, 0, s, op, it, p, -1);
  launch_pdl2(sweep_dual_final_kernel, 1 + op.nblk, 0, s, op, it);
}

void launch_panel_primal(const PanelView& ktp, const DevIter& it, int mode_override, cudaStream_t s) {
  const SweepOp& op = ktp;
  for (int p = 0; p + 1 < op.panels; ++p)
    launch_pdl2(sweep_pass_kernel<true>, op.nblk, 0, s, op, it, p, mode_override);
  const int grid = op.nblk + it.avg_blocks;
  if (it.nonneg)
    launch_pdl2(sweep_primal_final_kernel<true>, grid, 0, s, op, it, mode_override);
  else
    launch_pdl2(sweep_primal_final_kernel<false>, grid, 0, s, op, it, mode_override);
}

void launch_panel_spmv(const PanelView& pv, const double* v, double* out, cudaStream_t s) {
  const SweepOp& op = pv;
  for (int p = 0; p < op.panels; ++p) {
    if (op.transposed)
      sweep_spmv_kernel<kChunkT><<<op.nblk, kThreads, 0, s>>>(op, v, p, out);
    else
      sweep_spmv_kernel<kChunkK><<<op.nblk, kThreads, 0, s>>>(op, v, p, out);
    PDLP_CUDA(cudaGetLastError());
  }
}

}  // namespace pdlp
