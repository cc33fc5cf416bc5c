// panels.cu — column-panel SpMV for operators whose gathered vector is much
// larger than L2 and whose rows scatter over it (C4: random columns over a
// 320 MB x; ncu shows ~100 B of DRAM traffic per gathered element, 6x the
// algorithmic bytes, because every miss fetches a line for one double).
//
// The operator's entries are re-ordered panel-major: panel p holds the entries
// whose column lies in [p w, (p+1) w), stored as a CSR of P * rows "stacked"
// rows (p, r). One pass of the ordinary tiled SpMV over the stacked CSR, in
// tile order, walks the panels one after another, so the running CTAs gather
// from one L2-sized slice of the vector at a time; it writes one partial sum
// per (panel, row). A combine kernel then adds each row's P partials in panel
// order and applies the fused update of the dual or primal kernel (the same
// epilogue code, DualEpi / PrimalEpi) with its reductions.
//
// Fast mode on one device only (the per-row sum order changes: panels first).
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

struct PartialEpi : EpiBase<PartialEpi> {
  static constexpr int NP = 1, NA = 1, NR = 1;
  static constexpr bool kEvictFirst = true;  // the stacked operator streams through L2 once per pass
  // (no kUniform: stacked rows are short and irregular)
  static constexpr TileGeom kGeom = kPanelGeom;
  static constexpr bool kNeedCol = false;
  const double* __restrict__ x;
  double* __restrict__ out;
  __device__ __forceinline__ void gather(int c, double (&g)[1]) const { g[0] = __ldg(x + c); }
  __device__ __forceinline__ void add(double (&a)[1], const double (&p)[1], int) const { a[0] += p[0]; }
  __device__ __forceinline__ void row_done(int r, const double (&a)[1], double (&)[1]) const { out[r] = a[0]; }
};
}  // namespace

// ---- setup: stacked panel CSR ---------------------------------------------

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

// ---- iteration ------------------------------------------------------------

// Pass 1: partial[p * rows + r] = sum over panel p of row r. The dual gathers
// x' (the trial primal); the primal gathers the current y after the decision
// (decide_kernel committed it) and skips when the branch needs no K'y.
template <bool kPrimal>
__global__ void __launch_bounds__(kThreads, 4) panel_spmv_kernel(DevCsr A, DevIter it, double* partial,
                                                                 int mode_override) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Tile t = A.tiles[blockIdx.x];
  if (it.prefetch) prefetch_tile(t, A.rp, A.col, A.val);
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
  PartialEpi epi;
  epi.x = src;
  epi.out = partial;
  double red[1] = {0.0};
  run_tile<PartialEpi, false>(t, A.rp, A.col, A.val, epi, red, A.chunk_part, A.chunk_ctr, smem);
  griddep_launch_dependents();
}

// Pass 2 of the dual: CTA 0 is the helper (state snapshot, dx^2 of x'); CTA
// b >= 1 combines rows [(b-1) R, b R), R = kIterGeom.stream_rows, and applies
// the dual update (DualEpi) with its partials at slot b-1.
__global__ void __launch_bounds__(kThreads, 4) dual_combine_kernel(DevIter it, const double* partial,
                                                                   int panels) {
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
  constexpr int RPT = kIterGeom.stream_rows / kThreads;
  const int b = blockIdx.x - 1;
  const int r0 = b * kIterGeom.stream_rows + threadIdx.x;
  DualEpi<false> epi;
  epi.xg = nullptr;
  epi.y = it.y[st->iy_cur];
  epi.kx = it.kx[st->ikx_cur];
  epi.q = it.q;
  epi.yt = it.y[st->iy_trial];
  epi.kxt = it.kx[1 - st->ikx_cur];
  epi.sigma = st->eta * st->omega;  // sigma = eta * omega, solver.hpp:402
  epi.m1 = it.m1;
  double acc[RPT][1];
  int nvalid = 0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = r0 + i * kThreads;
    acc[i][0] = 0.0;
    if (r < it.m) {
      nvalid = i + 1;
      for (int p = 0; p < panels; ++p) acc[i][0] += __ldcg(partial + size_t(p) * it.m + r);
    }
  }
  double red[3] = {0.0, 0.0, 0.0};
  epi.rows_strided<RPT>(r0, kThreads, nvalid, acc, red);
  griddep_launch_dependents();
  store_partial<3, 0>(red, it.d_part, b, it.d_tiles);
}

// Pass 2 of the primal (decision already committed by decide_kernel): CTAs
// b < nblk combine columns [b R, (b+1) R) and apply PrimalEpi (accept: with the
// averages; restart / lazy retry: without), or recompute x' from the kept K'y
// (retry); the trailing CTAs update avg_y on accepted steps.
template <bool kNonneg>
__global__ void __launch_bounds__(kThreads, 4) primal_combine_kernel(DevIter it, const double* partial,
                                                                     int panels, int nblk,
                                                                     int mode_override) {
  griddep_wait();
  DevState* st = it.st;
  const DevState& s = *st;
  const int mode = mode_override >= 0 ? mode_override : s.p_mode;
  if (mode == kPNone) return;
  const double tau = s.eta / s.omega;  // tau = eta / omega, solver.hpp:401
  const int bid = blockIdx.x;
  if (bid >= nblk) {  // avg_y .add (solver.hpp:839)
    if (mode == kPAccept) {
      const int nb = gridDim.x - nblk, b = bid - nblk;
      const int per = (it.m + nb - 1) / nb;
      const int i0 = b * per, i1 = min(it.m, i0 + per);
      const double* yc = it.y[s.iy_cur];
      for (int i = i0 + threadIdx.x; i < i1; i += kThreads)
        it.avg_y[i] = s.avg_first ? yc[i] : it.avg_y[i] + s.avg_ratio * (yc[i] - it.avg_y[i]);
    }
    return;
  }
  constexpr int RPT = kIterGeom.stream_rows / kThreads;
  const int j0 = bid * kIterGeom.stream_rows + threadIdx.x;
  const bool lazy_retry = it.kty_lazy && mode == kPRetry && mode_override < 0;
  double red[2] = {0.0, 0.0};
  if (mode == kPAccept || mode == kPRestart || lazy_retry) {
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
    double acc[RPT][1];
    int nvalid = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int j = j0 + i * kThreads;
      acc[i][0] = 0.0;
      if (j < it.n) {
        nvalid = i + 1;
        for (int p = 0; p < panels; ++p) acc[i][0] += __ldcg(partial + size_t(p) * it.n + j);
      }
    }
    epi.rows_strided<RPT>(j0, kThreads, nvalid, acc, red);
  } else if (mode == kPRetry) {
    const double* xc = it.x[s.ix_cur];
    const double* kty = it.kty[s.ikty_cur];
    double* xt = it.x[s.ix_trial];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int j = j0 + i * kThreads;
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

int panel_combine_blocks(int rows) { return (rows + kIterGeom.stream_rows - 1) / kIterGeom.stream_rows; }

void launch_panel_dual(const DevCsr& kp, int panels, double* partial, const DevIter& it, cudaStream_t s) {
  const size_t sm = stream_smem_bytes<PartialEpi>();
  launch_pdl2(panel_spmv_kernel<false>, kp.ntiles, sm, s, kp, it, partial, -1);
  launch_pdl2(dual_combine_kernel, 1 + panel_combine_blocks(it.m), 0, s, it, (const double*)partial, panels);
}

void launch_panel_primal(const DevCsr& ktp, int panels, double* partial, const DevIter& it, int mode_override,
                         cudaStream_t s) {
  const size_t sm = stream_smem_bytes<PartialEpi>();
  launch_pdl2(panel_spmv_kernel<true>, ktp.ntiles, sm, s, ktp, it, partial, mode_override);
  const int nblk = panel_combine_blocks(it.n);
  const int grid = nblk + it.avg_blocks;
  if (it.nonneg)
    launch_pdl2(primal_combine_kernel<true>, grid, 0, s, it, (const double*)partial, panels, nblk, mode_override);
  else
    launch_pdl2(primal_combine_kernel<false>, grid, 0, s, it, (const double*)partial, panels, nblk, mode_override);
}

}  // namespace pdlp
