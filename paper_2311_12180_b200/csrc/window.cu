// window.cu — persistent, cooperative "window" kernel: one launch runs a whole
// evaluation window (up to evaluation_frequency accepted iterations of
// adaptive_step_cached, solver.hpp:381-467 / :794-841) in fast mode.
//
// Structure per trial (all CTAs co-resident, 2 per SM):
//   D phase   each CTA walks its share of K's tiles: y' = proj(y + sigma(q - 2Kx' + Kx)),
//             dy^2 / interaction partials (solver.hpp:409-435)
//   barrier   the last CTA to arrive sums the per-CTA partials in CTA order and
//             takes the step decision (eta_bar, eta', accept, averages' weight,
//             buffer rotation, :436-466) before releasing the others
//   P phase   accept: K'y' fused with avg_x/avg_y and the next trial's x' and dx^2;
//             reject: x' recomputed for the shrunk step
//   barrier
// Static operator data (indices, values, row offsets) of every tile is streamed
// into shared memory by the Tensor Memory Accelerator (cp.async.bulk, one
// elected thread, mbarrier transaction counts) through a 3-stage ring that runs
// ahead across phase and barrier boundaries, so matrix traffic overlaps the
// gathers, epilogues and barriers. Data written during the launch is read with
// coherent loads after each barrier's gpu-scope fence (no .nc path).
#include <cooperative_groups.h>

#include "../../include/pdlp_b200.h"
#include "epilogues.cuh"
#include "kernels.cuh"
#include "tma.cuh"
#include "window.cuh"

namespace pdlp {

namespace {

__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kStages = 3;
constexpr int kStageNnz = kWinGeom.stream_nnz + 8;     // quad-aligned tile span
constexpr int kStageRows = kWinGeom.stream_rows + 12;  // quad-aligned offsets span

struct Stage {
  int col[kStageNnz];
  double val[kStageNnz];
  int rp[kStageRows];
};
static_assert(sizeof(int) * kStageNnz % 16 == 0, "stage alignment");

struct WinSmem {
  Stage stage[kStages];
  double prod[kWinGeom.stream_nnz];
  uint64_t full[kStages];
};

// A tile of the stream: operator + tile id.
struct TileRef {
  const Tile* tile;
  int op;  // 0 = K (dual), 1 = K^T (primal)
};

// ---------------------------------------------------------------------------
// Tile computation from a staged copy. STREAM rows are summed in index order
// (bitwise equal to the reference's spmv, like spmv_engine.cuh); WARP/CHUNK rows
// use a fixed lane-strided order with a fixed butterfly (deterministic).
// ---------------------------------------------------------------------------
template <class Epi>
__device__ __forceinline__ void staged_tile(const Tile& t, const Stage& sg, double* prod,
                                            const Epi& epi, double (&red)[Epi::NR],
                                            double* chunk_part, unsigned* chunk_ctr) {
  const int tid = threadIdx.x;
  const int k0a = t.k0 & ~3;
  if (t.kind == kTileStream) {
    const int r0a = t.row0 & ~3;
    const int nq = (t.k1 - k0a + 3) >> 2;
    constexpr int U = 3;  // kStageNnz / 4 <= 3 * kThreads
    double g[U][4];
    double v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = tid + u * kThreads;
      if (q < nq) {
        const int4 c4 = *reinterpret_cast<const int4*>(sg.col + 4 * q);
        const double2 va = *reinterpret_cast<const double2*>(sg.val + 4 * q);
        const double2 vb = *reinterpret_cast<const double2*>(sg.val + 4 * q + 2);
        const int cs[4] = {c4.x, c4.y, c4.z, c4.w};
        v[u][0] = va.x, v[u][1] = va.y, v[u][2] = vb.x, v[u][3] = vb.y;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = k0a + 4 * q + i;
          double gg[1] = {0.0};
          if (e >= t.k0 && e < t.k1) epi.gather(cs[i], gg);
          g[u][i] = gg[0];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = tid + u * kThreads;
      if (q < nq) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = k0a + 4 * q + i;
          if (e >= t.k0 && e < t.k1) prod[e - t.k0] = v[u][i] * g[u][i];
        }
      }
    }
    __syncthreads();
    constexpr int RPT = kWinGeom.stream_rows / kThreads;  // round-robin rows (no bank conflicts)
    double acc[RPT][1];
    int nvalid = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = t.row0 + tid + i * kThreads;
      acc[i][0] = 0.0;
      if (r < t.row1) {
        nvalid = i + 1;
        const int a = sg.rp[r - r0a] - t.k0, b = sg.rp[r + 1 - r0a] - t.k0;
        for (int s2 = a; s2 < b; ++s2) acc[i][0] += prod[s2];
      }
    }
    epi.template rows_strided<RPT>(t.row0 + tid, kThreads, nvalid, acc, red);
  } else if (t.kind == kTileWarp) {
    const int r0a = t.row0 & ~3;
    const int G = t.part;
    const int grp = tid / G, lane = tid % G;
    const int r = t.row0 + grp;
    double acc = 0.0;
    if (r < t.row1) {
      const int a = sg.rp[r - r0a], b = sg.rp[r + 1 - r0a];
      // ~8 elements per lane: gathers first, then the ordered sum
      constexpr int U = 8;
      for (int e0 = a + lane; e0 < b; e0 += U * G) {
        double gv[U], vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * G;
          double gg[1] = {0.0};
          vv[u] = 0.0;
          if (e < b) {
            epi.gather(sg.col[e - k0a], gg);
            vv[u] = sg.val[e - k0a];
          }
          gv[u] = gg[0];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (e0 + u * G < b) acc += vv[u] * gv[u];
      }
    }
    const int width = G < 32 ? G : 32;
    for (int o = width >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (G > 32) {
      __shared__ double sgrp[kWarps];
      const int warp = tid >> 5;
      if ((tid & 31) == 0) sgrp[warp] = acc;
      __syncthreads();
      if (lane == 0) {
        double s = sgrp[warp];
        for (int w = 1; w < G / 32; ++w) s += sgrp[warp + w];
        acc = s;
      }
      __syncthreads();
    }
    if (lane == 0 && r < t.row1) {
      const double a1[1] = {acc};
      epi.row_done(r, a1, red);
    }
  } else {  // kTileChunk
    __shared__ double sred[kWarps];
    __shared__ bool last_part;
    double acc = 0.0;
    {
      constexpr int U = 8;  // kStageNnz <= U * kThreads
      double gv[U], vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = t.k0 + tid + u * kThreads;
        double gg[1] = {0.0};
        vv[u] = 0.0;
        if (e < t.k1) {
          epi.gather(sg.col[e - k0a], gg);
          vv[u] = sg.val[e - k0a];
        }
        gv[u] = gg[0];
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t.k0 + tid + u * kThreads < t.k1) acc += vv[u] * gv[u];
    }
    double a1[1] = {acc};
    block_sum<1>(a1, sred);
    if (t.nparts == 1) {
      if (tid == 0) epi.row_done(t.row0, a1, red);
    } else {
      if (tid == 0) {
        chunk_part[size_t(t.slot + t.part) * 8] = a1[0];
        __threadfence();
        const unsigned ticket = atomicAdd(chunk_ctr + t.row1, 1u);
        last_part = (ticket == unsigned(t.nparts - 1));
      }
      __syncthreads();
      if (last_part && tid == 0) {
        __threadfence();
        double tot[1] = {0.0};
        for (int p = 0; p < t.nparts; ++p) tot[0] += __ldcg(chunk_part + size_t(t.slot + p) * 8);
        chunk_ctr[t.row1] = 0u;
        // the row's reduction terms go to a fixed place (the first slice's
        // chunk slot), not into this CTA's partial: see WinBufs::k_split
        double rr[Epi::NR];
#pragma unroll
        for (int i = 0; i < Epi::NR; ++i) rr[i] = 0.0;
        epi.row_done(t.row0, tot, rr);
#pragma unroll
        for (int i = 0; i < Epi::NR; ++i) chunk_part[size_t(t.slot) * 8 + 1 + i] = rr[i];
      }
    }
  }
}

// adds the split rows' terms (fixed order) to the leader's sums
template <int NR>
__device__ __forceinline__ void add_split_terms(const DevCsr& op, const int* split, int nsplit, double (&sum)[NR]) {
  for (int s = 0; s < nsplit; ++s) {
    const Tile& t = op.tiles[split[s]];
#pragma unroll
    for (int i = 0; i < NR; ++i) sum[i] += __ldcg(op.chunk_part + size_t(t.slot) * 8 + 1 + i);
  }
}

// Grid barrier; the last CTA to arrive runs `leader()` (whole CTA) before the
// release. Every CTA leaves with its L1 invalidated (gpu-scope fence), so data
// written by other CTAs before the barrier is read fresh.
template <class F>
__device__ __forceinline__ void grid_barrier(GridBar* bar, unsigned nctas, F&& leader) {
  __shared__ unsigned s_gen;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_volatile(&bar->gen);
    __threadfence();
    const unsigned t = atomicAdd(&bar->count, 1u);
    s_last = (t == nctas - 1u);
    s_gen = g;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    leader();
    __syncthreads();
    if (threadIdx.x == 0) {
      bar->count = 0u;
      __threadfence();
      atomicAdd(&bar->gen, 1u);
    }
  } else if (threadIdx.x == 0) {
    while (ld_volatile(&bar->gen) == s_gen) __nanosleep(20);
  }
  if (threadIdx.x == 0) __threadfence();
  __syncthreads();
}

}  // namespace

template <bool kNonneg>
__global__ void __launch_bounds__(kThreads, 2) window_kernel(DevCsr K, DevCsr KT, DevIter it,
                                                              WinBufs wb) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WinSmem& sm = *reinterpret_cast<WinSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int cta = blockIdx.x, nctas = gridDim.x;
  DevState* st = it.st;

  // this CTA's tiles: round-robin over each operator's tile list
  const int nd = cta < K.ntiles ? (K.ntiles - cta + nctas - 1) / nctas : 0;
  const int np = cta < KT.ntiles ? (KT.ntiles - cta + nctas - 1) / nctas : 0;
  const int L = nd + np;
  auto tile_at = [&](long s, const DevCsr*& op) -> const Tile* {
    const int pos = int(s % L);
    if (pos < nd) {
      op = &K;
      return K.tiles + cta + pos * nctas;
    }
    op = &KT;
    return KT.tiles + cta + (pos - nd) * nctas;
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&sm.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // producer (thread 0): keep up to kStages tiles in flight ahead of the consumer
  long ps = 0, cs = 0;
  auto produce = [&]() {
    if (tid != 0 || L == 0) return;
    fence_proxy_async();  // the generic-proxy reads of a recycled stage are done
    while (ps - cs < kStages) {
      const DevCsr* op;
      const Tile* tp = tile_at(ps, op);
      const Tile t = *tp;
      Stage& sg = sm.stage[ps % kStages];
      const int k0a = t.k0 & ~3, k1a = (t.k1 + 3) & ~3;
      const uint32_t cbytes = uint32_t(k1a - k0a) * 4u, vbytes = uint32_t(k1a - k0a) * 8u;
      uint32_t rbytes = 0;
      int r0a = 0;
      if (t.kind != kTileChunk) {
        r0a = t.row0 & ~3;
        const int r1a = (t.row1 + 1 + 3) & ~3;
        rbytes = uint32_t(r1a - r0a) * 4u;
      }
      uint64_t* fb = &sm.full[ps % kStages];
      mbar_arrive_expect_tx(fb, cbytes + vbytes + rbytes);
      if (cbytes) {
        bulk_g2s(sg.col, op->col + k0a, cbytes, fb);
        bulk_g2s(sg.val, op->val + k0a, vbytes, fb);
      }
      if (rbytes) bulk_g2s(sg.rp, op->rp + r0a, rbytes, fb);
      ++ps;
    }
  };
  auto consume_begin = [&]() -> const Stage& {
    mbar_wait(&sm.full[cs % kStages], uint32_t((cs / kStages) & 1));
    return sm.stage[cs % kStages];
  };
  auto consume_end = [&]() {
    __syncthreads();  // every thread is done with this stage
    ++cs;
    produce();
  };
  produce();

  // the primal partials of the trial x' produced before this launch
  const double* p_src = wb.p_src;
  int p_count = wb.p_src_count;
  int p_window = wb.p_src_window;

  for (;;) {
    // ================= D phase (dual update of this trial) =================
    DualEpi<false, true> de;
    de.xg = it.x[st->ix_trial];
    de.y = it.y[st->iy_cur];
    de.kx = it.kx[st->ikx_cur];
    de.q = it.q;
    de.yt = it.y[st->iy_trial];
    de.kxt = it.kx[1 - st->ikx_cur];
    de.seq_dy2 = nullptr;
    de.seq_inter = nullptr;
    const double omega = st->omega, eta = st->eta;
    de.sigma = eta * omega;
    de.m1 = it.m1;
    double dred[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < nd; ++i) {
      const DevCsr* op;
      const Tile t = *tile_at(cs, op);
      const Stage& sg = consume_begin();
      staged_tile(t, sg, sm.prod, de, dred, K.chunk_part, K.chunk_ctr);
      consume_end();
    }
    store_partial<3, 0>(dred, wb.wd_part, cta, nctas);

    // ---- barrier + step decision by the last CTA (solver.hpp:436-466) ----
    grid_barrier(wb.bar, unsigned(nctas), [&]() {
      double dp[3], pp[2];
      sum_partials<3, 0>(wb.wd_part, nctas, dp);
      sum_partials<2, 0>(p_src, p_count, pp);
      if (threadIdx.x != 0) return;
      add_split_terms<3>(K, wb.k_split, wb.k_nsplit, dp);
      if (p_window) add_split_terms<2>(KT, wb.kt_split, wb.kt_nsplit, pp);
      const double dy2 = dp[0], inter = dp[1], dx2 = pp[0];
      const bool finite = dp[2] == 0.0 && pp[1] == 0.0;
      int cont = 0;
      st->trials_total += 1;
      st->trials_in_step += 1;
      if (!finite) {
        st->failure = 1;
        st->p_mode = kPNone;
      } else {
        const double movement = omega * dx2 + dy2 / omega;
        const double ia = fabs(inter);
        const double eta_bar = ia > 0.0 ? movement / (2.0 * ia) : INFINITY;
        const int64_t ti = st->total - st->table_base;
        const double eta_next = smin(it.red_tab[2 * ti] * eta_bar, it.red_tab[2 * ti + 1] * eta);
        if (eta <= eta_bar) {
          if (st->record_log) {
            pdlp_step_log_entry* log = reinterpret_cast<pdlp_step_log_entry*>(it.step_log);
            pdlp_step_log_entry e;
            e.step_counter = st->total + 1;
            e.omega = omega;
            e.eta_accepted = eta;
            e.eta_bar = eta_bar;
            e.eta_next = eta_next;
            e.movement_sq = movement;
            e.interaction = inter;
            log[st->window_accepts] = e;
          }
          st->eta_acc = eta;
          st->eta_bar = eta_bar;
          st->eta_next = eta_next;
          st->mov = movement;
          st->inter = inter;
          st->total += 1;
          st->inner += 1;
          st->window_accepts += 1;
          const double w = st->wsum + eta;
          st->wsum = w;
          st->avg_first = (w == eta) ? 1 : 0;
          st->avg_ratio = eta / w;
          int t0 = st->ix_prev;
          st->ix_prev = st->ix_cur;
          st->ix_cur = st->ix_trial;
          st->ix_trial = t0;
          t0 = st->iy_prev;
          st->iy_prev = st->iy_cur;
          st->iy_cur = st->iy_trial;
          st->iy_trial = t0;
          st->ikx_cur = 1 - st->ikx_cur;
          st->ikty_cur = 1 - st->ikty_cur;
          st->eta = eta_next;
          st->trials_in_step = 0;
          st->accepted = 1;
          st->p_mode = kPAccept;
          cont = st->window_accepts < st->window_target;
        } else {
          st->eta = eta_next;
          st->accepted = 0;
          if (!(eta_next > 0.0) || !isfinite(eta_next) || st->trials_in_step >= 80) {
            st->failure = 1;
            st->p_mode = kPNone;
          } else {
            st->p_mode = kPRetry;
            cont = 1;
          }
        }
      }
      st->window_cont = cont;
      __threadfence();
    });

    const int mode = st->p_mode;
    const int cont = st->window_cont;
    if (mode == kPNone) break;

    // ================= P phase ====================================================
    double pred[2] = {0.0, 0.0};
    const double tau = st->eta / st->omega;
    if (mode == kPAccept) {
      PrimalEpi<false, kNonneg, true> pe;
      pe.yg = it.y[st->iy_cur];
      pe.xc = it.x[st->ix_cur];
      pe.c = it.c;
      pe.l = it.l;
      pe.u = it.u;
      pe.kty_out = it.kty[st->ikty_cur];
      pe.store_kty = 1;
      pe.xt = it.x[st->ix_trial];
      pe.avg_x = it.avg_x;
      pe.seq_dx2 = nullptr;
      pe.tau = tau;
      pe.ratio = st->avg_ratio;
      pe.do_avg = 1;
      pe.avg_first = st->avg_first;
      for (int i = 0; i < np; ++i) {
        const DevCsr* op;
        const Tile t = *tile_at(cs, op);
        const Stage& sg = consume_begin();
        staged_tile(t, sg, sm.prod, pe, pred, KT.chunk_part, KT.chunk_ctr);
        consume_end();
      }
      // avg_y .add on this CTA's slice (solver.hpp:839)
      const int per = (it.m + nctas - 1) / nctas;
      const int i0 = cta * per, i1 = min(it.m, i0 + per);
      const double* yc = it.y[st->iy_cur];
      const double ratio = st->avg_ratio;
      const int first = st->avg_first;
      for (int i = i0 + tid; i < i1; i += kThreads)
        it.avg_y[i] = first ? yc[i] : it.avg_y[i] + ratio * (yc[i] - it.avg_y[i]);
    } else {  // kPRetry: x' for the shrunk step; the prefetched K^T tiles are skipped
      for (int i = 0; i < np; ++i) {
        consume_begin();
        consume_end();
      }
      const int per = (it.n + nctas - 1) / nctas;
      const int j0 = cta * per, j1 = min(it.n, j0 + per);
      const double* xc = it.x[st->ix_cur];
      const double* kty = it.kty[st->ikty_cur];
      double* xt = it.x[st->ix_trial];
      for (int j = j0 + tid; j < j1; j += kThreads) {
        const double xa = xc[j];
        const double v = xa - tau * (it.c[j] - kty[j]);
        const double xn = kNonneg ? smax(v, 0.0) : clamp_box(v, it.l[j], it.u[j]);
        xt[j] = xn;
        const double d = xn - xa;
        pred[0] += d * d;
        pred[1] += isfinite(xn) ? 0.0 : 1.0;
      }
    }
    store_partial<2, 0>(pred, wb.wp_part, cta, nctas);
    p_src = wb.wp_part;
    p_count = nctas;
    p_window = mode == kPRetry ? 0 : 1;  // a retry phase ran no split columns
    if (!cont) break;
    grid_barrier(wb.bar, unsigned(nctas), []() {});
  }
  // drain TMA copies still in flight before the CTA retires
  while (cs < ps) {
    consume_begin();
    ++cs;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

size_t window_smem_bytes() { return sizeof(WinSmem) + 128; }

int window_grid(int device) {
  int sms = 0, per = 0;
  PDLP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  PDLP_CUDA(cudaFuncSetAttribute(window_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(window_smem_bytes())));
  PDLP_CUDA(cudaFuncSetAttribute(window_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(window_smem_bytes())));
  PDLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, window_kernel<false>, kThreads,
                                                          window_smem_bytes()));
  int per2 = 0;
  PDLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, window_kernel<true>, kThreads,
                                                          window_smem_bytes()));
  per = std::min(std::min(per, per2), 2);
  if (per < 1) throw CudaError("window kernel does not fit on an SM");
  return sms * per;
}

void launch_window(const DevCsr& k, const DevCsr& kt, const DevIter& it, const WinBufs& wb,
                   int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = window_smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barriers
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (it.nonneg)
    PDLP_CUDA(cudaLaunchKernelEx(&cfg, window_kernel<true>, k, kt, it, wb));
  else
    PDLP_CUDA(cudaLaunchKernelEx(&cfg, window_kernel<false>, k, kt, it, wb));
}

}  // namespace pdlp
