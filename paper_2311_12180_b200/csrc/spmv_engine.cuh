// spmv_engine.cuh — the tiled CSR engine every fused kernel is built on.
//
// One CTA processes one Tile (tiles.h). The engine computes, for every row r of
// the tile, acc_r = sum_k v_k * g(col_k) where g gathers NP doubles per column
// (1 for the iteration kernels, 4 for the evaluation kernels, which carry four
// points side by side so one pass over the matrix serves all of them), and
// hands (r, acc_r) to the epilogue exactly once. The epilogue performs the fused
// projected update and accumulates NR reduction terms per thread; the engine
// block-sums those in a fixed order and stores one partial per tile.
#pragma once

#include "common.cuh"
#include "tiles.h"

namespace pdlp {

#ifndef PDLP_SHIFT_UNROLL
#define PDLP_SHIFT_UNROLL 4
#endif
constexpr int kShiftUnroll = PDLP_SHIFT_UNROLL;  // elements in flight per lane in shifted-row groups

// what run_tile did with the tile's reduction terms (see store_tile_partial)
enum PartialRole : int { kRoleOwn = 0, kRoleSlice = 1, kRoleSliceLast = 2 };

// Epilogues opt in to L2 evict-first matrix streams with
// `static constexpr bool kEvictFirst` (column-panel passes only).
template <class Epi, class = void>
struct has_evict_first { static constexpr bool value = false; };
template <class Epi>
struct has_evict_first<Epi, decltype(void(Epi::kEvictFirst))> { static constexpr bool value = Epi::kEvictFirst; };
template <class Epi>
__host__ __device__ constexpr bool evict_first() { return has_evict_first<Epi>::value; }


// Epi concept:
//   static constexpr int NP, NA, NR; static constexpr bool kNeedCol;
//   __device__ void gather(int col, double (&g)[NP]) const;
//   __device__ void add(double (&acc)[NA], const double (&p)[NP], int col) const;
//   __device__ void row_done(int row, const double (&acc)[NA], double (&red)[NR]) const;

template <class Epi>
constexpr size_t stream_smem_bytes() {
  return size_t(Epi::kGeom.stream_nnz) * Epi::NP * sizeof(double) +
         (Epi::kNeedCol ? size_t(Epi::kGeom.stream_nnz) * sizeof(int) : 0) + 64;
}

template <class Epi>
__device__ __forceinline__ void zero_acc(double (&a)[Epi::NA]) {
#pragma unroll
  for (int i = 0; i < Epi::NA; ++i) a[i] = 0.0;
}

// Sequential (reference-order) sum of one row straight from global memory.
template <class Epi>
__device__ __forceinline__ void row_sum_sequential(const Epi& epi, const int* __restrict__ col,
                                                   const double* __restrict__ val, int k0, int k1,
                                                   double (&acc)[Epi::NA]) {
  zero_acc<Epi>(acc);
  for (int k = k0; k < k1; ++k) {
    const int c = col[k];
    double g[Epi::NP], p[Epi::NP];
    epi.gather(c, g);
    const double v = val[k];
#pragma unroll
    for (int i = 0; i < Epi::NP; ++i) p[i] = v * g[i];
    epi.add(acc, p, c);
  }
}

// CRTP base: the default group epilogue hands each row to row_done. Epilogues
// that touch several dense arrays per row override rows_done to use 128-bit
// loads over the 4 consecutive rows one thread owns in a STREAM tile.
template <class D>
struct EpiBase {
  template <int NA, int NR>
  __device__ __forceinline__ void rows_done(int r0, int nr, const double (&acc)[4][NA],
                                            double (&red)[NR]) const {
    for (int i = 0; i < nr; ++i) static_cast<const D*>(this)->row_done(r0 + i, acc[i], red);
  }
  // rows r0 + i * stride, i < nvalid (the STREAM tile's round-robin rows)
  template <int RPT, int NA, int NR>
  __device__ __forceinline__ void rows_strided(int r0, int stride, int nvalid,
                                               const double (&acc)[RPT][NA],
                                               double (&red)[NR]) const {
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < nvalid) static_cast<const D*>(this)->row_done(r0 + i * stride, acc[i], red);
  }
};

// Loads in flight per lane: 2 quads (8 nnz) per batch for the scalar-gather kernels.
#ifndef PDLP_QUAD_UNROLL
#define PDLP_QUAD_UNROLL 2
#endif
template <class Epi>
__host__ __device__ constexpr int quad_unroll() { return Epi::NP == 1 ? PDLP_QUAD_UNROLL : 1; }

// Strided partial sum over [k0, k1) by `nthreads` threads with lane index `t`,
// using aligned 128-bit loads of indices and values; U quads of index/value
// loads are issued before their gathers so each lane keeps ~3U+4U requests in
// flight. Each lane accumulates its quads in increasing order (deterministic).
template <class Epi>
__device__ __forceinline__ void strided_partial(const Epi& epi, const int* __restrict__ col,
                                                const double* __restrict__ val, int k0, int k1,
                                                int t, int nthreads, double (&acc)[Epi::NA]) {
  constexpr int U = quad_unroll<Epi>();
  zero_acc<Epi>(acc);
  const int base = k0 & ~3;
  const int nq = (k1 - base + 3) >> 2;
  for (int q0 = t; q0 < nq; q0 += nthreads * U) {
    int cs[U][4];
    double vs[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * nthreads;
      if (q < nq) {
        const int k = base + 4 * q;
        const int4 c4 = ld_stream_i4_t<evict_first<Epi>()>(col + k);
        const double2 va = ld_stream_d2_t<evict_first<Epi>()>(val + k);
        const double2 vb = ld_stream_d2_t<evict_first<Epi>()>(val + k + 2);
        cs[u][0] = c4.x, cs[u][1] = c4.y, cs[u][2] = c4.z, cs[u][3] = c4.w;
        vs[u][0] = va.x, vs[u][1] = va.y, vs[u][2] = vb.x, vs[u][3] = vb.y;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) cs[u][i] = 0, vs[u][i] = 0.0;
      }
    }
    double g[U][4][Epi::NP];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + 4 * (q0 + u * nthreads);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = k + i;
        if (e >= k0 && e < k1) epi.gather(cs[u][i], g[u][i]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + 4 * (q0 + u * nthreads);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = k + i;
        if (e >= k0 && e < k1) {
          double p[Epi::NP];
#pragma unroll
          for (int j = 0; j < Epi::NP; ++j) p[j] = vs[u][i] * g[u][i][j];
          epi.add(acc, p, cs[u][i]);
        }
      }
    }
  }
}

// Element-interleaved partial sum over [k0, k1): lane t takes elements
// k0 + t, k0 + t + nthreads, ... so neighbouring lanes gather neighbouring
// columns (one L1 wavefront per 32 gathers when a row's columns are
// contiguous, instead of one per quad-strided lane). Used for WARP tiles whose
// rows the planner found column-contiguous (Tile::slot == 1).
template <class Epi, int U = 4>
__device__ __forceinline__ void elem_partial(const Epi& epi, const int* __restrict__ col,
                                             const double* __restrict__ val, int k0, int k1, int t,
                                             int nthreads, double (&acc)[Epi::NA]) {
  zero_acc<Epi>(acc);
  for (int e0 = k0 + t; e0 < k1; e0 += nthreads * U) {
    int cs[U];
    double vs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nthreads;
      cs[u] = e < k1 ? ld_stream_i1_t<evict_first<Epi>()>(col + e) : 0;
      vs[u] = e < k1 ? ld_stream_d1_t<evict_first<Epi>()>(val + e) : 0.0;
    }
    double g[U][Epi::NP];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * nthreads < k1) epi.gather(cs[u], g[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * nthreads < k1) {
        double p[Epi::NP];
#pragma unroll
        for (int j = 0; j < Epi::NP; ++j) p[j] = vs[u] * g[u][j];
        epi.add(acc, p, cs[u]);
      }
  }
}

// Pulls a tile's static operator data (offsets, indices, values) toward L2
// before griddep_wait(), so the loads after it overlap the predecessor's tail.
__device__ __forceinline__ void prefetch_tile(const Tile& t, const int* rp, const int* col,
                                              const double* val) {
  const int k0 = t.k0 & ~31, k1 = t.k1;
  // 128-byte lines: 32 indices or 16 values per line
  for (int k = k0 + 32 * int(threadIdx.x); k < k1; k += 32 * kThreads) prefetch_l2(col + k);
  for (int k = (t.k0 & ~15) + 16 * int(threadIdx.x); k < k1; k += 16 * kThreads) prefetch_l2(val + k);
  if (t.kind == kTileWarp || (t.kind == kTileStream && t.part == 0)) {
    const int r = (t.row0 & ~31) + 32 * int(threadIdx.x);
    if (r <= t.row1) prefetch_l2(rp + r);
  }
}

// Epilogues opt in to the uniform-row path with `static constexpr bool kUniform`
// (it costs registers; the dual kernel's K rows are rarely uniform).
template <class Epi, class = void>
struct has_uniform { static constexpr bool value = false; };
template <class Epi>
struct has_uniform<Epi, decltype(void(Epi::kUniform))> { static constexpr bool value = Epi::kUniform; };
template <class Epi>
__host__ __device__ constexpr bool uniform_ok() { return has_uniform<Epi>::value; }

// STREAM tile whose rows all have the same short length L (Tile::part): each
// thread sums its round-robin rows straight from global memory in index order
// (bitwise the staged path's result) without the shared-memory staging pass.
// Rows are processed in pairs so a thread keeps 2L loads and gathers in flight.
template <class Epi, int L>
__device__ __forceinline__ void uniform_rows(const Tile& t, const int* __restrict__ col,
                                             const double* __restrict__ val, const Epi& epi,
                                             double (&red)[Epi::NR]) {
  constexpr int RPT = Epi::kGeom.stream_rows / kThreads;
  constexpr int PAIR = L <= 4 ? 2 : 1;
  const int tid = threadIdx.x;
  double acc[RPT][Epi::NA];
  int nvalid = 0;
#pragma unroll
  for (int i0 = 0; i0 < RPT; i0 += PAIR) {
    int cs[PAIR][L];
    double vs[PAIR][L];
    double g[PAIR][L][Epi::NP];
#pragma unroll
    for (int h = 0; h < PAIR; ++h) {
      const int r = t.row0 + tid + (i0 + h) * kThreads;
      const int k = t.k0 + (r - t.row0) * L;
#pragma unroll
      for (int j = 0; j < L; ++j) {
        cs[h][j] = r < t.row1 ? ld_stream_i1_t<evict_first<Epi>()>(col + k + j) : 0;
        vs[h][j] = r < t.row1 ? ld_stream_d1_t<evict_first<Epi>()>(val + k + j) : 0.0;
      }
    }
#pragma unroll
    for (int h = 0; h < PAIR; ++h) {
      const int r = t.row0 + tid + (i0 + h) * kThreads;
#pragma unroll
      for (int j = 0; j < L; ++j)
        if (r < t.row1) epi.gather(cs[h][j], g[h][j]);
    }
#pragma unroll
    for (int h = 0; h < PAIR; ++h) {
      const int i = i0 + h;
      const int r = t.row0 + tid + i * kThreads;
#pragma unroll
      for (int a = 0; a < Epi::NA; ++a) acc[i][a] = 0.0;
      if (r < t.row1) {
        nvalid = i + 1;
#pragma unroll
        for (int j = 0; j < L; ++j) {
          double p[Epi::NP];
#pragma unroll
          for (int q = 0; q < Epi::NP; ++q) p[q] = vs[h][j] * g[h][j][q];
          epi.add(acc[i], p, cs[h][j]);
        }
      }
    }
  }
  epi.template rows_strided<RPT>(t.row0 + tid, kThreads, nvalid, acc, red);
}

// Uniform short rows for wide epilogues (several points per gather, 4-8 sums
// per row: the evaluation kernels): one row at a time, index order.
template <class Epi, int L>
__device__ __forceinline__ void uniform_rows_wide(const Tile& t, const int* __restrict__ col,
                                                  const double* __restrict__ val, const Epi& epi,
                                                  double (&red)[Epi::NR]) {
  constexpr int RPT = Epi::kGeom.stream_rows / kThreads;
#pragma unroll 1
  for (int i = 0; i < RPT; ++i) {
    const int r = t.row0 + threadIdx.x + i * kThreads;
    if (r >= t.row1) break;
    const int k = t.k0 + (r - t.row0) * L;
    int cs[L];
    double vs[L], g[L][Epi::NP];
#pragma unroll
    for (int j = 0; j < L; ++j) {
      cs[j] = ld_stream_i1_t<evict_first<Epi>()>(col + k + j);
      vs[j] = ld_stream_d1_t<evict_first<Epi>()>(val + k + j);
    }
#pragma unroll
    for (int j = 0; j < L; ++j) epi.gather(cs[j], g[j]);
    double acc[Epi::NA];
    zero_acc<Epi>(acc);
#pragma unroll
    for (int j = 0; j < L; ++j) {
      double p[Epi::NP];
#pragma unroll
      for (int q = 0; q < Epi::NP; ++q) p[q] = vs[j] * g[j][q];
      epi.add(acc, p, cs[j]);
    }
    epi.row_done(r, acc, red);
  }
}

// Processes one tile; `red` holds this thread's reduction terms.
// `chunk_part` ([chunk_slots][NA]) and `chunk_ctr` ([split_rows]) serve split rows.
// Returns the tile's partial role for store_tile_partial (kRoleOwn, or for a
// slice of a split row kRoleSlice / kRoleSliceLast).
template <class Epi, bool kSeq>
__device__ int run_tile(const Tile& t, const int* __restrict__ rp, const int* __restrict__ col,
                         const double* __restrict__ val, const Epi& epi, double (&red)[Epi::NR],
                         double* chunk_part, unsigned* chunk_ctr, unsigned char* smem) {
  const int tid = threadIdx.x;
  if constexpr (Epi::NA > 2) {
    if (t.kind == kTileStream && t.part >= 1 && t.part <= 4 && uniform_ok<Epi>()) {
      switch (t.part) {
        case 1: uniform_rows_wide<Epi, 1>(t, col, val, epi, red); return kRoleOwn;
        case 2: uniform_rows_wide<Epi, 2>(t, col, val, epi, red); return kRoleOwn;
        case 3: uniform_rows_wide<Epi, 3>(t, col, val, epi, red); return kRoleOwn;
        default: uniform_rows_wide<Epi, 4>(t, col, val, epi, red); return kRoleOwn;
      }
    }
  }
  if (t.kind == kTileStream && t.part >= 1 && t.part <= 5 && Epi::NP == 1 && Epi::NA <= 2 && uniform_ok<Epi>()) {
    switch (t.part) {
      case 1: uniform_rows<Epi, 1>(t, col, val, epi, red); return kRoleOwn;
      case 2: uniform_rows<Epi, 2>(t, col, val, epi, red); return kRoleOwn;
      case 3: uniform_rows<Epi, 3>(t, col, val, epi, red); return kRoleOwn;
      case 4: uniform_rows<Epi, 4>(t, col, val, epi, red); return kRoleOwn;
      default: uniform_rows<Epi, 5>(t, col, val, epi, red); return kRoleOwn;
    }
  }
  if (t.kind == kTileStream) {
    constexpr int U = quad_unroll<Epi>() > 2 ? 2 : quad_unroll<Epi>();
    double* sprod = reinterpret_cast<double*>(smem);
    int* scol = reinterpret_cast<int*>(sprod + size_t(Epi::kGeom.stream_nnz) * Epi::NP);
    const int base = t.k0 & ~3;
    const int nq = (t.k1 - base + 3) >> 2;
    for (int q0 = tid; q0 < nq; q0 += kThreads * U) {
      int cs[U][4];
      double vs[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * kThreads;
        if (q < nq) {
          const int k = base + 4 * q;
          const int4 c4 = ld_stream_i4_t<evict_first<Epi>()>(col + k);
          const double2 va = ld_stream_d2_t<evict_first<Epi>()>(val + k);
          const double2 vb = ld_stream_d2_t<evict_first<Epi>()>(val + k + 2);
          cs[u][0] = c4.x, cs[u][1] = c4.y, cs[u][2] = c4.z, cs[u][3] = c4.w;
          vs[u][0] = va.x, vs[u][1] = va.y, vs[u][2] = vb.x, vs[u][3] = vb.y;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) cs[u][i] = 0, vs[u][i] = 0.0;
        }
      }
      double g[U][4][Epi::NP];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + 4 * (q0 + u * kThreads);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = k + i;
          if (e >= t.k0 && e < t.k1) epi.gather(cs[u][i], g[u][i]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + 4 * (q0 + u * kThreads);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = k + i;
          if (e >= t.k0 && e < t.k1) {
            const int s = e - t.k0;
#pragma unroll
            for (int j = 0; j < Epi::NP; ++j) sprod[size_t(s) * Epi::NP + j] = vs[u][i] * g[u][i][j];
            if (Epi::kNeedCol) scol[s] = cs[u][i];
          }
        }
      }
    }
    __syncthreads();
    // rows are dealt round-robin (thread t: rows row0 + t + i * kThreads), so a
    // warp reads neighbouring products from shared memory (no bank conflicts)
    // and neighbouring epilogue operands from HBM (coalesced); each row is
    // summed in index order
    constexpr int RPT = Epi::kGeom.stream_rows / kThreads;
    if constexpr (Epi::NA > 2) {
      // wide accumulators (the evaluation epilogues carry 4-8 sums per row):
      // finish each row before the next so only one row's sums are live
#pragma unroll 1
      for (int i = 0; i < RPT; ++i) {
        const int r = t.row0 + tid + i * kThreads;
        if (r >= t.row1) break;
        double acc1[Epi::NA];
        zero_acc<Epi>(acc1);
        const int a = t.part ? (r - t.row0) * t.part : rp[r] - t.k0;
        const int b = t.part ? a + t.part : rp[r + 1] - t.k0;
        for (int s = a; s < b; ++s) {
          double p[Epi::NP];
#pragma unroll
          for (int j = 0; j < Epi::NP; ++j) p[j] = sprod[size_t(s) * Epi::NP + j];
          epi.add(acc1, p, Epi::kNeedCol ? scol[s] : 0);
        }
        epi.row_done(r, acc1, red);
      }
    } else {
      double acc[RPT][Epi::NA];
      int nvalid = 0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = t.row0 + tid + i * kThreads;
#pragma unroll
        for (int j = 0; j < Epi::NA; ++j) acc[i][j] = 0.0;
        if (r < t.row1) {
          nvalid = i + 1;
          const int a = t.part ? (r - t.row0) * t.part : rp[r] - t.k0;
          const int b = t.part ? a + t.part : rp[r + 1] - t.k0;
          for (int s = a; s < b; ++s) {
            double p[Epi::NP];
#pragma unroll
            for (int j = 0; j < Epi::NP; ++j) p[j] = sprod[size_t(s) * Epi::NP + j];
            epi.add(acc[i], p, Epi::kNeedCol ? scol[s] : 0);
          }
        }
      }
      epi.template rows_strided<RPT>(t.row0 + tid, kThreads, nvalid, acc, red);
    }
    __syncthreads();
  } else if (t.kind == kTileWarp && t.slot == 2 && !kSeq) {
    // Four column-shifted rows (row r0 + i has the columns of row r0 shifted by
    // +i, e.g. the demand rows of a transportation LP): thread t works on row
    // t % 4, elements t / 4, t / 4 + 64, ...; the four lanes that share an
    // element index gather x[c], x[c+1], x[c+2], x[c+3] from one 32-byte sector.
    const int r = t.row0 + (tid & 3);
    double acc[Epi::NA];
    zero_acc<Epi>(acc);
    elem_partial<Epi, kShiftUnroll>(epi, col, val, rp[r], rp[r + 1], tid >> 2, kThreads / 4, acc);
    __shared__ double sgrp4[kWarps * 4 * Epi::NA];
#pragma unroll
    for (int i = 0; i < Epi::NA; ++i) {
      double v = acc[i];
      for (int o = 16; o >= 4; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // same row
      acc[i] = v;
    }
    const int warp = tid >> 5, lane32 = tid & 31;
    if (lane32 < 4) {
#pragma unroll
      for (int i = 0; i < Epi::NA; ++i) sgrp4[(warp * 4 + lane32) * Epi::NA + i] = acc[i];
    }
    __syncthreads();
    if (tid < 4) {
#pragma unroll
      for (int i = 0; i < Epi::NA; ++i) {
        double v = sgrp4[tid * Epi::NA + i];
        for (int w = 1; w < kWarps; ++w) v += sgrp4[(w * 4 + tid) * Epi::NA + i];
        acc[i] = v;
      }
      epi.row_done(t.row0 + tid, acc, red);
    }
    __syncthreads();
  } else if (t.kind == kTileWarp) {
    // G lanes per row (t.part in {8,...,256}, ~8 nnz per lane: one batch of
    // loads), kThreads / G rows per tile; lane partials combine by a fixed
    // butterfly inside the warp, then warps of a group in warp order.
    const int G = t.part;
    const int grp = tid / G, lane = tid % G;
    const int r = t.row0 + grp;
    double acc[Epi::NA];
    zero_acc<Epi>(acc);
    if (r < t.row1) {
      const int k0 = rp[r], k1 = rp[r + 1];
      if (kSeq) {
        if (lane == 0) row_sum_sequential(epi, col, val, k0, k1, acc);
      } else if (t.slot == 1) {
        elem_partial(epi, col, val, k0, k1, lane, G, acc);
      } else {
        strided_partial(epi, col, val, k0, k1, lane, G, acc);
      }
    }
    if (!kSeq) {
      const int width = G < 32 ? G : 32;
#pragma unroll
      for (int i = 0; i < Epi::NA; ++i) {
        double v = acc[i];
        for (int o = width >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[i] = v;
      }
      if (G > 32) {
        __shared__ double sgrp[kWarps * Epi::NA];
        const int warp = tid >> 5;
        if ((tid & 31) == 0) {
#pragma unroll
          for (int i = 0; i < Epi::NA; ++i) sgrp[warp * Epi::NA + i] = acc[i];
        }
        __syncthreads();
        if (lane == 0) {
          const int w0 = warp, nw = G / 32;
#pragma unroll
          for (int i = 0; i < Epi::NA; ++i) {
            double v = sgrp[w0 * Epi::NA + i];
            for (int w = 1; w < nw; ++w) v += sgrp[(w0 + w) * Epi::NA + i];
            acc[i] = v;
          }
        }
        __syncthreads();
      }
    }
    if (lane == 0 && r < t.row1) epi.row_done(r, acc, red);
  } else {  // kTileChunk
    __shared__ double sred[kWarps * Epi::NA];
    __shared__ bool last_part;
    double acc[Epi::NA];
    if (kSeq) {
      if (tid == 0) row_sum_sequential(epi, col, val, t.k0, t.k1, acc);
    } else {
      strided_partial(epi, col, val, t.k0, t.k1, tid, kThreads, acc);
      block_sum<Epi::NA>(acc, sred);
    }
    if (t.nparts == 1) {
      if (tid == 0) epi.row_done(t.row0, acc, red);
    } else {
      if (tid == 0) {
        double* dst = chunk_part + size_t(t.slot + t.part) * Epi::NA;
#pragma unroll
        for (int i = 0; i < Epi::NA; ++i) dst[i] = acc[i];
        __threadfence();
        const unsigned ticket = atomicAdd(chunk_ctr + t.row1, 1u);
        last_part = (ticket == unsigned(t.nparts - 1));
      }
      __syncthreads();
      if (last_part && tid == 0) {
        __threadfence();
        double tot[Epi::NA];
        zero_acc<Epi>(tot);
        for (int p = 0; p < t.nparts; ++p) {
          const double* src = chunk_part + size_t(t.slot + p) * Epi::NA;
#pragma unroll
          for (int i = 0; i < Epi::NA; ++i) tot[i] += __ldcg(src + i);
        }
        chunk_ctr[t.row1] = 0u;
        epi.row_done(t.row0, tot, red);
      }
      return last_part ? kRoleSliceLast : kRoleSlice;
    }
  }
  return kRoleOwn;
}

// Block-reduces `red` in fixed order (NS sums then NM maxima) and writes it as
// partial `slot`. Partial arrays are component-major ([NS+NM][stride], stride =
// the array's partial count), so sum_partials reads them coalesced.
template <int NS, int NM>
__device__ __forceinline__ void store_partial(double (&red)[NS + NM], double* partials, int slot,
                                              int stride) {
  __shared__ double sred[kWarps * (NS + NM)];
  block_reduce<NS, NM>(red, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS + NM; ++i) partials[size_t(i) * stride + slot] = red[i];
  }
}

// Where a tile's partial goes. A split row's reduction terms are added by
// whichever of its slice CTAs arrives last, so they are stored under the row's
// FIRST slice (and the other slices' partials hold the identity): the
// fixed-order partial sums then do not depend on arrival order, and repeated
// solves are bitwise identical.
struct PartialSlots {
  int main;   // slot receiving `red` (-1: none)
  int ident;  // slot receiving the identity (-1: none)
};
__device__ __forceinline__ PartialSlots partial_slots(const Tile& t, int role, int tile) {
  if (role == kRoleOwn) return {tile, -1};
  const int first = tile - t.part;
  if (role == kRoleSliceLast) return {first, t.part > 0 ? tile : -1};
  return {-1, t.part > 0 ? tile : -1};  // the first slice's slot is the last CTA's
}

template <int NS, int NM>
__device__ __forceinline__ PartialSlots store_tile_partial(double (&red)[NS + NM], double* partials,
                                                          const Tile& t, int role, int tile, int stride) {
  const PartialSlots ps = partial_slots(t, role, tile);
  if (ps.main >= 0) store_partial<NS, NM>(red, partials, ps.main, stride);
  if (ps.ident >= 0 && threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS + NM; ++i) partials[size_t(i) * stride + ps.ident] = i < NS ? 0.0 : -INFINITY;
  }
  return ps;
}

// Grid-level "am I the last CTA" ticket; resets the counter for the next replay.
__device__ __forceinline__ bool grid_last_block(unsigned* counter, unsigned total) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    // thread 0 wrote this CTA's partial; publish it before taking a ticket (a
    // fence in every thread would also flush every SM's L1 on sm_100)
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == total - 1u);
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Fixed-order reduction of the partials [j0, j1) of a component-major array
// with row stride `stride` (single CTA); the result is valid in thread 0.
template <int NS, int NM>
__device__ __forceinline__ void sum_partials_range(const double* partials, int stride, int j0, int j1,
                                                   double (&out)[NS + NM]) {
  constexpr int K = NS + NM;
  constexpr int B = K <= 4 ? 8 : 2;  // loads in flight per thread
  __shared__ double sred[kWarps * K];
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = i < NS ? 0.0 : -INFINITY;
  for (int jb = j0 + threadIdx.x; jb < j1; jb += kThreads * B) {
    double v[B][K];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int j = jb + b * kThreads;
#pragma unroll
      for (int i = 0; i < K; ++i)
        v[b][i] = j < j1 ? __ldcg(partials + size_t(i) * stride + j) : (i < NS ? 0.0 : -INFINITY);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
#pragma unroll
      for (int i = 0; i < K; ++i) out[i] = i < NS ? out[i] + v[b][i] : fmax(out[i], v[b][i]);
    }
  }
  block_reduce<NS, NM>(out, sred);
}

// All `count` partials of a component-major array of width NS+NM.
template <int NS, int NM>
__device__ __forceinline__ void sum_partials(const double* partials, int count, double (&out)[NS + NM]) {
  sum_partials_range<NS, NM>(partials, count, 0, count, out);
}

}  // namespace pdlp
