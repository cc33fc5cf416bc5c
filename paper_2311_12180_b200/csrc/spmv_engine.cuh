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

// Epi concept:
//   static constexpr int NP, NA, NR; static constexpr bool kNeedCol;
//   __device__ void gather(int col, double (&g)[NP]) const;
//   __device__ void add(double (&acc)[NA], const double (&p)[NP], int col) const;
//   __device__ void row_done(int row, const double (&acc)[NA], double (&red)[NR]) const;

template <class Epi>
constexpr size_t stream_smem_bytes() {
  return size_t(kStreamNnz) * Epi::NP * sizeof(double) +
         (Epi::kNeedCol ? size_t(kStreamNnz) * sizeof(int) : 0) + 64;
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

// Strided partial sum over [k0, k1) by `nthreads` threads with lane index `t`,
// using aligned 128-bit loads of indices and values.
template <class Epi>
__device__ __forceinline__ void strided_partial(const Epi& epi, const int* __restrict__ col,
                                                const double* __restrict__ val, int k0, int k1,
                                                int t, int nthreads, double (&acc)[Epi::NA]) {
  zero_acc<Epi>(acc);
  const int base = k0 & ~3;
  const int nq = (k1 - base + 3) >> 2;
  for (int q = t; q < nq; q += nthreads) {
    const int k = base + 4 * q;
    const int4 c4 = ld_stream_i4(col + k);
    const double2 va = ld_stream_d2(val + k);
    const double2 vb = ld_stream_d2(val + k + 2);
    const int cs[4] = {c4.x, c4.y, c4.z, c4.w};
    const double vs[4] = {va.x, va.y, vb.x, vb.y};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = k + i;
      if (e >= k0 && e < k1) {
        double g[Epi::NP], p[Epi::NP];
        epi.gather(cs[i], g);
#pragma unroll
        for (int j = 0; j < Epi::NP; ++j) p[j] = vs[i] * g[j];
        epi.add(acc, p, cs[i]);
      }
    }
  }
}

// Processes one tile; `red` holds this thread's reduction terms.
// `chunk_part` ([chunk_slots][NA]) and `chunk_ctr` ([split_rows]) serve split rows.
template <class Epi, bool kSeq>
__device__ void run_tile(const Tile& t, const int* __restrict__ rp, const int* __restrict__ col,
                         const double* __restrict__ val, const Epi& epi, double (&red)[Epi::NR],
                         double* chunk_part, unsigned* chunk_ctr, unsigned char* smem) {
  const int tid = threadIdx.x;
  if (t.kind == kTileStream) {
    double* sprod = reinterpret_cast<double*>(smem);
    int* scol = reinterpret_cast<int*>(sprod + size_t(kStreamNnz) * Epi::NP);
    const int base = t.k0 & ~3;
    const int nq = (t.k1 - base + 3) >> 2;
    for (int q = tid; q < nq; q += kThreads) {
      const int k = base + 4 * q;
      const int4 c4 = ld_stream_i4(col + k);
      const double2 va = ld_stream_d2(val + k);
      const double2 vb = ld_stream_d2(val + k + 2);
      const int cs[4] = {c4.x, c4.y, c4.z, c4.w};
      const double vs[4] = {va.x, va.y, vb.x, vb.y};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = k + i;
        if (e >= t.k0 && e < t.k1) {
          double g[Epi::NP];
          epi.gather(cs[i], g);
          const int s = e - t.k0;
#pragma unroll
          for (int j = 0; j < Epi::NP; ++j) sprod[size_t(s) * Epi::NP + j] = vs[i] * g[j];
          if (Epi::kNeedCol) scol[s] = cs[i];
        }
      }
    }
    __syncthreads();
    for (int r = t.row0 + tid; r < t.row1; r += kThreads) {
      const int a = rp[r] - t.k0, b = rp[r + 1] - t.k0;
      double acc[Epi::NA];
      zero_acc<Epi>(acc);
      for (int s = a; s < b; ++s) {
        double p[Epi::NP];
#pragma unroll
        for (int j = 0; j < Epi::NP; ++j) p[j] = sprod[size_t(s) * Epi::NP + j];
        epi.add(acc, p, Epi::kNeedCol ? scol[s] : 0);
      }
      epi.row_done(r, acc, red);
    }
    __syncthreads();
  } else if (t.kind == kTileWarp) {
    const int warp = tid >> 5, lane = tid & 31;
    const int r = t.row0 + warp;
    if (r < t.row1) {
      const int k0 = rp[r], k1 = rp[r + 1];
      double acc[Epi::NA];
      if (kSeq) {
        if (lane == 0) row_sum_sequential(epi, col, val, k0, k1, acc);
      } else {
        strided_partial(epi, col, val, k0, k1, lane, 32, acc);
#pragma unroll
        for (int i = 0; i < Epi::NA; ++i) acc[i] = warp_sum(acc[i]);
      }
      if (lane == 0) epi.row_done(r, acc, red);
    }
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
    }
  }
}

// Block-reduces `red` in fixed order (NS sums then NM maxima) and writes it as
// partial `slot` (NS+NM doubles).
template <int NS, int NM>
__device__ __forceinline__ void store_partial(double (&red)[NS + NM], double* partials, int slot) {
  __shared__ double sred[kWarps * (NS + NM)];
  block_reduce<NS, NM>(red, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS + NM; ++i) partials[size_t(slot) * (NS + NM) + i] = red[i];
  }
}

// Grid-level "am I the last CTA" ticket; resets the counter for the next replay.
__device__ __forceinline__ bool grid_last_block(unsigned* counter, unsigned total) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == total - 1u);
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Fixed-order reduction of `count` partials of width NS+NM (single CTA); the
// result is valid in thread 0.
template <int NS, int NM>
__device__ __forceinline__ void sum_partials(const double* partials, int count, double (&out)[NS + NM]) {
  constexpr int K = NS + NM;
  constexpr int B = K <= 4 ? 8 : 2;  // loads in flight per thread
  __shared__ double sred[kWarps * K];
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = i < NS ? 0.0 : -INFINITY;
  for (int j0 = threadIdx.x; j0 < count; j0 += kThreads * B) {
    double v[B][K];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int j = j0 + b * kThreads;
#pragma unroll
      for (int i = 0; i < K; ++i)
        v[b][i] = j < count ? __ldcg(partials + size_t(j) * K + i) : (i < NS ? 0.0 : -INFINITY);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
#pragma unroll
      for (int i = 0; i < K; ++i) out[i] = i < NS ? out[i] + v[b][i] : fmax(out[i], v[b][i]);
    }
  }
  block_reduce<NS, NM>(out, sred);
}

}  // namespace pdlp
