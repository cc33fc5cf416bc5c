// shard.cuh — device side of row sharding: peer stores and
// BSP barriers over NVLink peer memory.
//
// Every rank keeps FULL-length iterate buffers (x, y) and runs only its own
// contiguous range of the global tile plans. A producer kernel writes each
// value it owns both locally and straight into every peer's copy (st.global to
// CUDA-IPC-mapped peer memory: the all-gather is fused into the kernel that
// computes the data, tile by tile), together with its per-tile reduction
// partials at their GLOBAL tile index. Its last CTA then publishes a per-kind
// epoch to every rank's flag slot. A consumer kernel waits until every rank's
// flag reached its own local epoch before it reads gathered data, so every
// rank sums the same partial array in the same order: decisions are identical
// on all ranks and the iterates are bitwise independent of the rank count.
#pragma once

#include "common.cuh"
#include "device_state.h"

namespace pdlp {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr unsigned long long kShardTimeoutNs = 30ull * 1000ull * 1000ull * 1000ull;

// Consumer: all CTAs wait until every rank published `kind` up to this rank's
// local count (the number of participating producer launches so far, equal on
// every rank). Returns false if a peer did not arrive within the timeout (the
// caller turns that into a numerical-error exit instead of a hang).
__device__ __forceinline__ bool shard_wait(ShardSync* sync, int world, int kind) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (int(threadIdx.x) < world) {
    const unsigned long long want = *reinterpret_cast<volatile unsigned long long*>(&sync->count[kind]);
    const unsigned long long* f = &sync->flag[kind][threadIdx.x];
    unsigned long long t0 = 0;
    while (ld_acquire_sys(f) < want) {
      const unsigned long long now = global_ns();
      if (!t0) {
        t0 = now;
      } else if (now - t0 > kShardTimeoutNs) {
        s_ok = 0;
        sync->timeout = 1;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  return s_ok != 0;
}

// Producer: every CTA makes its (peer) stores visible system-wide and takes a
// ticket; the last CTA bumps the local count and publishes it to every rank.
__device__ __forceinline__ void shard_signal(const ShardView* shv, ShardSync* sync, int world, int rank,
                                             int kind) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned t = atomicAdd(&sync->ticket[kind], 1u);
    s_last = (t == gridDim.x - 1u);
    if (s_last) {
      sync->ticket[kind] = 0u;
      __threadfence_system();
      const unsigned long long c = sync->count[kind] + 1ull;
      sync->count[kind] = c;
      for (int q = 0; q < world; ++q) st_release_sys(&shv->sync[q]->flag[kind][rank], c);
    }
  }
}

// Writes v to base_q[off] of every peer q != rank (the own copy is written by
// the caller). `field` selects one pointer array of the ShardView.
__device__ __forceinline__ void push_peers(double* const* field, int world, int rank, size_t off,
                                           double v) {
#pragma unroll 1
  for (int q = 0; q < world; ++q)
    if (q != rank) {
      double* b = reinterpret_cast<double*>(__ldg(reinterpret_cast<const unsigned long long*>(field + q)));
      b[off] = v;
    }
}

// push_peers restricted to the ranks of `mask` (bit q: rank q).
__device__ __forceinline__ void push_peers_mask(double* const* field, int world, int rank, size_t off, double v,
                                                unsigned mask) {
#pragma unroll 1
  for (int q = 0; q < world; ++q)
    if (q != rank && ((mask >> q) & 1u)) {
      double* b = reinterpret_cast<double*>(__ldg(reinterpret_cast<const unsigned long long*>(field + q)));
      b[off] = v;
    }
}

// Thread 0 holds a block-reduced partial of width W (after store_partial):
// copy it to every peer's (component-major) partial array at the same slot.
template <int W>
__device__ __forceinline__ void push_partial(double* const* field, int world, int rank, size_t base,
                                             size_t slot, size_t stride, const double (&v)[W]) {
  if (threadIdx.x != 0) return;
#pragma unroll
  for (int i = 0; i < W; ++i) push_peers(field, world, rank, base + size_t(i) * stride + slot, v[i]);
}

// push_partial for store_tile_partial's slots (the main slot gets `v`, the
// identity slot zeros / -inf)
template <int NS, int NM, class Slots>
__device__ __forceinline__ void push_tile_partial(double* const* field, int world, int rank, size_t base,
                                                  const Slots& ps, size_t stride,
                                                  const double (&v)[NS + NM]) {
  if (ps.main >= 0) push_partial<NS + NM>(field, world, rank, base, size_t(ps.main), stride, v);
  if (ps.ident >= 0) {
    double id[NS + NM];
#pragma unroll
    for (int i = 0; i < NS + NM; ++i) id[i] = i < NS ? 0.0 : -INFINITY;
    push_partial<NS + NM>(field, world, rank, base, size_t(ps.ident), stride, id);
  }
}

}  // namespace pdlp
