// common.cuh — error handling and deterministic reduction helpers shared by
// the sm_100a kernels of the restarted-PDHG hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace pdlp {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

#define PDLP_CUDA(expr)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::pdlp::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" + \
                              __FILE__ + ":" + std::to_string(__LINE__));                \
  } while (0)

constexpr int kThreads = 256;        // CTA size of every tiled kernel
constexpr int kWarps = kThreads / 32;
constexpr int kStreamMaxRow = 128;   // rows up to this length go to STREAM tiles (C3: dual 189 -> 145 us vs 32)
constexpr int kWarpMaxRow = 4096;    // (32, 4096] -> a lane group per row (tiles.h)
constexpr int kVecPad = 8;           // index/value arrays padded for 128-bit tail loads

// Tile geometry per kernel family (tiles.h). The iteration kernels take fat
// tiles (16 nnz per thread) so C2-sized operators run in about one wave; the
// evaluation kernels gather 4 values per nonzero and keep their staging small.
struct TileGeom {
  int stream_nnz;  // nnz per STREAM tile (staged products in shared memory)
  int stream_rows; // rows per STREAM tile = rows_per_thread * kThreads
  int lane_nnz;    // target nnz per lane in WARP tiles
  int chunk_nnz;   // nnz per CHUNK tile of a split row
};
#ifndef PDLP_ITER_ROWS
#define PDLP_ITER_ROWS 1024
#endif
constexpr TileGeom kIterGeom{4096, PDLP_ITER_ROWS, 16, 4096};
constexpr TileGeom kEvalGeom{1024, 1024, 8, 2048};
constexpr int kStreamNnz = 4096;     // largest STREAM tile of any geometry
constexpr int kStreamRows = 2048;

// ---------------------------------------------------------------------------
// IEEE helpers with the reference's semantics (libstdc++ std::min/std::max are
// ternaries that propagate a NaN first argument; CUDA fmin/fmax drop NaN).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__host__ __device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// Streaming loads of matrix data: read once per launch, so they bypass L1.
// (An L2 evict-first policy on them was measured: it evicts the operators that
// stay L2-resident across iterations on C2-sized problems, 8.2 -> 20.5 us per
// SpMV, and did not help the gather-bound C4 either.)
__device__ __forceinline__ int4 ld_stream_i4(const int* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_stream_i1(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream_d1(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

// Variants with an L2 evict-first cache policy, for matrix streams that will
// not be reused from L2 (the column-panel SpMV over operators far larger than
// L2, where the gathered vector slice must stay resident).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <bool kEF>
__device__ __forceinline__ int4 ld_stream_i4_t(const int* p) {
  if (!kEF) return ld_stream_i4(p);
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(l2_evict_first_policy()));
  return r;
}
template <bool kEF>
__device__ __forceinline__ int ld_stream_i1_t(const int* p) {
  if (!kEF) return ld_stream_i1(p);
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(r)
               : "l"(p), "l"(l2_evict_first_policy()));
  return r;
}
template <bool kEF>
__device__ __forceinline__ double ld_stream_d1_t(const double* p) {
  if (!kEF) return ld_stream_d1(p);
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(r)
               : "l"(p), "l"(l2_evict_first_policy()));
  return r;
}
template <bool kEF>
__device__ __forceinline__ double2 ld_stream_d2_t(const double* p) {
  if (!kEF) return ld_stream_d2(p);
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(l2_evict_first_policy()));
  return r;
}

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; everything before griddep_wait() must only touch data the
// predecessor does not write (static matrix, tile plan).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// Fixed-order warp sum (xor butterfly): identical result on every replay.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum of K doubles per thread; result valid in thread 0.
// Warp butterflies, then warp partials summed by thread 0 in warp order.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* smem /* kWarps*K */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) smem[warp * K + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double s = smem[i];
      for (int w = 1; w < kWarps; ++w) s += smem[w * K + i];
      v[i] = s;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block reduction: the first NS entries are summed, the last NM are
// max-reduced (maxima never see NaN: callers only store guarded comparisons).
template <int NS, int NM>
__device__ __forceinline__ void block_reduce(double (&v)[NS + NM], double* smem /* kWarps*(NS+NM) */) {
  constexpr int K = NS + NM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = i < NS ? warp_sum(v[i]) : warp_max(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) smem[warp * K + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double s = smem[i];
      for (int w = 1; w < kWarps; ++w) s = i < NS ? s + smem[w * K + i] : fmax(s, smem[w * K + i]);
      v[i] = s;
    }
  }
  __syncthreads();
}

}  // namespace pdlp
