// l2_gather.cu — how much of the 126 MB L2 a random fp64 gather can use.
// For a vector of S MB: each thread gathers G random doubles (hashed indices)
// while streaming `stream_bytes_per_gather` of a large array (the matrix
// stream of a panel SpMV, optionally evict_first). Reports ns per gather and
// the implied DRAM bytes per gather from the timing model (printed GB/s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 l2_gather.cu -o l2_gather
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__device__ __forceinline__ double ld_stream(const double* p, int ef) {
  double v;
  if (ef) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  }
  else asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_gather(const double* p, int el) {
  double v;
  if (el) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  }
  else asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__global__ void gather_kernel(const double* x, uint32_t nx, const double* st, uint64_t nst, int per,
                              int stream_per, int ef, int el, uint32_t seed, double* out) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  for (int i = 0; i < per; ++i) {
    const uint32_t h = hash32(uint32_t(tid * per + i) ^ seed);
    acc += ld_gather(x + (h % nx), el);
    for (int s = 0; s < stream_per; ++s) {
      const uint64_t k = (tid + uint64_t(s + i * stream_per) * gridDim.x * blockDim.x) % nst;
      acc += ld_stream(st + k, ef);
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const size_t max_x = size_t(320) << 20;
  const size_t nst = size_t(1) << 28;  // 2 GB stream array
  double *x, *st, *out;
  cudaMalloc(&x, max_x);
  cudaMalloc(&st, nst * 8);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, max_x);
  cudaMemset(st, 0, nst * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = 148 * 8 * 4, per = 64;
  const double gathers = double(threads) * blocks * per;
  int sizes[] = {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 160, 320};
  for (int sp : {0, 1, 2}) {
    for (int ef = 0; ef < 2; ++ef) {
      for (int el = 0; el < 2; ++el) {
        if (sp == 0 && ef) continue;
        printf("stream %d doubles/gather, evict_first %d, evict_last %d\n", sp, ef, el);
        for (int mb : sizes) {
          const uint32_t nx = uint32_t((size_t(mb) << 20) / 8);
          // warm the vector into L2
          gather_kernel<<<blocks, threads>>>(x, nx, st, nst, per, sp, ef, el, 1u, out);
          float best = 1e30f;
          for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            gather_kernel<<<blocks, threads>>>(x, nx, st, nst, per, sp, ef, el, 7u + r, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          const double ns = best * 1e6 / gathers;
          const double gbs_stream = gathers * sp * 8.0 / (best * 1e-3) / 1e9;
          printf("  S=%4d MB  %.3f ms  %.4f ns/gather  gathers %.1f G/s  stream %.0f GB/s\n", mb, best, ns,
                 gathers / (best * 1e-3) / 1e9, gbs_stream);
        }
      }
    }
  }
  return 0;
}
