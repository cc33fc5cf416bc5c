// csr_build.cu — CsrMatrix::from_triplets and explicit_transpose on the GPU
// (sparse_matrix.hpp:57-108, :167-178; the step before
// the path, single-threaded O(nnz log nnz) on the host in the reference).
//
//   1. range check; the first offending triplet is reported with the
//      reference's message ("triplet i at (r, c) is outside a RxC matrix");
//   2. stable LSD radix sort of (row * cols + col) keys with the triplet index
//      as payload, so duplicates keep their input order;
//   3. duplicates summed sequentially in that order (one thread per run of
//      equal keys), exact zeros dropped, rows counted and scanned.
// Integer output (offsets, column indices) is bit-exact with the reference;
// values are bit-exact wherever a (row, col) pair occurs at most twice (the
// reference's per-row std::sort is unstable, so the summation order of three
// or more duplicates is unspecified there).
#include <limits>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdio>
#include <string>
#include <vector>

#include "../../include/pdlp_b200.h"
#include "common.cuh"

namespace pdlp {
void set_last_error(const std::string& msg);  // capi.cu

namespace {

template <class T>
struct Buf {
  T* p = nullptr;
  explicit Buf(size_t n) { PDLP_CUDA(cudaMalloc(&p, (n ? n : 1) * sizeof(T))); }
  ~Buf() {
    if (p) cudaFree(p);
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

__global__ void check_range_kernel(const int64_t* r, const int64_t* c, int64_t nt, int64_t rows,
                                   int64_t cols, unsigned long long* first_bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt; i += int64_t(gridDim.x) * blockDim.x)
    if (r[i] < 0 || r[i] >= rows || c[i] < 0 || c[i] >= cols) atomicMin(first_bad, (unsigned long long)i);
}

__global__ void make_keys_kernel(const int64_t* r, const int64_t* c, int64_t nt, int64_t cols,
                                 unsigned long long* key, int64_t* idx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt; i += int64_t(gridDim.x) * blockDim.x) {
    key[i] = (unsigned long long)(r[i] * cols + c[i]);
    idx[i] = i;
  }
}

// head[i] = 1 when sorted element i starts a run of equal keys
__global__ void run_heads_kernel(const unsigned long long* key, int64_t nt, int64_t* head) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt; i += int64_t(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// One thread per run: sum its values in input order, keep it when nonzero.
__global__ void fold_runs_kernel(const unsigned long long* key, const int64_t* idx, const double* v,
                                 const int64_t* head, const int64_t* run_of, int64_t nt, int64_t cols,
                                 double* run_val, int64_t* run_row, int64_t* run_col, int64_t* keep) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt; i += int64_t(gridDim.x) * blockDim.x) {
    if (!head[i]) continue;
    double s = v[idx[i]];
    for (int64_t j = i + 1; j < nt && key[j] == key[i]; ++j) s += v[idx[j]];
    const int64_t k = run_of[i];
    run_val[k] = s;
    run_row[k] = int64_t(key[i] / (unsigned long long)cols);
    run_col[k] = int64_t(key[i] % (unsigned long long)cols);
    keep[k] = s != 0.0 ? 1 : 0;
  }
}

__global__ void compact_kernel(const int64_t* keep, const int64_t* pos, int64_t runs, const double* run_val,
                               const int64_t* run_row, const int64_t* run_col, double* val, int64_t* col,
                               int64_t* row_count) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < runs; k += int64_t(gridDim.x) * blockDim.x)
    if (keep[k]) {
      val[pos[k]] = run_val[k];
      col[pos[k]] = run_col[k];
      atomicAdd(reinterpret_cast<unsigned long long*>(row_count + run_row[k]), 1ull);  // integer: order-free
    }
}

int grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return int(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

void csr_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* hr, const int64_t* hc,
                       const double* hv, int64_t* row_offsets, int64_t* col_indices, double* values,
                       int64_t* nnz_out) {
  if (rows < 0 || cols < 0 || nt < 0) throw std::invalid_argument("from_triplets: negative dimension");
  // the sort key is row * cols + col in 63 bits: distinct (row, col) pairs must
  // not alias (the reference's per-row sort has no such limit)
  if (cols > 0 && rows > std::numeric_limits<int64_t>::max() / cols)
    throw std::invalid_argument("from_triplets: rows * cols exceeds the 63-bit key range");
  cudaStream_t s;
  PDLP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{s};
  const size_t n = size_t(nt);
  Buf<int64_t> r(n), c(n), idx(n), idx2(n), head(n), run_of(n);
  Buf<double> v(n);
  Buf<unsigned long long> key(n), key2(n), bad(1);
  if (nt) {
    PDLP_CUDA(cudaMemcpyAsync(r.p, hr, n * 8, cudaMemcpyHostToDevice, s));
    PDLP_CUDA(cudaMemcpyAsync(c.p, hc, n * 8, cudaMemcpyHostToDevice, s));
    PDLP_CUDA(cudaMemcpyAsync(v.p, hv, n * 8, cudaMemcpyHostToDevice, s));
  }
  PDLP_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  check_range_kernel<<<grid(nt), 256, 0, s>>>(r.p, c.p, nt, rows, cols, bad.p);
  unsigned long long first_bad = 0;
  PDLP_CUDA(cudaMemcpyAsync(&first_bad, bad.p, 8, cudaMemcpyDeviceToHost, s));
  PDLP_CUDA(cudaStreamSynchronize(s));
  if (first_bad != ~0ull) {  // sparse_matrix.hpp:59-67
    const size_t i = size_t(first_bad);
    throw std::invalid_argument("triplet " + std::to_string(i) + " at (" + std::to_string(hr[i]) + ", " +
                                std::to_string(hc[i]) + ") is outside a " + std::to_string(rows) + "x" +
                                std::to_string(cols) + " matrix");
  }
  int64_t stored = 0;
  std::vector<int64_t> counts(size_t(rows) + 1, 0);
  if (nt) {
    make_keys_kernel<<<grid(nt), 256, 0, s>>>(r.p, c.p, nt, cols, key.p, idx.p);
    int end_bit = 1;
    const unsigned long long maxkey = (unsigned long long)(rows) * (unsigned long long)(cols);
    while (end_bit < 64 && (1ull << end_bit) < maxkey) ++end_bit;
    size_t tmp = 0;
    PDLP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, idx.p, idx2.p, nt, 0, end_bit, s));
    Buf<unsigned char> tmpb(tmp);
    PDLP_CUDA(cub::DeviceRadixSort::SortPairs(tmpb.p, tmp, key.p, key2.p, idx.p, idx2.p, nt, 0, end_bit, s));
    run_heads_kernel<<<grid(nt), 256, 0, s>>>(key2.p, nt, head.p);
    size_t tmp2 = 0;
    PDLP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, head.p, run_of.p, nt, s));
    Buf<unsigned char> tmpc(tmp2);
    PDLP_CUDA(cub::DeviceScan::ExclusiveSum(tmpc.p, tmp2, head.p, run_of.p, nt, s));
    int64_t last_head = 0, last_run = 0;
    PDLP_CUDA(cudaMemcpyAsync(&last_head, head.p + (n - 1), 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaMemcpyAsync(&last_run, run_of.p + (n - 1), 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
    const int64_t runs = last_run + last_head;
    const size_t nr = static_cast<size_t>(runs), nrows = static_cast<size_t>(rows) + 1;
    Buf<double> run_val{nr}, val{nr};
    Buf<int64_t> run_row{nr}, run_col{nr}, keep{nr}, pos{nr + 1}, col{nr}, rc{nrows};
    fold_runs_kernel<<<grid(nt), 256, 0, s>>>(key2.p, idx2.p, v.p, head.p, run_of.p, nt, cols, run_val.p,
                                              run_row.p, run_col.p, keep.p);
    size_t tmp3 = 0;
    PDLP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp3, keep.p, pos.p, runs, s));
    Buf<unsigned char> tmpd(tmp3);
    PDLP_CUDA(cub::DeviceScan::ExclusiveSum(tmpd.p, tmp3, keep.p, pos.p, runs, s));
    int64_t last_keep = 0, last_pos = 0;
    PDLP_CUDA(cudaMemcpyAsync(&last_keep, keep.p + (runs - 1), 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaMemcpyAsync(&last_pos, pos.p + (runs - 1), 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaMemsetAsync(rc.p, 0, (size_t(rows) + 1) * 8, s));
    compact_kernel<<<grid(runs), 256, 0, s>>>(keep.p, pos.p, runs, run_val.p, run_row.p, run_col.p, val.p,
                                              col.p, rc.p);
    PDLP_CUDA(cudaStreamSynchronize(s));
    stored = last_pos + last_keep;
    if (stored) {
      PDLP_CUDA(cudaMemcpyAsync(col_indices, col.p, size_t(stored) * 8, cudaMemcpyDeviceToHost, s));
      PDLP_CUDA(cudaMemcpyAsync(values, val.p, size_t(stored) * 8, cudaMemcpyDeviceToHost, s));
    }
    if (rows) PDLP_CUDA(cudaMemcpyAsync(counts.data(), rc.p, size_t(rows) * 8, cudaMemcpyDeviceToHost, s));
    PDLP_CUDA(cudaStreamSynchronize(s));
  }
  row_offsets[0] = 0;
  for (int64_t i = 0; i < rows; ++i) row_offsets[i + 1] = row_offsets[i] + counts[size_t(i)];
  *nnz_out = stored;
}

}  // namespace pdlp

extern "C" int pdlp_csr_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* r,
                                      const int64_t* c, const double* v, int32_t device,
                                      int64_t* row_offsets, int64_t* col_indices, double* values,
                                      int64_t* nnz_out) {
  if ((nt > 0 && (!r || !c || !v || !col_indices || !values)) || !row_offsets || !nnz_out) {
    pdlp::set_last_error("null argument");
    return PDLP_EINVAL;
  }
  try {
    PDLP_CUDA(cudaSetDevice(device));
    pdlp::csr_from_triplets(rows, cols, nt, r, c, v, row_offsets, col_indices, values, nnz_out);
    pdlp::set_last_error("");
    return PDLP_OK;
  } catch (const pdlp::CudaError& e) {
    pdlp::set_last_error(e.what());
    return PDLP_ECUDA;
  } catch (const std::invalid_argument& e) {
    pdlp::set_last_error(e.what());
    return PDLP_EINVAL;
  } catch (const std::exception& e) {
    pdlp::set_last_error(e.what());
    return PDLP_ERUNTIME;
  }
}
