// window.cuh — host interface of the persistent window kernel (window.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_state.h"

namespace pdlp {

struct GridBar {
  unsigned count;
  unsigned gen;
};

struct WinBufs {
  double* wd_part;        // [grid * 3] per-CTA dual partials
  double* wp_part;        // [grid * 2] per-CTA primal partials
  const double* p_src;    // partials of the trial x' produced before the launch
  int p_src_count;
  GridBar* bar;
};

size_t window_smem_bytes();
int window_grid(int device);
void launch_window(const DevCsr& k, const DevCsr& kt, const DevIter& it, const WinBufs& wb,
                   int grid, cudaStream_t s);

}  // namespace pdlp
