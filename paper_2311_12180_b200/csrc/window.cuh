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
  int p_src_window;       // 1: p_src is wp_part (its split-column terms are in KT's chunk slots)
  GridBar* bar;
  // split rows of the window plans: the tile index of each one's first slice.
  // Their reduction terms sit in that slice's chunk slot (elements 1..NR) and
  // are added by the barrier leader in this order, so the sums do not depend
  // on which CTA finished a split row.
  const int* k_split;
  int k_nsplit;
  const int* kt_split;
  int kt_nsplit;
};

size_t window_smem_bytes();
int window_grid(int device);
void launch_window(const DevCsr& k, const DevCsr& kt, const DevIter& it, const WinBufs& wb,
                   int grid, cudaStream_t s);

}  // namespace pdlp
