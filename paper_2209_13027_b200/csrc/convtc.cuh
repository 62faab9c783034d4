// Tensor-core (tcgen05, 3xTF32) fused last-layer conv + sign hash + block histograms.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ddcca {

struct TcHistArgs {
  const float* in;
  int64_t n_maps;
  int p, q, top, left, l;  // map size, "same" padding, square window l x l
  int count, center;       // filters (<= 8), per-window centering
  int bh, bw, nby, nbx, kind, nbits;
  void* counts;
  int64_t gpr, row_stride, group_stride;
};

// DDCCA_ECONFIG when the shape is not covered (the caller falls back to the FFMA kernel).
int conv_hist_tc(const TcHistArgs& a, const float* pack_host, cudaStream_t st);

}  // namespace ddcca
