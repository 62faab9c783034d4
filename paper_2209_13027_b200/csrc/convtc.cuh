// Tensor-core (tcgen05 kind::f16, scaled two-term split) fused last-layer conv + sign hash + block histograms.
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
  float* resp;   // responses mode: float32 output (n_maps * count, p, q), filter-minor
  int dc_shift;  // responses mode: shift each map by its mean first (centered windows only)
};

constexpr int TC_FILTERS = 8;  // filter slots of the tensor-core kernel (zero-padded)

// Shapes the tensor-core kernel takes (else the caller uses the FFMA kernel).
bool conv_hist_tc_covers(const TcHistArgs& a);
// taps_dev: zero-mean taps [(dy * l + dx) * TC_FILTERS + f] in device memory (stream-ordered).
// DDCCA_ECONFIG when the shape is not covered.
int conv_hist_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st);
// The same tensor-core convolution writing float32 responses ("same" padding, stride 1).
bool conv_resp_tc_covers(const TcHistArgs& a);
int conv_resp_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st);

}  // namespace ddcca
