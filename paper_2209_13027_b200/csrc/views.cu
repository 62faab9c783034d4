// Second-view construction on the device: the 8-neighbour LBP map of views.py:41-58
// (radius 1, strict neighbour > centre, bits clockwise from the top-left neighbour,
// bit n weighing 2^n, zero padding, code / 255). One thread per pixel, rows of a
// map read through the L1 (each input pixel is read by its 9 neighbours); float64
// division so the float32 result equals float32(code / 255.0) of the reference.
#include <algorithm>

#include "common.cuh"

namespace ddcca {

__global__ void lbp_kernel(const float* __restrict__ in, int64_t n, int p, int q, float* __restrict__ out) {
  const int64_t plane = (int64_t)p * q;
  const int64_t total = n * plane;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / plane;
    const int r = (int)((e - m * plane) / q), c = (int)(e - m * plane - (int64_t)r * q);
    const float* img = in + m * plane;
    const float ctr = img[(int64_t)r * q + c];
    constexpr int DY[8] = {-1, -1, -1, 0, 1, 1, 1, 0};
    constexpr int DX[8] = {-1, 0, 1, 1, 1, 0, -1, -1};
    int code = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int y = r + DY[b], x = c + DX[b];
      const float v = (y >= 0 && y < p && x >= 0 && x < q) ? __ldg(img + (int64_t)y * q + x) : 0.f;
      code |= (v > ctr) << b;
    }
    out[e] = (float)((double)code / 255.0);
  }
}

}  // namespace ddcca

using namespace ddcca;

extern "C" int ddcca_lbp(const float* images, int64_t n, int p, int q, float* out, void* stream) {
  if (n < 0 || p < 3 || q < 3) return fail(DDCCA_ESHAPE, "lbp_map needs at least a 3x3 image, got %dx%d", p, q);
  if (n == 0) return DDCCA_OK;
  const int64_t total = n * (int64_t)p * q;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  lbp_kernel<<<grid, 256, 0, as_stream(stream)>>>(images, n, p, q, out);
  return check_launch("lbp_kernel");
}
