// FFMA vs FFMA2 (fma.rn.f32x2, __ffma2_rn) in the conv inner-loop shape (diagnostic):
// 8 filters x 16 pixels per thread, weights from the constant bank (warp-uniform),
// x values from shared memory. Reports FLOP/s and instructions per FLOP.
#include <cuda_runtime.h>

#include <cstdio>

struct W {
  float w[7 * 8];  // one tap row: 7 taps x 8 filters
};

template <bool PAIR>
__global__ void __launch_bounds__(128, 3) k(W T, float* out, int iters) {
  __shared__ float sx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sx[i] = (i % 13) * 0.01f;
  __syncthreads();
  float acc[16][8];
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int g = 0; g < 8; ++g) acc[j][g] = 0.f;
  const int base = (threadIdx.x * 16) & 511;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    float x[22];
#pragma unroll
    for (int t4 = 0; t4 < 6; ++t4) {
      const float4 v = *reinterpret_cast<const float4*>(&sx[(base + 4 * t4 + (it & 7) * 4) & 1020]);
      if (4 * t4 + 0 < 22) x[4 * t4 + 0] = v.x - 0.5f;
      if (4 * t4 + 1 < 22) x[4 * t4 + 1] = v.y - 0.5f;
      if (4 * t4 + 2 < 22) x[4 * t4 + 2] = v.z - 0.5f;
      if (4 * t4 + 3 < 22) x[4 * t4 + 3] = v.w - 0.5f;
    }
    if (PAIR) {
#pragma unroll
      for (int b = 0; b < 7; ++b)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 xx = make_float2(x[j + b], x[j + b]);
#pragma unroll
          for (int g = 0; g < 8; g += 2) {
            const float2 ww = make_float2(T.w[b * 8 + g], T.w[b * 8 + g + 1]);
            float2 a = make_float2(acc[j][g], acc[j][g + 1]);
            a = __ffma2_rn(ww, xx, a);
            acc[j][g] = a.x;
            acc[j][g + 1] = a.y;
          }
        }
    } else {
#pragma unroll
      for (int b = 0; b < 7; ++b)
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j][g] = fmaf(T.w[b * 8 + g], x[j + b], acc[j][g]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int g = 0; g < 8; ++g) s += acc[j][g];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

int main() {
  W T;
  for (int i = 0; i < 56; ++i) T.w[i] = 0.001f * (i % 7) - 0.002f;
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 400, blocks = 148 * 3 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    for (int pair = 0; pair < 2; ++pair) {
      cudaEventRecord(a);
      if (pair) k<true><<<blocks, 128>>>(T, out, iters);
      else k<false><<<blocks, 128>>>(T, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double fl = 2.0 * 7 * 8 * 16 * (double)iters * blocks * 128;
      printf("%s: %.1f TFLOP/s\n", pair ? "FFMA2 (__ffma2_rn)" : "FFMA", fl / ms / 1e9);
    }
  }
  return 0;
}
