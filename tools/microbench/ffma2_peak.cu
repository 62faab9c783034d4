// Pure FP32 FMA throughput on sm_100a: scalar FFMA vs packed FFMA2 (fma.rn.f32x2), 16 independent
// accumulator chains per thread, 8 warps per SM quarter. Reports flop/clk/SM (clock64 per CTA).
#include <cuda_runtime.h>

#include <cstdio>

template <bool PAIR>
__global__ void __launch_bounds__(256) k(float* out, int iters, long long* cyc) {
  float a = threadIdx.x * 1e-3f, b = 0.999f;
  float acc[16];
  float2 acc2[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = i;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc2[i] = make_float2(i, i + 0.5f);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if constexpr (PAIR) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc2[i] = __ffma2_rn(make_float2(a, a), acc2[i], make_float2(b, b));
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(a, acc[i], b);
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc2[i].x + acc2[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  long long* c;
  cudaMalloc(&o, sms * 4 * 256 * 4);
  cudaMalloc(&c, sms * 4 * 8);
  const int iters = 4096, blocks = sms * 4;  // 4 CTAs x 8 warps = 32 warps per SM
  for (int pair = 0; pair < 2; ++pair) {
    for (int rep = 0; rep < 2; ++rep) {
      if (pair) k<true><<<blocks, 256>>>(o, iters, c);
      else k<false><<<blocks, 256>>>(o, iters, c);
      cudaDeviceSynchronize();
    }
    long long cy[1024];
    cudaMemcpy(cy, c, blocks * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += cy[i];
    mean /= blocks;
    // per SM: 4 CTAs x 256 threads x iters x 8 x 16 FMAs x 2 flop over the CTA's cycles
    const double flop = 4.0 * 256 * iters * 8 * 16 * 2;
    printf("%s: %.1f flop/clk/SM (%s)\n", pair ? "FFMA2" : "FFMA ", flop / mean, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
