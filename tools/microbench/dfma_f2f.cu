// DFMA ring pattern with float->double conversions of the loaded operands (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>

template <bool CONV>
__global__ void ring(double* out, const float* srcf, const double* srcd, int iters) {
  __shared__ float sf[1024];
  __shared__ double sd[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sf[i] = srcf[i]; sd[i] = srcd[i]; }
  __syncthreads();
  double acc[7][3];
#pragma unroll
  for (int a = 0; a < 7; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) acc[a][k] = 0;
  double ring[7][3];
#pragma unroll
  for (int a = 0; a < 7; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) ring[a][k] = 0;
  int base = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      const int idx = (base + it * 7 + u * 33) & 1023;
#pragma unroll
      for (int k = 0; k < 3; ++k) ring[(u + 6) % 7][k] = CONV ? (double)sf[(idx + k) & 1023] : sd[(idx + k) & 1023];
      double own = CONV ? (double)sf[(idx + 40) & 1023] : sd[(idx + 40) & 1023];
#pragma unroll
      for (int dy = 0; dy < 7; ++dy)
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[dy][k] = fma(own, ring[(u + dy) % 7][k], acc[dy][k]);
    }
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < 7; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) s += acc[a][k];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  double *out, *sd; float* sf;
  cudaMalloc(&out, 8192); cudaMalloc(&sd, 8192); cudaMalloc(&sf, 4096);
  cudaMemset(sd, 0, 8192); cudaMemset(sf, 0, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 160, iters = 512;
  for (int per = 2; per <= 4; ++per) {
    int blocks = 148 * per;
    float ms;
    double fl = 2.0 * 147 * iters * (double)blocks * threads;
    for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0); ring<false><<<blocks, threads>>>(out, sf, sd, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("blocks/SM %d fp64 smem: %.1f TFLOP/s\n", per, fl / ms / 1e9);
    cudaEventRecord(e0); ring<true><<<blocks, threads>>>(out, sf, sd, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("blocks/SM %d fp32 smem + F2F: %.1f TFLOP/s\n", per, fl / ms / 1e9);
    }
  }
  return 0;
}
