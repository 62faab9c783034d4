// DFMA throughput by operand pattern (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>

// acc[i] += x * y[i]: x reused, y[i] distinct registers, acc distinct (the lag ring pattern)
__global__ void dfma_ring(double* out, const double* src, int iters) {
  double y[21], acc[21];
#pragma unroll
  for (int i = 0; i < 21; ++i) { y[i] = src[i] + threadIdx.x; acc[i] = 0; }
  double x = src[30] + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 21; ++i) acc[i] = fma(x, y[i], acc[i]);
    x += 1e-9;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 21; ++i) s += acc[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// acc[i] += a * b with a, b uniform (the peak pattern)
__global__ void dfma_uniform(double* out, double a, double b, int iters) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// acc[i] += x[i] * y[i]: nothing reused
__global__ void dfma_none(double* out, const double* src, int iters) {
  double y[12], x[12], acc[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) { y[i] = src[i] + threadIdx.x; x[i] = src[i + 12]; acc[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = fma(x[i], y[(i + it) % 12 == 0 ? i : i], acc[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 12; ++i) s += acc[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  double *out, *src;
  cudaMalloc(&out, 8192); cudaMalloc(&src, 8192); cudaMemset(src, 0, 8192);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 128, iters = 2048;
  for (int per = 1; per <= 8; per *= 2) {
    int blocks = 148 * per;
    printf("warps/SM = %d\n", per * 4);
    float ms;
    cudaEventRecord(e0); dfma_ring<<<blocks, threads>>>(out, src, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("ring pattern: %.1f TFLOP/s\n", 2.0 * 21 * iters * (double)blocks * threads / ms / 1e9);
    cudaEventRecord(e0); dfma_uniform<<<blocks, threads>>>(out, 0.999, 0.001, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("uniform a,b: %.1f TFLOP/s\n", 2.0 * 16 * iters * (double)blocks * threads / ms / 1e9);
    cudaEventRecord(e0); dfma_none<<<blocks, threads>>>(out, src, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("no reuse: %.1f TFLOP/s\n", 2.0 * 12 * iters * (double)blocks * threads / ms / 1e9);
  }
  return 0;
}
