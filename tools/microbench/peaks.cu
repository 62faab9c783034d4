// Microbenchmark: FP32 FFMA, FP64 DFMA, F2F.F64.F32 throughput on the local GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void ffma_kernel(float* out, float a, float b, int iters) {
  float r[N];
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = fmaf(r[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += r[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int N>
__global__ void dfma_kernel(double* out, double a, double b, int iters) {
  double r[N];
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = threadIdx.x * 0.001 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += r[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int N>
__global__ void f2f_kernel(double* out, float a, int iters) {
  double acc[N];
  float x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { acc[i] = 0; x[i] = threadIdx.x * 0.001f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) { acc[i] += (double)x[i]; x[i] = x[i] * a; }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) s += acc[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock(kHz) %d smem/block optin %zu regs/SM %d\n", prop.name,
         prop.multiProcessorCount, clk, prop.sharedMemPerBlockOptin, prop.regsPerMultiprocessor);
  float* fo; double* dout;
  cudaMalloc(&fo, 4096); cudaMalloc(&dout, 8192);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ffma_kernel<16><<<blocks, threads>>>(fo, 0.999f, 0.001f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("FFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0);
    dfma_kernel<16><<<blocks, threads>>>(dout, 0.999, 0.001, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * (iters / 4) * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0);
    f2f_kernel<16><<<blocks, threads>>>(dout, 0.999f, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = 16.0 * (iters / 4) * (double)blocks * threads;
    printf("F2F+DADD: %.2f Gop/s (per SM per clk at max clk: %.1f)\n", ops / ms / 1e6,
           ops / (ms * 1e-3) / prop.multiProcessorCount / (clk * 1e3));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
