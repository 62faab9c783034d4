// FFMA throughput: register-only operands vs. one constant-bank operand (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_reg(float* out, const float* ab, int iters) {
  float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
  float r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fmaf(r[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

struct W { float w[16]; };
__global__ void ffma_const(float* out, W w, int iters) {
  float r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fmaf(w.w[i], r[(i + 1) & 15], r[i]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// x from registers, weight from registers loaded once (like the conv inner loop)
__global__ void ffma_reg3(float* out, const float* ab, int iters) {
  float w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = ab[i];
  float x = threadIdx.x * 0.001f;
  float r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fmaf(w[i & 7], r[(i + 3) & 15], r[i]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 1234.5f) out[threadIdx.x] = s + x;
}

int main() {
  float* out; float* ab;
  cudaMalloc(&out, 4096); cudaMalloc(&ab, 4096); cudaMemset(ab, 0, 4096);
  W w; for (int i = 0; i < 16; ++i) w.w[i] = 0.999f;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms; double fl = 2.0 * 16 * iters * (double)blocks * threads;
    cudaEventRecord(e0); ffma_reg<<<blocks, threads>>>(out, ab, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("reg (a,b uniform regs): %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0); ffma_const<<<blocks, threads>>>(out, w, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("const operand: %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0); ffma_reg3<<<blocks, threads>>>(out, ab, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("3 distinct regs: %.1f TFLOP/s\n", fl / ms / 1e9);
  }
  return 0;
}
