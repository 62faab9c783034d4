// Does the FP64 MMA path (mma.sync m8n8k4 f64) add throughput on top of the DFMA pipe on
// sm_100a? Three kernels over all SMs: DFMA only, DMMA only, and half the warps of each CTA
// on each. Prints TFLOP/s (2 flops per FMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_dfma dmma_dfma.cu
#include <cstdio>

constexpr int ITERS = 4096;

__device__ __forceinline__ void dfma_body(double (&a)[8], double x, double y) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = fma(a[i], x, y);
}

__device__ __forceinline__ void dmma_body(double (&d)[4][2], double a, double b) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[i][0]), "+d"(d[i][1])
                 : "d"(a), "d"(b));
}

// mode 0: all warps DFMA; 1: all warps DMMA; 2: even warps DFMA, odd warps DMMA
__global__ void __launch_bounds__(256) mix(int mode, double* out) {
  const int warp = threadIdx.x >> 5;
  const bool use_mma = mode == 1 || (mode == 2 && (warp & 1));
  double acc = 0.0;
  if (use_mma) {
    double d[4][2] = {};
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    for (int it = 0; it < ITERS; ++it) dmma_body(d, a, b);
    for (int i = 0; i < 4; ++i) acc += d[i][0] + d[i][1];
  } else {
    double r[8];
    for (int i = 0; i < 8; ++i) r[i] = threadIdx.x + i;
    const double x = 0.999999, y = 1e-7;
    for (int it = 0; it < ITERS; ++it) dfma_body(r, x, y);
    for (int i = 0; i < 8; ++i) acc += r[i];
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int blocks_per_sm : {2, 4}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int grid = sms * blocks_per_sm;
      mix<<<grid, 256>>>(mode, out);
      cudaEventRecord(s);
      mix<<<grid, 256>>>(mode, out);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms = 0;
      cudaEventElapsedTime(&ms, s, e);
      // flops: DFMA warps: 32 lanes x 8 FMA x ITERS x 2; DMMA warps: 4 mma x 8x8x4 FMA x ITERS x 2
      const double warps = grid * 8.0;
      const double fw = mode == 0 ? warps : mode == 1 ? 0 : warps / 2;
      const double mw = warps - fw;
      const double flops = fw * 32 * 8 * ITERS * 2.0 + mw * 4 * 256 * ITERS * 2.0;
      printf("%d CTAs/SM mode %d (%s): %.3f ms, %.2f TFLOP/s\n", blocks_per_sm, mode,
             mode == 0 ? "dfma" : mode == 1 ? "dmma" : "half/half", ms, flops / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
