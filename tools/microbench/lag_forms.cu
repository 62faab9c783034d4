// Lag-ring variants for the FP64 moment kernel (diagnostic): DFMA rate of
//   A<K>  : dy in [0,7) ring of 7 partner rows x K dx lags (current form, K = 3)
//   C<K>  : dx-major form, dy in [-6,6] ring of 13 partner rows x K dx lags
// with float32 tiles converted by F2F (CVT=0), by integer bit assembly (CVT=1),
// or float64 tiles (CVT=2). Reports useful DFMA TFLOP/s.
#include <cuda_runtime.h>

#include <cstdio>

template <int CVT>
__device__ __forceinline__ double ld(const float* f, const double* d, int i) {
  if (CVT == 2) return d[i];
  const float v = f[i];
  if (CVT == 0) return (double)v;
  // exact float->double through the integer pipe (normal numbers and zero)
  const unsigned b = __float_as_uint(v);
  const unsigned e = (b >> 23) & 0xffu;
  const unsigned hi = (b & 0x80000000u) | (e ? ((e + 896u) << 20) | ((b >> 3) & 0xfffffu) : 0u);
  const unsigned lo = b << 29;
  return __hiloint2double((int)hi, (int)lo);
}

template <int R, int K, int CVT>
__global__ void __launch_bounds__(256) lag(double* out, int iters, int W) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float* sf = reinterpret_cast<float*>(smraw);
  double* sd = reinterpret_cast<double*>(smraw);
  const int n = 64 * W;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (CVT == 2) sd[i] = (i % 7) * 0.25; else sf[i] = (i % 7) * 0.25f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cown = lane + 8, cpart = lane + warp * K;
  double acc[R][K], ring[R][K];
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int k = 0; k < K; ++k) acc[a][k] = 0.0, ring[a][k] = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int base = ((it * R) & 31) * W;
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int snew = (u + R - 1) % R;
#pragma unroll
      for (int k = 0; k < K; ++k) ring[snew][k] = ld<CVT>(sf, sd, base + (u + R - 1) * W + cpart + k);
      const double own = ld<CVT>(sf, sd, base + u * W + cown);
#pragma unroll
      for (int dy = 0; dy < R; ++dy)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[dy][k] = fma(own, ring[(u + dy) % R][k], acc[dy][k]);
    }
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int k = 0; k < K; ++k) s += acc[a][k];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int R, int K, int CVT>
void run(const char* name, int warps, int per_sm, double* out) {
  const int iters = 256, W = 64;
  const size_t smem = (CVT == 2 ? 8 : 4) * 64 * W;
  auto k = lag<R, K, CVT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * warps, smem);
  const int blocks = 148 * per_sm * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, 32 * warps, smem>>>(out, iters, W);
  cudaEventRecord(e0);
  k<<<blocks, 32 * warps, smem>>>(out, iters, W);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * R * R * K * iters * (double)blocks * 32 * warps;
  printf("%-26s warps/CTA %d occ %d CTAs/SM (%2d warps): %6.1f TFLOP/s\n", name, warps, occ, occ * warps,
         fl / ms / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 8192);
  for (int w : {5, 8}) {
    run<7, 3, 0>("A7x3 f32+F2F", w, 2, out);
    run<7, 3, 1>("A7x3 f32+int-cvt", w, 2, out);
    run<7, 3, 2>("A7x3 f64 smem", w, 2, out);
    run<13, 1, 0>("C13x1 f32+F2F", w, 2, out);
    run<13, 1, 1>("C13x1 f32+int-cvt", w, 2, out);
    run<13, 1, 2>("C13x1 f64 smem", w, 2, out);
    run<13, 2, 0>("C13x2 f32+F2F", w, 2, out);
    run<13, 2, 1>("C13x2 f32+int-cvt", w, 2, out);
    run<13, 2, 2>("C13x2 f64 smem", w, 2, out);
    run<7, 4, 0>("A7x4 f32+F2F", w, 2, out);
    run<7, 4, 2>("A7x4 f64 smem", w, 2, out);
  }
  return 0;
}
