// tcgen05.st (register -> TMEM) throughput on sm_100a: 4 warps (one per TMEM lane quadrant)
// or 8 warps (two per quadrant) store 32x32b.xN tiles to rotating columns; bytes per SM clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_st_probe tmem_st_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void st(uint32_t t, uint32_t v) {
  if constexpr (X == 4)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(t), "r"(v));
  else if constexpr (X == 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(t), "r"(v));
  else
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(t),
        "r"(v));
}

template <int X>
__global__ void probe(int warps, int R, long long* cyc) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  long long t0 = clock64();
  if (warp < warps) {
    const uint32_t q = warp & 3, h = warp >> 2;
    const uint32_t base = tm + ((32 * q) << 16) + h * 256;
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < 16; ++j) st<X>(base + ((j * X) & 255), (uint32_t)(r + j));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) cyc[0] = clock64() - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* dc;
  cudaMalloc(&dc, 8);
  const int R = 200;
  for (int warps : {4, 8})
    for (int x : {4, 8, 16}) {
      if (x == 4) probe<4><<<1, 256>>>(warps, R, dc);
      if (x == 8) probe<8><<<1, 256>>>(warps, R, dc);
      if (x == 16) probe<16><<<1, 256>>>(warps, R, dc);
      long long c = 0;
      const cudaError_t e = cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * R * 16 * 32 * x * 4;
      printf("%d warps, 32x32b.x%-2d: %.1f B/clk (%.1f cycles per warp-instruction) (%s)\n", warps, x, bytes / c,
             (double)c / (R * 16) , cudaGetErrorString(e));
    }
  return 0;
}
