// tcgen05 kind::f16 probe for the conv-histogram kernel (sm_100a):
//  (1) correctness of M128 N64 K16 f16 MMAs with A from TMEM (two halves per 32-bit column,
//      even k in the low half) and with A from SMEM (K-major, no swizzle, row-shifted start
//      address), B from SMEM (K-major, 8-row core matrices of 8 halves);
//  (2) issue throughput (one warp, elect.sync) of 21 such MMAs per step, TS and SS, alone and
//      with three warps streaming LDS.128 from shared memory at the same time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f16_probe f16_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
constexpr uint32_t IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
constexpr int RA = 136;                 // A rows staged (128 + shift)
constexpr int A_LBO = RA * 16;          // bytes between the two K chunks of A
constexpr int B_LBO = 64 * 16;          // bytes between the two K chunks of B

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %3, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(acc), "r"(IDESC));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %3, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(acc), "r"(IDESC));
}
__device__ __forceinline__ void commit_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)));
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity));
}

// A: [RA][16] halves (row-major), B: [16][64] halves; out: [2][128][64] floats (TS, SS)
__global__ void __launch_bounds__(128, 1) check(const __half* A, const __half* B, int shift, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;              // [kc][row][8 halves]
  uint8_t* sb = smem + 2 * A_LBO;  // [kc][n][8 halves]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < RA * 16; e += 128) {
    const int r = e / 16, k = e % 16;
    *reinterpret_cast<__half*>(sa + (k / 8) * A_LBO + r * 16 + (k % 8) * 2) = A[e];
  }
  for (int e = tid; e < 16 * 64; e += 128) {
    const int k = e / 64, n = e % 64;
    *reinterpret_cast<__half*>(sb + (k / 8) * B_LBO + n * 16 + (k % 8) * 2) = B[e];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // A rows into TMEM (lane = row m, A row m = staged row m + shift), columns 128..135
  {
    const int m = tid;
    uint32_t w[8];
    for (int j = 0; j < 8; ++j) {
      const __half lo = A[(m + shift) * 16 + 2 * j], hi = A[(m + shift) * 16 + 2 * j + 1];
      w[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tm + ((uint32_t)(32 * warp) << 16) + 128),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint64_t bd = sdesc(smem_u32(sb), B_LBO, 128);
    const uint64_t ad = sdesc(smem_u32(sa) + 16 * shift, A_LBO, 128);
    mma_ts(tm, tm + 128, bd, 0);
    mma_ss(tm + 64, ad, bd, 0);
    commit_wait(&bar, 0);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int s = 0; s < 2; ++s)
    for (int c = 0; c < 64; c += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tm + ((uint32_t)(32 * warp) << 16) + 64 * s + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) out[(s * 128 + tid) * 64 + c + j] = __uint_as_float(v[j]);
    }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// mode 0: TS, 1: SS; hammer: warps 1..3 stream LDS.128 over 64 KB while warp 0 issues.
template <int mode>
__global__ void __launch_bounds__(128, 1) tput(int dmode, int hammer, int R, long long* cyc, float* sink, int blay) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (96 * 1024) / 4; e += blockDim.x) reinterpret_cast<float*>(smem)[e] = 0.25f * (e & 7);
  if (tid == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 8 * A_LBO;
    // blay 0: K chunks 1 KB apart, 8-row groups at 128 B; 1: K chunks adjacent (128 B), groups at 256 B
    const uint64_t bd = blay ? sdesc(b0, 128, 256) : sdesc(b0, B_LBO, 128);
    const long long t0 = clock64();
    constexpr uint32_t ID32 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int dy = 0; dy < 7; ++dy)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          // dmode 0: two accumulators as the kernel (21 chained MMAs per block); 1: four rotating
          const uint32_t d = dmode == 0 ? tm + 64 * (j == 2) : tm + 64 * ((dy * 3 + j) & 3);
          const uint64_t bj = bd + (uint64_t)((((dy * 3 + j) % 8) * 2 * B_LBO) >> 4);
          if constexpr (mode == 0)
            mma_ts(d, tm + 256 + 16 * dy + 8 * (j & 1), bj, 1);
          else if constexpr (mode == 1)
            mma_ss(d, sdesc(a0 + 16 * dy, A_LBO, 128), bj, 1);
          else
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}\n" ::"r"(d),
                "r"(tm + 256 + 16 * dy + 8 * (j & 1)), "l"(bj), "r"(ID32));
        }
    }
    commit_wait(&bar, 0);
    if (lane == 0) {
      cyc[0] = clock64() - t0;
      stop = 1;
    }
  } else if (hammer) {
    float acc = 0.f;
    const float4* p = reinterpret_cast<const float4*>(smem);
    int i = tid;
    while (!stop) {
#pragma unroll 8
      for (int u = 0; u < 64; ++u) {
        const float4 v = p[(i + u * 96) & 4095];
        acc += v.x + v.w;
      }
      i += 7;
    }
    sink[tid] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  // correctness: small integers (exact in f16, exact f32 sums)
  std::vector<__half> A(RA * 16), B(16 * 64);
  std::vector<float> fa(RA * 16), fb(16 * 64);
  srand(3);
  for (int i = 0; i < RA * 16; ++i) fa[i] = (float)(rand() % 15 - 7), A[i] = __float2half(fa[i]);
  for (int i = 0; i < 16 * 64; ++i) fb[i] = (float)(rand() % 11 - 5), B[i] = __float2half(fb[i]);
  __half *dA, *dB;
  float *dout, *sink;
  long long* dc;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dout, 2 * 128 * 64 * 4);
  cudaMalloc(&dc, 8);
  cudaMalloc(&sink, 128 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int csmem = 2 * A_LBO + 2 * B_LBO;
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
  int fails = 0;
  for (int shift : {0, 3, 6}) {
    check<<<1, 128, csmem>>>(dA, dB, shift, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("check shift %d: %s\n", shift, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> out(2 * 128 * 64);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    long bad[2] = {0, 0};
    for (int s = 0; s < 2; ++s)
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double want = 0;
          for (int k = 0; k < 16; ++k) want += (double)fa[(m + shift) * 16 + k] * fb[k * 64 + n];
          const float got = out[(s * 128 + m) * 64 + n];
          if ((double)got != want) {
            if (bad[s] < 4) printf("  %s shift %d m %d n %d got %g want %g\n", s ? "SS" : "TS", shift, m, n, got, want);
            ++bad[s];
          }
        }
    printf("shift %d: TS %ld wrong, SS %ld wrong (of %d)\n", shift, bad[0], bad[1], 128 * 64);
    fails += bad[0] + bad[1] != 0;
  }
  cudaFuncSetAttribute(tput<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(tput<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(tput<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    for (int dmode = 0; dmode < 2; ++dmode)
      for (int hammer = 0; hammer < 2; ++hammer) {
        const int R = 400;
        (mode == 0 ? tput<0> : mode == 1 ? tput<1> : tput<2>)<<<1, 128, 96 * 1024>>>(dmode, hammer, R, dc, sink, 0);
        long long c = 0;
        const cudaError_t e = cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("%s %s%s: %.2f cycles per M128 N64 MMA (%s)\n", mode == 0 ? "TS f16 K16" : mode == 1 ? "SS f16 K16" : "TS tf32 K8",
               dmode ? "4 rotating D" : "2 D (kernel order)", hammer ? " +LDS.128 x3 warps" : "", (double)c / (R * 21),
               cudaGetErrorString(e));
      }
  for (int mode = 0; mode < 3; ++mode) {
    const int R = 400;
    (mode == 0 ? tput<0> : mode == 1 ? tput<1> : tput<2>)<<<1, 128, 96 * 1024>>>(0, 0, R, dc, sink, 1);
    long long c = 0;
    const cudaError_t e = cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%s, B K-chunks adjacent (LBO 128, SBO 256): %.2f cycles per M128 N64 MMA (%s)\n",
           mode == 0 ? "TS f16 K16" : mode == 1 ? "SS f16 K16" : "TS tf32 K8", (double)c / (R * 21), cudaGetErrorString(e));
  }
  printf("f16_probe: %s\n", fails ? "FAIL" : "ok");
  return fails != 0;
}
