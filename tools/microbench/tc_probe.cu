// Probe of the tcgen05 building blocks for a tensor-core conv-histogram (sm_100a):
//   * tcgen05.cp 128x256b SMEM -> TMEM from a K-major no-swizzle descriptor whose start
//     address is shifted by whole 16-byte rows (a row shift of the image = a tap row dy);
//   * tcgen05.mma kind::tf32, A from TMEM at an arbitrary column offset (an x shift),
//     B (banded tap matrix, N = 8 filters x 2 output columns, K = 8) from SMEM;
//   * tcgen05.commit -> mbarrier, tcgen05.ld 32x32b.x16 of the accumulators.
// Exact small-integer data, so every output must match the host convolution bit for bit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int ROWS = 134;   // 128 output rows + 6 halo rows
constexpr int COLS = 40;    // tile columns (10 chunks of 4)
constexpr int CHUNKS = COLS / 4;
constexpr int NX = 8;       // x0 values probed
__constant__ int c_x0[NX];
__constant__ int c_dyshift;  // 1: A_dy = rows shifted by dy (16 B steps); 0: no shift

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
  return d;                // base offset 0, no swizzle
}

__global__ void __launch_bounds__(128, 1) probe(const float* tile, const float* w /*[8][7][7]*/, float* out,
                                                 uint32_t* diag) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* A = reinterpret_cast<float*>(smem);                 // [CHUNKS][ROWS][4]
  float* B = reinterpret_cast<float*>(smem + CHUNKS * ROWS * 16);  // [7][512 B]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int e = tid; e < ROWS * COLS; e += blockDim.x) {
    const int r = e / COLS, c = e % COLS;
    A[((c >> 2) * ROWS + r) * 4 + (c & 3)] = tile[e];
  }
  // B_dy[n][k], n = f * 2 + xo, value w[f][dy][k - xo]; K-major core matrices 8 n x 4 k:
  // addr = (k / 4) * 128 + (n / 8) * 256 + (n % 8) * 16 + (k % 4) * 4
  for (int e = tid; e < 7 * 16 * 8; e += blockDim.x) {
    const int dy = e / 128, n = (e / 8) % 16, k = e % 8;
    const int f = n >> 1, xo = n & 1, dx = k - xo;
    const float v = (dx >= 0 && dx < 7) ? w[(f * 7 + dy) * 7 + dx] : 0.f;
    B[dy * 128 + ((k >> 2) * 128 + (n >> 3) * 256 + (n & 7) * 16 + (k & 3) * 4) / 4] = v;
  }
  if (tid == 0) {
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
  if (tid == 0) {
    diag[0] = tm;
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    // A_dy[y][k] = tile[y + dy][k]: 5 copies of 8 columns per dy into TMEM columns dy * 40 + 8 j
    for (int dy = 0; dy < 7; ++dy)
      for (int j = 0; j < CHUNKS / 2; ++j) {
        const uint64_t src = sdesc(a0 + (2 * j) * ROWS * 16 + 16 * dy * c_dyshift, ROWS * 16, 128);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + dy * 40 + 8 * j), "l"(src));
      }
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    for (int i = 0; i < NX; ++i) {
      const int x0 = c_x0[i];
      for (int dy = 0; dy < 7; ++dy) {
        const uint64_t bd = sdesc(b0 + dy * 512, 128, 256);
        const uint32_t acc = dy > 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm + 384 + 16 * i),
            "r"(tm + dy * 40 + x0), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int i = 0; i < NX; ++i) {
    uint32_t v[16];
    const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + 384 + 16 * i;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int y = 32 * warp + lane;
    for (int n = 0; n < 16; ++n) out[(i * 128 + y) * 16 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// Throughput probe: one CTA, one issuing thread. mode 0: R x (7 dy x 6 MMAs, N = n, K = 8),
// mode 1: R x (7 dy x 6 cps 128x256b), mode 2: both interleaved per dy. clock64 from the
// first issue to the mbarrier completion of the last op.
__global__ void __launch_bounds__(128, 1) tput(int mode, int R, int n, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (64 * 1024) / 4; e += blockDim.x) reinterpret_cast<float*>(smem)[e] = 0.25f * (e & 7);
  if (tid == 0) {
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
  if (tid == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 48 * 1024;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (((uint32_t)n >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bd = sdesc(b0, 128, 256);
    const long long t0 = clock64();
    for (int r = 0; r < R; ++r)
      for (int dy = 0; dy < 7; ++dy) {
        if (mode == 1 || mode == 2)
          for (int j = 0; j < 6; ++j) {
            const uint64_t src = sdesc(a0 + (j & 1) * 134 * 16 + 16 * dy, 134 * 16 * 2, 128);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 256 + 8 * j + 64 * (dy & 1)),
                         "l"(src));
          }
        if (mode == 0 || mode == 2)
          for (int j = 0; j < 6; ++j) {
            const uint32_t acc = (r | dy | j) != 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm + 64 * (j % 3)),
                "r"(tm + 256 + 8 * j + 64 * ((dy + 1) & 1)), "l"(bd), "r"(idesc), "r"(acc));
          }
        if (mode == 3)  // TS, one accumulator per MMA slot (no D reuse within the step)
          for (int j = 0; j < 6; ++j) {
            const uint32_t acc = r != 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm + (n <= 32 ? 32 : n) * ((dy * 6 + j) % (n <= 32 ? 8 : 4))),
                "r"(tm + 256 + 8 * j), "l"(bd), "r"(idesc), "r"(acc));
          }
        if (mode == 4)  // SS: A from SMEM (K-major, 8-row core matrices at 16 B)
          for (int j = 0; j < 6; ++j) {
            const uint32_t acc = (r | dy | j) != 0;
            const uint64_t ad = sdesc(a0 + (j & 1) * 134 * 16 + 16 * dy, 134 * 16 * 2, 128);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + 64 * (j % 3)),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
          }
        if (mode == 5)  // TS f16 (K = 16 per MMA)
          for (int j = 0; j < 6; ++j) {
            const uint32_t acc = (r | dy | j) != 0;
            const uint32_t id16 = (1u << 4) | (0u << 7) | (0u << 10) | (((uint32_t)n >> 3) << 17) | ((128u >> 4) << 24);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm + 64 * (j % 3)),
                "r"(tm + 256 + 8 * j + 64 * ((dy + 1) & 1)), "l"(bd), "r"(id16), "r"(acc));
          }
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&bar)));
    cyc[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}


// Warp-uniform issue: all of warp 0 runs the loop, elect.sync inside the asm picks the
// issuing lane (no divergent region around the tcgen05 instructions). mode 0: MMAs only
// (6 per step, 3 accumulators), mode 1: cps only, mode 2: both.
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void cp_128x256(uint32_t t, uint64_t src) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(t), "l"(src));
}
__global__ void __launch_bounds__(128, 1) tput2(int mode, int R, int n, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (64 * 1024) / 4; e += blockDim.x) reinterpret_cast<float*>(smem)[e] = 0.25f * (e & 7);
  if (tid == 0) {
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
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 48 * 1024;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (((uint32_t)n >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bd = sdesc(b0, 128, 256);
    const long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int dy = 0; dy < 7; ++dy) {
        if (mode != 0) {
#pragma unroll
          for (int j = 0; j < 6; ++j)
            cp_128x256(tm + 256 + 8 * j + 64 * (dy & 1), sdesc(a0 + (j & 1) * 134 * 16 + 16 * dy, 134 * 16 * 2, 128));
        }
        if (mode != 1) {
#pragma unroll
          for (int j = 0; j < 6; ++j) mma_ts(tm + 64 * (j % 3), tm + 256 + 8 * j + 64 * ((dy + 1) & 1), bd, idesc, 1);
        }
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&bar)));
    if (tid == 0) cyc[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 't') {
    long long* dc;
    cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int n : {16, 32, 64, 128})
      for (int mode = 0; mode < 6; ++mode) {
        const int R = 200;
        tput<<<1, 128, 64 * 1024>>>(mode, R, n, dc);
        long long c = 0;
        const cudaError_t e = cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d %-6s: %8.2f cycles per step of 6 ops (%s)\n", n,
               mode == 0 ? "mma" : mode == 1 ? "cp" : mode == 2 ? "cp+mma" : mode == 3 ? "mma-nodep" : mode == 4 ? "mma-SS" : "mma-f16", (double)c / (R * 7), cudaGetErrorString(e));
      }
    cudaFuncSetAttribute(tput2, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int n : {16, 64, 128, 256})
      for (int mode = 0; mode < 3; ++mode) {
        const int R = 200;
        tput2<<<1, 128, 64 * 1024>>>(mode, R, n, dc);
        long long c = 0;
        const cudaError_t e = cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("uniform N=%3d %-6s: %8.2f cycles per step of 6 ops (%s)\n", n,
               mode == 0 ? "mma" : mode == 1 ? "cp" : "cp+mma", (double)c / (R * 7), cudaGetErrorString(e));
      }
    return 0;
  }
  const int set = argc > 1 ? atoi(argv[1]) : 0, dyshift = argc > 2 ? atoi(argv[2]) : 1;
  const int sets[3][NX] = {{0, 1, 2, 3, 5, 8, 13, 32}, {0, 8, 16, 24, 32, 0, 8, 16}, {0, 2, 4, 6, 10, 12, 20, 30}};
  cudaMemcpyToSymbol(c_x0, sets[set], sizeof(int) * NX);
  cudaMemcpyToSymbol(c_dyshift, &dyshift, sizeof(int));
  printf("x0 set %d, dy shift %d\n", set, dyshift);
  std::vector<float> tile(ROWS * COLS), w(8 * 49), out(NX * 128 * 16, -1.f);
  srand(1);
  for (auto& v : tile) v = (float)(rand() % 9 - 4) * 0.25f;
  for (auto& v : w) v = (float)(rand() % 7 - 3) * 0.5f;
  float *dt, *dw, *dout;
  uint32_t* dd;
  cudaMalloc(&dt, tile.size() * 4);
  cudaMalloc(&dw, w.size() * 4);
  cudaMalloc(&dout, out.size() * 4);
  cudaMalloc(&dd, 64);
  cudaMemcpy(dt, tile.data(), tile.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  const int smem = CHUNKS * ROWS * 16 + 7 * 512;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dt, dw, dout, dd);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  const int* x0s = sets[set];
  long bad = 0, tot = 0;
  for (int i = 0; i < NX; ++i)
    for (int y = 0; y < 128; ++y)
      for (int f = 0; f < 8; ++f)
        for (int xo = 0; xo < 2; ++xo) {
          double s = 0;
          for (int dy = 0; dy < 7; ++dy)
            for (int dx = 0; dx < 7; ++dx) s += (double)tile[(y + dy * dyshift) * COLS + x0s[i] + xo + dx] * w[(f * 7 + dy) * 7 + dx];
          const float g = out[(i * 128 + y) * 16 + f * 2 + xo];
          ++tot;
          if ((double)g != s) {
            if (bad < 10) printf("x0=%d y=%d f=%d xo=%d got %g want %g\n", x0s[i], y, f, xo, g, s);
            ++bad;
          }
        }
  printf("tc_probe: %ld / %ld outputs wrong\n", bad, tot);
  return bad != 0;
}
