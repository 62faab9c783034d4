// K6-final + K7 + K8 on the 5th-generation tensor cores (tcgen05, 3xTF32).
//
// The last layer's convolution of a map is a sum over tap rows dy of banded GEMMs:
//   R[y, (f, xo)] = sum_dy sum_k  A_dy[y, k] * B_dy[k, (f, xo)],
//   A_dy[y, k] = P[y + dy, 8c + k]           (P: the zero-padded map, tile column 8c + k)
//   B_dy[k, (f, xo)] = W'[f, dy, k - xo]      (zero outside 0 <= k - xo < l)
// for the 8 output columns x = 8c + xo of column block c (K = 16 tile columns covers the
// 8 + l - 1 <= 16 inputs for l <= 9). M = 128 map rows = the 128 TMEM lanes, N = 8 filters
// x 8 columns = 64. W' are the zero-mean taps (per-window centering, as conv.cu), so the
// response equals the reference's centered cross-correlation (cascade.py:108-126).
//
// Precision: 3xTF32. Every operand v is split v = hi + lo with hi = rna_tf32(v) and the
// product is hi*hi' + hi*lo' + lo*hi' (the lo*lo' term is below float32 resolution), FP32
// accumulation in TMEM -- float32-level error, as the FFMA kernel, so the sign codes match
// the reference outside the same ~1e-7 relative band.
//
// Data movement (one CTA per SM, warp-specialized, persistent over maps):
//   producer warps : global map -> SMEM "slots" of 8 tile columns x 136 rows, split into
//                    hi / lo, K-major core-matrix layout (rows 16 B apart), ring of NS;
//   MMA warp       : per slot, tcgen05.cp SMEM -> TMEM of the l row-shifted copies A_dy
//                    (the row shift is the descriptor start address + 16 B * dy), ring of
//                    3 slots in TMEM; per column block 6 l MMAs M128 N64 K8 (A from TMEM,
//                    banded B from SMEM) into one of two TMEM accumulators; commits to
//                    mbarriers release SMEM slots and hand accumulators to the epilogue;
//   epilogue warps : tcgen05.ld of the 64 responses of a row (lane = map row), sign bits
//                    -> LSB-first code (encoder.py:50-68) -> atomic add into the map's
//                    per-block shared bins; at the end of the map the counts go straight
//                    into the feature row (encoder.py:71-99 layout) and the bins are cleared.
// Codes and responses never reach HBM; the map is read once.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "convtc.cuh"
#include "tma.cuh"

namespace ddcca {
namespace tc {

constexpr int X = 8;                       // output columns per column block
constexpr int NF = 8;                      // filter slots (count <= 8; missing filters are zero)
constexpr int N = NF * X;                  // MMA N
constexpr int NA = 3;                      // TMEM ring of A slots
constexpr int NS = 8;                      // SMEM ring of staged slots
constexpr int RP = 136;                    // staged rows per slot: 128 lanes + halo (l <= 9)
constexpr int EPI_WARPS = 8;                   // warps 0..7: lane quadrant w % 4, accumulator w / 4
constexpr int MMA_WARP0 = 8, MMA_WARPS = 2;    // alternate column blocks (one accumulator each)
constexpr int PROD_WARP0 = 10, PROD_WARPS = 4; // one per TMEM lane quadrant
constexpr int THREADS = 32 * (EPI_WARPS + MMA_WARPS + PROD_WARPS);
constexpr int CHUNK_BYTES = RP * 16;       // 4 columns x RP rows
constexpr int RAW_BYTES = 2 * CHUNK_BYTES; // one staged slot: 8 columns
constexpr int BMAT_BYTES = N * 8 * 4;      // one banded K = 8 chunk, hi or lo
constexpr int TMEM_COLS = 512;


__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // K-major, no swizzle: start, leading (K) byte offset, stride (8-row group) byte offset,
  // descriptor version 1 (sm_100)
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
// warp-uniform issue: the whole warp executes, one elected lane issues
__device__ __forceinline__ void mma_tf32(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         uint32_t leader) {
  // the whole warp executes (warp-uniform code), the lane elected once per warp issues
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 e, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(leader));
}
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(e));
  return e;
}
__device__ __forceinline__ void cp_tmem(uint32_t t, uint64_t src) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(t),
      "l"(src));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

}  // namespace tc

template <int L>
__global__ void __launch_bounds__(tc::THREADS, 1)
    conv_hist_tc_kernel(TcHistArgs A, const float* __restrict__ taps /* [(dy * L + dx) * NF + f], zero mean */,
                        const __grid_constant__ CUtensorMap tmap) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* bmat = smem;                                       // [L][2 kc][2 hl] banded B
  uint8_t* raw = smem + L * 4 * BMAT_BYTES;                   // [NS] TMA-staged slots (float32)
  unsigned* bins = reinterpret_cast<unsigned*>(raw + NS * RAW_BYTES);  // [nby * nbx][words]
  // landed: TMA bytes in raw slot; rawfree: 4 producer warps done with it; full: A slot
  // written to TMEM; tfree: MMAs done with the TMEM A slot; dfull / dempty: accumulators
  __shared__ uint64_t landed[NS], rawfree[NS], full[NA], tfree[NA], dfull[2], dempty[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbins = 1 << A.nbits, words = (nbins + 1) / 2;
  const int nblk = A.nby * A.nbx;
  const int cols = A.nbx * A.bw, rows = A.nby * A.bh;
  const int C = (cols + X - 1) / X;  // column blocks per map; slots 0..C

  // banded B matrices, hi / lo, K-major core matrices (8 rows of n x 16 B of k); tile
  // column t <-> image column t - 4, so tap dx of output 8 c + xo sits at k = xo + dx + 4 - left
  for (int e = tid; e < L * 4 * N * 8; e += THREADS) {
    const int k = e & 7, n = (e >> 3) % N, hl = (e / (8 * N)) & 1, kc = (e / (16 * N)) & 1, dy = e / (32 * N);
    const int f = n / X, xo = n % X, t = 8 * kc + k - xo - (4 - (L - 1) / 2);
    const float w = (t >= 0 && t < L) ? taps[(dy * L + t) * NF + f] : 0.f;
    const float hi = tf32_rna(w);
    const float v = hl ? (w - hi) : hi;
    *reinterpret_cast<float*>(bmat + ((dy * 2 + kc) * 2 + hl) * BMAT_BYTES + (k >> 2) * 128 + (n >> 3) * 256 +
                              (n & 7) * 16 + (k & 3) * 4) = v;
  }
  for (int w = tid; w < nblk * words; w += THREADS) bins[w] = 0u;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&landed[i], 1);
      mbar_init(&rawfree[i], PROD_WARPS);
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&full[i], PROD_WARPS);
      mbar_init(&tfree[i], 2);  // both column blocks that read the slot
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dempty[i], EPI_WARPS / 2);  // the four epilogue warps of that accumulator
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t dcol0 = NA * L * 16;  // accumulators after the A ring
  const uint32_t per_map = C + 1;
  const int64_t my_maps = A.n_maps > blockIdx.x ? (A.n_maps - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t total = (uint32_t)(my_maps * per_map);  // slots this CTA stages

  if (warp >= PROD_WARP0) {
    // ---------------------------------------------------------------- A producers
    // Slot j = (map, s): tile columns [8 s, 8 s + 8) = image columns 8 s - 4 + [0, 8) (a
    // 4-column left margin keeps the TMA boxes 16 B aligned; B absorbs the shift) x rows
    // -top .. RP - 1 - top, landed by TMA as two 4-column chunks of RP rows x 16 B. Each
    // producer warp owns the TMEM lane quadrant warp % 4: lane y receives, for every tap
    // row dy, tile row y + dy of the slot as hi (the float32 bits: the tensor core reads
    // the top 19, hi = trunc_tf32(v)) and lo = v - hi, via tcgen05.st (register -> TMEM).
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const int y = 32 * q + lane;
    const bool issuer = warp == PROD_WARP0 && lane == 0;
    auto issue = [&](uint32_t j) {
      const int i = j % NS;
      const int64_t m = blockIdx.x + (int64_t)(j / per_map) * gridDim.x;
      const int s = j % per_map;
      uint8_t* sb = raw + i * RAW_BYTES;
      mbar_expect_tx(&landed[i], (unsigned)RAW_BYTES);
      tma_load_3d(reinterpret_cast<float*>(sb), &tmap, 8 * s - 4, -A.top, (int)m, &landed[i]);
      tma_load_3d(reinterpret_cast<float*>(sb + CHUNK_BYTES), &tmap, 8 * s, -A.top, (int)m, &landed[i]);
    };
    if (issuer)
      for (uint32_t j = 0; j < NS && j < total; ++j) issue(j);
    for (uint32_t g = 0; g < total; ++g) {
      const int i = g % NS;
      const uint32_t ia = g % NA;
      mbar_wait(&landed[i], (g / NS) & 1);
      if (g >= NA) mbar_wait(&tfree[ia], ((g / NA) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* sb = raw + i * RAW_BYTES;
      const uint32_t ta = tm + ((uint32_t)(32 * q) << 16) + ia * (L * 16);
#pragma unroll
      for (int dy = 0; dy < L; ++dy) {
        const float4 c0 = *reinterpret_cast<const float4*>(sb + (y + dy) * 16);
        const float4 c1 = *reinterpret_cast<const float4*>(sb + CHUNK_BYTES + (y + dy) * 16);
        const float v[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          hi[k] = __float_as_uint(v[k]);
          lo[k] = __float_as_uint(v[k] - __uint_as_float(hi[k] & 0xffffe000u));
        }
        st8(ta + dy * 16, hi);
        st8(ta + dy * 16 + 8, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&full[ia]);
        mbar_arrive(&rawfree[i]);
      }
      // restage the raw slot once all four producer warps have read it
      if (issuer && g + NS < total) {
        mbar_wait(&rawfree[i], (g / NS) & 1);
        issue(g + NS);
      }
    }
  } else if (warp >= MMA_WARP0) {
    // ---------------------------------------------------------------- MMA issue
    // Two issuing warps take alternate column blocks (block b -> accumulator b & 1), so two
    // instruction streams feed the tensor pipe (one warp alone cannot issue an N = 64 MMA
    // every 32 cycles).
    const uint32_t w = warp - MMA_WARP0;
    const uint32_t leader = elect_one();
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    // B descriptors are a base plus compile-time offsets (start address field = bytes >> 4)
    const uint64_t bd0 = sdesc(smem_u32(bmat), 128, 256);
    auto commit1 = [&](uint64_t* bar) {
      if (leader)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                     : "memory");
      __syncwarp();
    };
    uint32_t b = 0, use = 0;  // global column-block index, uses of this warp's accumulator
    for (uint32_t mi = 0; mi < (uint32_t)my_maps; ++mi) {
      for (int c = 0; c < C; ++c, ++b) {
        if ((b & 1) != w) continue;
        const uint32_t g = mi * per_map + c;  // slots g (kc = 0) and g + 1 (kc = 1)
        mbar_wait(&full[g % NA], (g / NA) & 1);
        mbar_wait(&full[(g + 1) % NA], ((g + 1) / NA) & 1);
        if (use > 0) mbar_wait(&dempty[w], (use - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tm + dcol0 + w * N;
        const uint32_t a0 = tm + (g % NA) * (L * 16), a1 = tm + ((g + 1) % NA) * (L * 16);
#pragma unroll
        for (int dy = 0; dy < L; ++dy)
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) {
            const uint32_t ahi = (kc ? a1 : a0) + dy * 16, alo = ahi + 8;
            const uint64_t bhi = bd0 + (uint64_t)((((dy * 2 + kc) * 2) * BMAT_BYTES) >> 4);
            const uint64_t blo = bhi + (uint64_t)(BMAT_BYTES >> 4);
            mma_tf32(d, alo, bhi, idesc, (dy | kc) != 0, leader);
            mma_tf32(d, ahi, blo, idesc, 1, leader);
            mma_tf32(d, ahi, bhi, idesc, 1, leader);
          }
        commit1(&dfull[w]);
        // each slot is read by two column blocks (the map's first and last slot by one:
        // their reader arrives twice)
        commit1(&tfree[g % NA]);
        if (c == 0) commit1(&tfree[g % NA]);
        commit1(&tfree[(g + 1) % NA]);
        if (c == C - 1) commit1(&tfree[(g + 1) % NA]);
        ++use;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    // Two groups of four warps, one per accumulator (column-block parity): each group
    // reads its accumulator while the other group's block is still being multiplied.
    const int q = warp & 3, grp = warp >> 2;
    const int y = 32 * q + lane;  // map row of this lane (maps of <= 128 rows)
    const bool row_ok = y < rows;
    unsigned* rbins = bins + (row_ok ? (y / A.bh) * A.nbx * words : 0);
    uint32_t use = 0;
    for (int64_t m = blockIdx.x; m < A.n_maps; m += gridDim.x) {
      const uint32_t b0 = (uint32_t)((m - blockIdx.x) / gridDim.x) * C;  // global block index of column 0
      for (int c = 0; c < C; ++c) {
        if (((b0 + c) & 1) != (uint32_t)grp) continue;
        mbar_wait(&dfull[grp], use & 1);
        ++use;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t v0[32], v1[32];
        const uint32_t ta = tm + ((uint32_t)(32 * q) << 16) + dcol0 + grp * N;
        ld32(ta, v0);
        ld32(ta + 32, v1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[grp]);
        if (!row_ok) continue;
        // sign bits -> LSB-first code; column n = f * X + xo: filters 0..3 in v0, 4..7 in v1
        unsigned code[X];
#pragma unroll
        for (int xo = 0; xo < X; ++xo) {
          unsigned cd = 0;
#pragma unroll
          for (int f = 0; f < NF; ++f)
            if (__uint_as_float(f < 4 ? v0[f * X + xo] : v1[(f - 4) * X + xo]) > 0.f) cd |= 1u << f;
          code[xo] = cd;
        }
        const int x0 = X * c;
        const int bx0 = x0 / A.bw, rem0 = x0 - bx0 * A.bw;
        if (x0 + X <= cols && rem0 + X <= A.bw) {
          // all eight pixels inside one histogram block
          unsigned* bb = rbins + bx0 * words;
#pragma unroll
          for (int xo = 0; xo < X; ++xo) atomicAdd(&bb[code[xo] >> 1], 1u << ((code[xo] & 1u) << 4));
        } else {
          int bx = bx0, rem = rem0;
#pragma unroll
          for (int xo = 0; xo < X; ++xo) {
            if (x0 + xo < cols) atomicAdd(&rbins[bx * words + (code[xo] >> 1)], 1u << ((code[xo] & 1u) << 4));
            if (++rem == A.bw) {
              rem = 0;
              ++bx;
            }
          }
        }
      }
      // the map's histograms are complete: counts into the feature row, bins cleared
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
      for (int b = warp; b < nblk; b += EPI_WARPS) {  // all epilogue warps
        unsigned* wb = bins + b * words;
        const int64_t base = (m / A.gpr) * A.row_stride + (m % A.gpr) * A.group_stride + (int64_t)b * nbins;
        if (A.kind == 2) {
          uint16_t* o = static_cast<uint16_t*>(A.counts) + base;
          for (int k = lane; k < nbins; k += 32) o[k] = (uint16_t)((wb[k >> 1] >> ((k & 1) * 16)) & 0xffffu);
        } else if ((nbins & 7) == 0) {
          uint8_t* o = static_cast<uint8_t*>(A.counts) + base;
          for (int b8 = lane * 8; b8 < nbins; b8 += 256) {
            const uint4 wv = *reinterpret_cast<const uint4*>(wb + (b8 >> 1));
            const unsigned ww[4] = {wv.x, wv.y, wv.z, wv.w};
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              unsigned cnt = (ww[k >> 1] >> ((k & 1) * 16)) & 0xffffu;
              cnt = cnt > 255u ? 255u : cnt;
              if (k < 4) lo |= cnt << (8 * k);
              else hi |= cnt << (8 * (k - 4));
            }
            *reinterpret_cast<uint2*>(o + b8) = make_uint2(lo, hi);
          }
        } else {
          uint8_t* o = static_cast<uint8_t*>(A.counts) + base;
          for (int k = lane; k < nbins; k += 32) {
            const unsigned cnt = (wb[k >> 1] >> ((k & 1) * 16)) & 0xffffu;
            o[k] = (uint8_t)(cnt > 255u ? 255u : cnt);
          }
        }
        __syncwarp();
        for (int w = lane; w < words; w += 32) wb[w] = 0u;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == MMA_WARP0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(TMEM_COLS));
}

template <int L>
static int launch_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st) {
  using namespace tc;
  const int nbins = 1 << a.nbits;
  size_t smem = (size_t)L * 4 * BMAT_BYTES + (size_t)NS * RAW_BYTES +
                sizeof(unsigned) * (size_t)a.nby * a.nbx * ((nbins + 1) / 2);
  if (smem > 225 * 1024) return DDCCA_ECONFIG;
  // one CTA per SM: it allocates all 512 TMEM columns (a second resident CTA would spin in
  // tcgen05.alloc until the first exits), so ask for more than half the shared memory
  smem = std::max<size_t>(smem, 116 * 1024);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (!make_map(&tmap, a.in, a.n_maps, a.p, a.q, 4, RP, 1)) return DDCCA_ECONFIG;
  auto kern = conv_hist_tc_kernel<L>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(a.n_maps, sms);
  kern<<<grid, THREADS, smem, st>>>(a, taps_dev, tmap);
  return check_launch("conv_hist_tc_kernel");
}

bool conv_hist_tc_covers(const TcHistArgs& a) {
  if (const char* e = getenv("DDCCA_CONV_TC"))
    if (e[0] == '0') return false;  // A/B switch: FFMA kernel
  // maps of <= 128 rows (one TMEM lane per row), <= 8 filters / 8-bit codes, odd windows up
  // to 7 (the TMEM A ring of 3 x l x 16 columns plus 2 accumulators), TMA-aligned rows
  if (a.p > 128 || a.count > tc::NF || a.nbits > 8 || a.n_maps < 1 || a.n_maps > INT32_MAX) return false;
  if (a.q % 4 != 0 || (reinterpret_cast<uintptr_t>(a.in) & 15)) return false;
  if (a.top != (a.l - 1) / 2 || a.left != (a.l - 1) / 2) return false;
  return a.l == 3 || a.l == 5 || a.l == 7;
}

int conv_hist_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st) {
  if (!conv_hist_tc_covers(a)) return DDCCA_ECONFIG;
  switch (a.l) {
    case 3: return launch_tc<3>(a, taps_dev, st);
    case 5: return launch_tc<5>(a, taps_dev, st);
    case 7: return launch_tc<7>(a, taps_dev, st);
    default: return DDCCA_ECONFIG;
  }
}

}  // namespace ddcca
