// K6-final + K7 + K8 on the 5th-generation tensor cores (tcgen05, kind::f16, two-term split).
//
// The last layer's convolution of a map is a sum over tap rows dy of banded GEMMs:
//   R[y, (f, xo)] = sum_dy sum_k  A_dy[y, k] * B_dy[k, (f, xo)],
//   A_dy[y, k] = P[y + dy, 8c - 4 + k]        (P: the zero-padded map, K = 16 columns)
//   B_dy[k, (f, xo)] = W'[f, dy, k - xo - 4 + left]   (zero outside the window)
// for the 8 output columns x = 8c + xo of column block c (K = 16 covers the 8 + l - 1 inputs
// for l <= 9). M = 128 map rows = the 128 TMEM lanes, N = 8 filters x 8 columns = 64, one
// M128 N64 K16 MMA per tap row and product term. W' are the zero-mean taps (per-window
// centering, as conv.cu), so the response equals the reference's centered cross-correlation
// (cascade.py:108-126).
//
// Precision: every operand is scaled by a power of two (A: per map, from the map's largest
// magnitude; B: per filter) into [2^14, 2^15) and split v = hi + lo with hi = rn_f16(v), lo =
// rn_f16(v - hi) (22 significant bits); the product is hi*hi' + hi*lo' + lo*hi' (lo*lo' is below
// float32 resolution), FP32 accumulation in TMEM -- the same ~2^-22 relative error as a 3xTF32
// split at half the tensor-pipe cycles (a K16 f16 MMA takes the cycles of a K8 tf32 one:
// tools/microbench/f16_probe.cu). Only the response's sign is used (K7), and positive scale
// factors do not change it: no rescaling in the epilogue.
//
// Data movement (one CTA per SM, warp-specialized, persistent over maps):
//   loader warps   : TMA of the whole zero-padded map (RP rows x (2C+2) 4-column chunks, rows
//                    16 B apart) into one of two SMEM map buffers; the map's largest magnitude
//                    (-> its power-of-two scale); the map split in place into f16 hi / lo pairs;
//                    one map ahead of the producers;
//   producer warps : two per TMEM lane quadrant (tap rows split in halves); per 8-column slot,
//                    lane y loads split tile rows y + dy and, with the previous slot's words kept
//                    in registers, writes block c's A_dy (8 hi + 8 lo TMEM columns: K = 16 f16)
//                    by tcgen05.st into a TMEM ring of 3 blocks;
//   MMA warps      : per column block 3 l MMAs M128 N64 K16 (A from TMEM, banded B from SMEM)
//                    into one of two TMEM accumulators; two warps take alternate blocks;
//                    commits to mbarriers release the A block and hand the accumulator over;
//   epilogue warps : tcgen05.ld of the 64 responses of a row (lane = map row), sign bits
//                    -> LSB-first code (encoder.py:50-68) -> atomic add into the map's
//                    per-block shared bins; at the end of the map the bins are copied (u8
//                    saturated or u16) straight into the feature row (encoder.py:71-99 layout)
//                    and cleared.
// tools/microbench/tc_trace.cu records the hand-off timeline (DDCCA_TC_TRACE).
// Codes and responses never reach HBM; the map is read once.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "convtc.cuh"
#include "tma.cuh"

namespace ddcca {
namespace tc {

constexpr int X = 8;                       // output columns per column block
constexpr int NF = 8;                      // filter slots (count <= 8; missing filters are zero)
constexpr int N = NF * X;                  // MMA N
constexpr int NA = 3;                      // TMEM ring of A blocks
constexpr int RP = 136;                    // staged rows: 128 lanes + halo (l <= 9)
constexpr int EPI_WARPS = 8;                   // warps 0..7: lane quadrant w % 4, accumulator w / 4
constexpr int MMA_WARP0 = 8, MMA_WARPS = 2;    // alternate column blocks (one accumulator each)
constexpr int PROD_WARP0 = 10, PROD_WARPS = 8; // two per TMEM lane quadrant (tap rows split in halves)
constexpr int LOAD_WARP0 = PROD_WARP0 + PROD_WARPS, LOAD_WARPS = 2;  // map TMA, scale, f16 split
constexpr int THREADS = 32 * (EPI_WARPS + MMA_WARPS + PROD_WARPS + LOAD_WARPS);
constexpr int CHUNK_BYTES = RP * 16;       // 4 columns x RP rows (one TMA box)
constexpr int BMAT_BYTES = N * 16 * 2;     // one tap row's banded B, hi or lo: N x K16 halves
constexpr int A_COLS = 16;                 // TMEM columns per tap row and block: 8 hi + 8 lo
constexpr int TMEM_COLS = 512;
constexpr int SCALE_EXP = 15;              // operands scaled into [2^14, 2^15)

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // K-major, no swizzle: start, leading (K) byte offset, stride (8-row group) byte offset,
  // descriptor version 1 (sm_100)
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// warp-uniform issue: the whole warp executes, the lane elected once per warp issues
__device__ __forceinline__ void mma_f16(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                        uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 e, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(leader));
}
// 2^(SCALE_EXP - e) for a largest magnitude mx = f 2^e (f in [0.5, 1)); 1 for 0 / non-finite
__device__ __forceinline__ float pow2_scale(float mx) {
  if (!(mx > 0.f) || !isfinite(mx)) return 1.f;
  int e;
  frexpf(mx, &e);
  return ldexpf(1.f, max(-126, min(127, SCALE_EXP - e)));
}
// Two map values (scaled by sc) -> f16 pairs: hi = the scaled value truncated to 11 significant
// bits (exact in f16 over its normal range), lo = rn_f16(value - hi) (the residual is exact in
// float32); element 2 j in the low half of word j
__device__ __forceinline__ void split2(float a, float b, float2 sc, float2 off, uint32_t& hi, uint32_t& lo) {
  const float2 v = __ffma2_rn(make_float2(a, b), sc, off);  // (value - shift) * scale, one rounding
  const float2 h = make_float2(__uint_as_float(__float_as_uint(v.x) & 0xffffe000u),
                               __uint_as_float(__float_as_uint(v.y) & 0xffffe000u));
  const float2 r = __fadd2_rn(v, make_float2(-h.x, -h.y));
  const __half2 hh = __floats2half2_rn(h.x, h.y);
  const __half2 ll = __floats2half2_rn(r.x, r.y);
  hi = *reinterpret_cast<const uint32_t*>(&hh);
  lo = *reinterpret_cast<const uint32_t*>(&ll);
}
// mbarrier wait: try_wait without a suspend-time hint (the instruction itself blocks for a
// hardware time window; with a hint the wait compiles to a NANOSLEEP.SYNCS loop that wakes on
// every barrier event of the CTA and spends issue slots)
__device__ __forceinline__ void mbar_wait_hw(uint64_t* b, unsigned parity) {
  for (;;) {
    unsigned done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
  }
}
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(e));
  return e;
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

__device__ __forceinline__ void st4(uint32_t taddr, const uint32_t (&v)[4]) {
  // no "memory" clobber: TMEM is not compiler-visible memory (tcgen05.wait::st and the fences,
  // which do clobber memory, order the stores against the barrier arrive)
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]));
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}

// Pipeline trace for tools/microbench/tc_trace.cu (compiled in only with DDCCA_TC_TRACE): CTA 0,
// first 256 column blocks, clock64 per hand-off event kind.
#ifdef DDCCA_TC_TRACE
__device__ long long g_tc_trace[12][256];
#define TC_TRACE(kind, idx)                                                     \
  do {                                                                          \
    if (blockIdx.x == 0 && (idx) < 256 && lane == 0) g_tc_trace[(kind)][(idx)] = clock64(); \
  } while (0)
#else
#define TC_TRACE(kind, idx) \
  do {                      \
  } while (0)
#endif

}  // namespace tc

// RESP: write the float32 responses (unscaled) instead of hashing them into block histograms
template <int L, bool RESP>
__global__ void __launch_bounds__(tc::THREADS, 1)
    conv_hist_tc_kernel(TcHistArgs A, const float* __restrict__ taps /* [(dy * L + dx) * NF + f], zero mean */,
                        int nbuf /* staged map buffers: 2, or 1 when shared memory is short */,
                        const __grid_constant__ CUtensorMap tmap) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int nbins = 1 << A.nbits, words = (nbins + 1) / 2;
  const int nblk = A.nby * A.nbx;
  const int cols = RESP ? A.q : A.nbx * A.bw, rows = RESP ? A.p : A.nby * A.bh;
  const int C = (cols + X - 1) / X;  // column blocks per map
  const int nch = 2 * C + 2;         // 4-column chunks staged per map (image columns -4 .. 8C + 3)
  uint8_t* bmat = smem;                                          // [L][hi, lo] banded B
  uint8_t* mbuf = smem + L * 2 * BMAT_BYTES;                     // [nbuf] staged maps [nch][RP][16 B]
  unsigned* bins = reinterpret_cast<unsigned*>(mbuf + nbuf * nch * CHUNK_BYTES);  // [nby * nbx][words]
  // landed: map bytes arrived; ready: the map is split; mapfree: the producers are
  // done with the buffer; full: A block written to TMEM; tfree: MMAs done with the TMEM A
  // block; dfull / dempty: accumulators
  __shared__ uint64_t landed[2], ready[2], mapfree[2], full[NA], tfree[NA], dfull[2], dempty[2];
  __shared__ uint32_t tbase;
  __shared__ float fscale[NF], lmax[2][LOAD_WARPS], lsum[2][LOAD_WARPS], mscale[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // per-filter power-of-two scales, then the banded B matrices (hi / lo), K-major core
  // matrices: element (n, k) at (n / 8) * 256 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2
  if (tid < NF) {
    float mx = 0.f;
    for (int t = 0; t < L * L; ++t) mx = fmaxf(mx, fabsf(taps[t * NF + tid]));
    fscale[tid] = pow2_scale(mx);
  }
  __syncthreads();
  for (int e = tid; e < L * 2 * N * 16; e += THREADS) {
    const int k = e & 15, n = (e >> 4) % N, hl = (e / (16 * N)) & 1, dy = e / (32 * N);
    const int f = n / X, xo = n % X, t = k - xo - (4 - (L - 1) / 2);
    const float w = (t >= 0 && t < L) ? taps[(dy * L + t) * NF + f] * fscale[f] : 0.f;
    const __half h = __float2half_rn(w);
    const __half v = hl ? __float2half_rn(w - __half2float(h)) : h;
    *reinterpret_cast<__half*>(bmat + (dy * 2 + hl) * BMAT_BYTES + (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 +
                               (k & 7) * 2) = v;
  }
  if constexpr (!RESP)
    for (int w = tid; w < nblk * words; w += THREADS) bins[w] = 0u;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&landed[i], 1);
      mbar_init(&ready[i], 1);
      mbar_init(&mapfree[i], PROD_WARPS);
      mbar_init(&dfull[i], 1);
      mbar_init(&dempty[i], EPI_WARPS / 2);  // the four epilogue warps of that accumulator
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&full[i], PROD_WARPS);
      mbar_init(&tfree[i], 1);
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
  const uint32_t dcol0 = NA * L * A_COLS;  // accumulators after the A ring
  const int64_t my_maps = A.n_maps > blockIdx.x ? (A.n_maps - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t total_blocks = (uint32_t)(my_maps * C);

  if (warp >= LOAD_WARP0) {
    // ---------------------------------------------------------------- map loads + split
    // Map i of this CTA lands in buffer i % nbuf as nch TMA boxes (chunk j = image columns
    // 4 j - 4 .. 4 j - 1, rows -top .. RP - 1 - top, zero outside the map). The two loader
    // warps reduce the map's largest magnitude to its power-of-two scale and split the map in
    // place: every 16-byte chunk row (4 floats) becomes {hi(e0, e1), hi(e2, e3), lo(e0, e1),
    // lo(e2, e3)} as f16 pairs; then the buffer is handed to the producers. They run a map
    // ahead of the producers (nbuf = 2).
    const uint32_t map_bytes = (uint32_t)nch * CHUNK_BYTES;
    const int lt = tid - 32 * LOAD_WARP0;  // 0 .. 63
    const int n16 = nch * RP;
    for (int64_t i = 0; i < my_maps; ++i) {
      const int bsel = (int)(i % nbuf);
      const uint32_t use_par = (uint32_t)((i / nbuf) & 1);
      if (i >= nbuf) mbar_wait_hw(&mapfree[bsel], use_par ^ 1u);
      uint8_t* dst = mbuf + bsel * nch * CHUNK_BYTES;
      if (lt == 0) {
        const int64_t m = blockIdx.x + i * gridDim.x;
        mbar_expect_tx(&landed[bsel], map_bytes);
        for (int j = 0; j < nch; ++j)
          tma_load_3d(reinterpret_cast<float*>(dst + j * CHUNK_BYTES), &tmap, 4 * j - 4, -A.top, (int)m, &landed[bsel]);
      }
      mbar_wait_hw(&landed[bsel], use_par);
      // largest magnitude (and, with a DC shift, the sum): eight loads in flight per thread
      float mx = 0.f, sm = 0.f;
      int e = lt;
      for (; e + 7 * 64 < n16; e += 8 * 64) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const float4*>(dst + (e + 64 * u) * 16);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
          if (RESP) sm += (v[u].x + v[u].y) + (v[u].z + v[u].w);
        }
      }
      for (; e < n16; e += 64) {
        const float4 v = *reinterpret_cast<const float4*>(dst + e * 16);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        if (RESP) sm += (v.x + v.y) + (v.z + v.w);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (RESP) sm += __shfl_xor_sync(0xffffffffu, sm, o);
      }
      if (lane == 0) {
        lmax[i & 1][warp - LOAD_WARP0] = mx;
        lsum[i & 1][warp - LOAD_WARP0] = sm;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * LOAD_WARPS) : "memory");
      // DC shift (responses of centered windows: zero-mean taps make the result independent of
      // a constant shift of the whole padded map, padding included): the map mean; the
      // scale then bounds |v - shift| <= max |v| + |shift|
      const float shift = (RESP && A.dc_shift) ? (lsum[i & 1][0] + lsum[i & 1][1]) / (float)(A.p * A.q) : 0.f;
      const float sc = pow2_scale(fmaxf(lmax[i & 1][0], lmax[i & 1][1]) + fabsf(shift));
      const float2 sc2 = make_float2(sc, sc), off2 = make_float2(-shift * sc, -shift * sc);
      if (RESP && lt == 0) mscale[i & 7] = sc;  // read by the epilogue (at most ~5 blocks behind)
      e = lt;
      for (; e + 3 * 64 < n16; e += 4 * 64) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(dst + (e + 64 * u) * 16);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 o;
          split2(v[u].x, v[u].y, sc2, off2, o.x, o.z);
          split2(v[u].z, v[u].w, sc2, off2, o.y, o.w);
          *reinterpret_cast<uint4*>(dst + (e + 64 * u) * 16) = o;
        }
      }
      for (; e < n16; e += 64) {
        const float4 v = *reinterpret_cast<const float4*>(dst + e * 16);
        uint4 o;
        split2(v.x, v.y, sc2, off2, o.x, o.z);
        split2(v.z, v.w, sc2, off2, o.y, o.w);
        *reinterpret_cast<uint4*>(dst + e * 16) = o;
      }
      // generic-proxy writes that the next TMA into this buffer overwrites
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 3, %0;" ::"n"(32 * LOAD_WARPS) : "memory");
      if (lt == 0) mbar_arrive(&ready[bsel]);
    }
  } else if (warp >= PROD_WARP0) {
    // ---------------------------------------------------------------- A producers
    // Block c = image columns 8 c - 4 .. 8 c + 11 = split chunks 2 c .. 2 c + 3. Producer warp
    // w owns the TMEM lane quadrant w % 4 and half of the tap rows: lane y copies split tile
    // row y + dy of the four chunks into block c's A_dy (8 hi + 8 lo TMEM columns).
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const int y = 32 * q + lane;
    constexpr int HALF = (L + 1) / 2;
    const int dy0 = (warp - PROD_WARP0) < 4 ? 0 : HALF;  // tap rows dy0 .. dy0 + HALF - 1 (< L)
    uint32_t blk = 0;  // this CTA's global column-block index (A ring position)
    for (int64_t i = 0; i < my_maps; ++i) {
      const int bsel = (int)(i % nbuf);
      const uint32_t use_par = (uint32_t)((i / nbuf) & 1);  // parity of this use of the buffer
      mbar_wait_hw(&ready[bsel], use_par);
      // slot s = split chunks 2 s, 2 s + 1: hi words {c0.x, c0.y, c1.x, c1.y}, lo words {.z, .w};
      // block c = slots c, c + 1. The previous slot's words stay in registers (two sets
      // alternate), so each slot is read from shared memory once per thread.
      const uint8_t* buf = mbuf + bsel * nch * CHUNK_BYTES + (y + dy0) * 16;
      uint4 sa[HALF][2], sb[HALF][2];  // [d][0] = hi words, [d][1] = lo words
      auto load_slot = [&](int sl, uint4 (&dst)[HALF][2]) {
        const uint8_t* cp = buf + (2 * sl) * CHUNK_BYTES;
#pragma unroll
        for (int d = 0; d < HALF; ++d)
          if (dy0 + d < L) {
            const uint4 c0 = *reinterpret_cast<const uint4*>(cp + d * 16);
            const uint4 c1 = *reinterpret_cast<const uint4*>(cp + CHUNK_BYTES + d * 16);
            dst[d][0] = make_uint4(c0.x, c0.y, c1.x, c1.y);
            dst[d][1] = make_uint4(c0.z, c0.w, c1.z, c1.w);
          }
      };
      // block(lf, rt, next): stores block c from slots c (lf) and c + 1 (rt), and loads slot
      // `next` into lf while the stores drain (lf's words are consumed by the stores' issue)
      auto block = [&](uint4 (&lf)[HALF][2], const uint4 (&rt)[HALF][2], int next) {
        const uint32_t ia = blk % NA;
        if (blk >= NA) mbar_wait_hw(&tfree[ia], ((blk / NA) - 1) & 1);
        if (warp == PROD_WARP0) TC_TRACE(5, blk);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tm + ((uint32_t)(32 * q) << 16) + ia * (L * A_COLS);
#pragma unroll
        for (int d = 0; d < HALF; ++d) {
          if (dy0 + d >= L) break;
          const uint32_t col = (dy0 + d) * A_COLS;
          const uint32_t hv[8] = {lf[d][0].x, lf[d][0].y, lf[d][0].z, lf[d][0].w,
                                  rt[d][0].x, rt[d][0].y, rt[d][0].z, rt[d][0].w};
          const uint32_t lv[8] = {lf[d][1].x, lf[d][1].y, lf[d][1].z, lf[d][1].w,
                                  rt[d][1].x, rt[d][1].y, rt[d][1].z, rt[d][1].w};
          st8(ta + col, hv);
          st8(ta + col + 8, lv);
        }
        if (next <= C) load_slot(next, lf);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[ia]);
        if (warp == PROD_WARP0) TC_TRACE(6, blk);
        ++blk;
      };
      load_slot(0, sa);
      load_slot(1, sb);
      for (int c = 0; c < C; c += 2) {
        block(sa, sb, c + 2);      // block c = slots c, c + 1; sa <- slot c + 2
        if (c + 1 < C) block(sb, sa, c + 3);  // block c + 1 = slots c + 1, c + 2; sb <- slot c + 3
      }
      // the map buffer is free once all producer warps are past it
      __syncwarp();
      if (lane == 0) mbar_arrive(&mapfree[bsel]);
    }
  } else if (warp >= MMA_WARP0) {
    // ---------------------------------------------------------------- MMA issue
    // Two issuing warps take alternate column blocks (block b -> accumulator b & 1).
    const uint32_t w = warp - MMA_WARP0;
    const uint32_t leader = elect_one();
    // kind::f16: f32 accumulator (bit 4), f16 A and B (formats 0), K-major, N >> 3, M >> 4
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bd0 = sdesc(smem_u32(bmat), 128, 256);
    auto commit1 = [&](uint64_t* bar) {
      if (leader)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                     : "memory");
      __syncwarp();
    };
    for (uint32_t b = w, use = 0; b < total_blocks; b += 2, ++use) {
      const uint32_t ia = b % NA;
      mbar_wait_hw(&full[ia], (b / NA) & 1);
      TC_TRACE(0, b);
      if (use > 0) mbar_wait_hw(&dempty[w], (use - 1) & 1);
      TC_TRACE(1, b);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tm + dcol0 + w * N;
      const uint32_t a = tm + ia * (L * A_COLS);
#pragma unroll
      for (int dy = 0; dy < L; ++dy) {
        const uint32_t ahi = a + dy * A_COLS, alo = ahi + 8;
        const uint64_t bhi = bd0 + (uint64_t)((dy * 2 * BMAT_BYTES) >> 4);
        const uint64_t blo = bhi + (uint64_t)(BMAT_BYTES >> 4);
        mma_f16(d, alo, bhi, idesc, dy != 0, leader);
        mma_f16(d, ahi, blo, idesc, 1, leader);
        mma_f16(d, ahi, bhi, idesc, 1, leader);
      }
      TC_TRACE(2, b);
      commit1(&dfull[w]);
      commit1(&tfree[ia]);
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
        mbar_wait_hw(&dfull[grp], use & 1);
        if (q == 0) TC_TRACE(3, b0 + c);
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
        if (q == 0) TC_TRACE(4, b0 + c);
        if (!row_ok) continue;
        if constexpr (RESP) {
          // responses: undo the power-of-two scales (exact) and store row y of the 8 columns of
          // each filter (filter-minor output, cascade.py:123-125)
          const float inv_m = 1.f / mscale[(uint32_t)((m - blockIdx.x) / gridDim.x) & 7];
          const int x0 = X * c;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            if (f >= A.count) break;
            const float inv = inv_m / fscale[f];
            float* o = A.resp + ((m * A.count + f) * (int64_t)A.p + y) * A.q + x0;
            float r[X];
#pragma unroll
            for (int xo = 0; xo < X; ++xo) r[xo] = __uint_as_float(f < 4 ? v0[f * X + xo] : v1[(f - 4) * X + xo]) * inv;
            if (x0 + X <= A.q && (A.q & 7) == 0) {
              // one 256-bit store per (row, filter): a full 32-byte sector
              asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o), "f"(r[0]), "f"(r[1]),
                           "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                           : "memory");
            } else if (x0 + X <= A.q) {
              reinterpret_cast<float4*>(o)[0] = make_float4(r[0], r[1], r[2], r[3]);
              reinterpret_cast<float4*>(o)[1] = make_float4(r[4], r[5], r[6], r[7]);
            } else {
#pragma unroll
              for (int xo = 0; xo < X; ++xo)
                if (x0 + xo < A.q) o[xo] = r[xo];
            }
          }
        } else {
        // sign bits -> LSB-first code; column n = f * X + xo: filters 0..3 in v0, 4..7 in v1.
        // Filters (2j, 2j + 1) are packed to bf16x2 (sign and zero preserved, no overflow; only
        // |r| < 1e-38 would flush, far below the float32 noise of responses scaled ~2^28) and
        // compared in one instruction: halves 0xffff where r > 0. The four masks fold into
        // the 8-bit code with immediates.
        unsigned code[X];
#pragma unroll
        for (int xo = 0; xo < X; ++xo) {
          const __nv_bfloat162 zero = __float2bfloat162_rn(0.f);
          const auto pk = [&](uint32_t a, uint32_t b) {
            return __hgt2_mask(__floats2bfloat162_rn(__uint_as_float(a), __uint_as_float(b)), zero);
          };
          const unsigned m0 = pk(v0[0 * X + xo], v0[1 * X + xo]), m1 = pk(v0[2 * X + xo], v0[3 * X + xo]);
          const unsigned m2 = pk(v1[0 * X + xo], v1[1 * X + xo]), m3 = pk(v1[2 * X + xo], v1[3 * X + xo]);
          const unsigned t = (m0 & 0x00020001u) | (m1 & 0x00080004u) | (m2 & 0x00200010u) | (m3 & 0x00800040u);
          code[xo] = (t | (t >> 16)) & 0xffu;
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
        }  // RESP / histogram epilogue
      }
      if constexpr (!RESP) {
        // the map's histograms are complete: counts into the feature row, bins cleared
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (warp == 0) TC_TRACE(7, (int)(2 * ((m - blockIdx.x) / gridDim.x)));
        // The feature row holds the map's blocks' bins contiguously (encoder.py:71-99 layout), so
        // the flush is a linear copy: bins (two 16-bit counts per word) -> u8 (saturated) or u16,
        // 8 bins per thread step, the bins cleared behind it
        {
          const int64_t rowbase = (m / A.gpr) * A.row_stride + (m % A.gpr) * A.group_stride;
          const int et = warp * 32 + lane;  // 0 .. 255
          uint4* bins4 = reinterpret_cast<uint4*>(bins);
          if ((nbins & 7) == 0) {
            const int chunks = nblk * nbins / 8;
            if (A.kind == 2) {
              uint4* o = reinterpret_cast<uint4*>(static_cast<uint16_t*>(A.counts) + rowbase);
              for (int k = et; k < chunks; k += 32 * EPI_WARPS) {
                o[k] = bins4[k];  // little-endian 16-bit halves are the u16 counts in bin order
                bins4[k] = make_uint4(0u, 0u, 0u, 0u);
              }
            } else {
              uint2* o = reinterpret_cast<uint2*>(static_cast<uint8_t*>(A.counts) + rowbase);
              constexpr int U = 4, S = 32 * EPI_WARPS;  // four chunks in flight per thread
              int k = et;
              for (; k + (U - 1) * S < chunks; k += U * S) {
                uint4 w[U];
  #pragma unroll
                for (int u = 0; u < U; ++u) w[u] = bins4[k + u * S];
  #pragma unroll
                for (int u = 0; u < U; ++u) {
                  const unsigned x = __vminu2(w[u].x, 0x00ff00ffu), y = __vminu2(w[u].y, 0x00ff00ffu);
                  const unsigned z = __vminu2(w[u].z, 0x00ff00ffu), v = __vminu2(w[u].w, 0x00ff00ffu);
                  o[k + u * S] = make_uint2(__byte_perm(x, y, 0x6420), __byte_perm(z, v, 0x6420));
                  bins4[k + u * S] = make_uint4(0u, 0u, 0u, 0u);
                }
              }
              for (; k < chunks; k += S) {
                const uint4 w = bins4[k];
                const unsigned x = __vminu2(w.x, 0x00ff00ffu), y = __vminu2(w.y, 0x00ff00ffu);
                const unsigned z = __vminu2(w.z, 0x00ff00ffu), v = __vminu2(w.w, 0x00ff00ffu);
                o[k] = make_uint2(__byte_perm(x, y, 0x6420), __byte_perm(z, v, 0x6420));
                bins4[k] = make_uint4(0u, 0u, 0u, 0u);
              }
            }
          } else {
            for (int k = et; k < nblk * nbins; k += 32 * EPI_WARPS) {
              const unsigned cnt = (bins[k >> 1] >> ((k & 1) * 16)) & 0xffffu;
              if (A.kind == 2)
                static_cast<uint16_t*>(A.counts)[rowbase + k] = (uint16_t)cnt;
              else
                static_cast<uint8_t*>(A.counts)[rowbase + k] = (uint8_t)(cnt > 255u ? 255u : cnt);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
            for (int w = et; w < nblk * words; w += 32 * EPI_WARPS) bins[w] = 0u;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (warp == 0) TC_TRACE(7, (int)(2 * ((m - blockIdx.x) / gridDim.x) + 1));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == MMA_WARP0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(TMEM_COLS));
}

template <int L>
static size_t tc_smem(const TcHistArgs& a, int nbuf, bool resp) {
  using namespace tc;
  const int C = ((resp ? a.q : a.nbx * a.bw) + X - 1) / X;
  const int nbins = 1 << a.nbits;
  return (size_t)L * 2 * BMAT_BYTES + nbuf * (size_t)(2 * C + 2) * CHUNK_BYTES +
         (resp ? 0 : sizeof(unsigned) * (size_t)a.nby * a.nbx * ((nbins + 1) / 2));
}
constexpr size_t TC_SMEM_MAX = 225 * 1024;

template <int L, bool RESP>
static int launch_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st) {
  using namespace tc;
  // two map buffers (the next map lands while this one is converted) when they fit
  const int nbuf = tc_smem<L>(a, 2, RESP) <= TC_SMEM_MAX ? 2 : 1;
  size_t smem = tc_smem<L>(a, nbuf, RESP);
  if (smem > TC_SMEM_MAX) return DDCCA_ECONFIG;
  // one CTA per SM: it allocates all 512 TMEM columns (a second resident CTA would spin in
  // tcgen05.alloc until the first exits), so ask for more than half the shared memory
  smem = std::max<size_t>(smem, 116 * 1024);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (!make_map(&tmap, a.in, a.n_maps, a.p, a.q, 4, RP, 1)) return DDCCA_ECONFIG;
  auto kern = conv_hist_tc_kernel<L, RESP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(a.n_maps, sms);
  kern<<<grid, THREADS, smem, st>>>(a, taps_dev, nbuf, tmap);
  return check_launch(RESP ? "conv_resp_tc_kernel" : "conv_hist_tc_kernel");
}

static bool tc_shape_ok(const TcHistArgs& a) {
  if (const char* e = getenv("DDCCA_CONV_TC"))
    if (e[0] == '0') return false;  // A/B switch: FFMA kernels
  // maps of <= 128 rows (one TMEM lane per row), <= 8 filters, odd windows up to 7 (the TMEM A
  // ring of 3 x l x 16 columns plus 2 accumulators), TMA-aligned rows, "same" padding
  if (a.p > 128 || a.count > tc::NF || a.n_maps < 1 || a.n_maps > INT32_MAX) return false;
  if (a.q % 4 != 0 || (reinterpret_cast<uintptr_t>(a.in) & 15)) return false;
  if (a.top != (a.l - 1) / 2 || a.left != (a.l - 1) / 2) return false;
  return a.l == 3 || a.l == 5 || a.l == 7;
}

bool conv_hist_tc_covers(const TcHistArgs& a) {
  if (!tc_shape_ok(a) || a.nbits > 8) return false;
  // a staged map, the banded B and the bins in shared memory
  return tc_smem<7>(a, 1, false) <= TC_SMEM_MAX;
}

bool conv_resp_tc_covers(const TcHistArgs& a) {
  // >= 2 column blocks per map (the epilogue's per-map scale ring assumes it), 32-byte stores
  if (!tc_shape_ok(a) || a.q < 16 || (reinterpret_cast<uintptr_t>(a.resp) & 31)) return false;
  return tc_smem<7>(a, 1, true) <= TC_SMEM_MAX;
}

int conv_hist_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st) {
  if (!conv_hist_tc_covers(a)) return DDCCA_ECONFIG;
  switch (a.l) {
    case 3: return launch_tc<3, false>(a, taps_dev, st);
    case 5: return launch_tc<5, false>(a, taps_dev, st);
    case 7: return launch_tc<7, false>(a, taps_dev, st);
    default: return DDCCA_ECONFIG;
  }
}

int conv_resp_tc(const TcHistArgs& a, const float* taps_dev, cudaStream_t st) {
  if (!conv_resp_tc_covers(a)) return DDCCA_ECONFIG;
  switch (a.l) {
    case 3: return launch_tc<3, true>(a, taps_dev, st);
    case 5: return launch_tc<5, true>(a, taps_dev, st);
    case 7: return launch_tc<7, true>(a, taps_dev, st);
    default: return DDCCA_ECONFIG;
  }
}

}  // namespace ddcca
