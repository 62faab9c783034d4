// K6 / K6-final+K7+K8 with filter taps in the constant bank.
//
// Same arithmetic as conv.cu (zero-mean taps, per-thread DC shift c, float32
// FFMA, filter-minor output; sign-hash LSB-first; block histograms), but the
// taps travel as a kernel parameter block, so every FFMA reads its weight
// straight from the constant bank (FFMA R, R, c[0x0][imm], R): no weight
// loads, no register-bank pressure from a third register operand, and the
// whole (L1 x L2 x NF) tap loop is unrolled with immediate offsets.
//
// conv_hist_kernel fuses the last layer: a CTA owns BR block-rows of one map
// (BR * bh output rows x nbx * bw columns, the only pixels the histograms
// read), computes the sign codes of that band into shared memory and builds
// the per-block histograms with warp-private shared bins, writing the counts
// straight into the feature matrix. Codes never reach HBM.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "convtc.cuh"
#include "tma.cuh"

namespace ddcca {

constexpr int CC_THREADS = 256;
// packed f32x2 FMAs in the tap loop (sm_100a): on for the fused last layer, where the
// histogram phases compete for issue slots; the plain conv measured faster without
constexpr bool CC_FFMA2_HIST = true;
constexpr bool CC_FFMA2_CONV = false;
// FFMAs per strip up to which the tap-row loop is unrolled. 0: always rolled. (Unrolling
// does not turn the taps into immediate constant operands on sm_100a: the compiler
// still stages them through uniform registers, at more LDCU per FFMA for short strips.)
constexpr int CC_FULL_UNROLL = 0;

// Zero-mean taps of the current launch, [(row * L2 + col) * NF + filter]. Written per
// launch on the launching stream (cudaMemcpyToSymbolAsync from g_taps_stage, which a
// one-CTA prep kernel fills from the device filter pack, or from the host pack): the
// FFMAs read them straight from the constant bank and no host copy of the solve's filters
// is needed (device-resident hand-off between solve and conv). Launches on one stream are
// ordered; the entry points document that concurrent streams must be ordered by the caller.
constexpr int MAX_TAPS = 9 * 9 * 16;
__constant__ float c_taps[MAX_TAPS];
__device__ float g_taps_stage[MAX_TAPS];

struct CArgs {
  const float* in;
  int64_t n_maps;
  int p, q, top, left, oh, ow, count, center;
  int responses;  // conv_hist: input maps are filter responses (DDCCA_CONV_RESPONSES)
  void* out;
  // fused histogram
  int bh, bw, nby, nbx, br, kind, nbits;
  void* counts;
  int64_t gpr, row_stride, group_stride;
  int use_tma;  // stage tiles with one cp.async.bulk.tensor per tile (else per-element cp.async)
};

__device__ __forceinline__ void cp_async4c(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 4 : 0));
}

// Staged tile row: sh leading columns (so the TMA box origin is 16 B aligned), the
// strips' inputs, and float4 over-read slack; a multiple of 4 floats.
__host__ __device__ inline int cc_tile_width(int cols, int l2, int px, int sh) {
  const int G = (cols + px - 1) / px;
  return ((G * px + l2 + sh + 2) + 3) / 4 * 4;
}
// Tile buffer stride in floats (128 B aligned buffers for the TMA destination).
__host__ __device__ inline int cc_buf_elems(int rows_in, int wt) { return (rows_in * wt + 31) / 32 * 32; }

// PY x PX x NF responses of the strip whose top-left output sits at tile row r0, column v0.
// Each staged input row feeds the PY output rows it overlaps, so one row of x values
// and one row of taps serve PY * PX * NF FFMAs.
// Tile column v + SH holds padded column v.
template <int L1, int L2, int NF, int PX, int PY, int SH, bool F2 = false, bool CEN = true>
__device__ __forceinline__ void cc_strip(const float* __restrict__ tile, int Wt, int r0,
                                         int v0, bool center, float (&acc)[PY][PX][NF]) {
  const float c = (CEN && center) ? tile[(r0 + (L1 - 1) / 2) * Wt + v0 + SH + (L2 - 1) / 2] : 0.f;
#pragma unroll
  for (int y = 0; y < PY; ++y)
#pragma unroll
    for (int j = 0; j < PX; ++j)
#pragma unroll
      for (int g = 0; g < NF; ++g) acc[y][j][g] = 0.f;
  auto row_step = [&](int a) {
    const float* row = tile + (r0 + a) * Wt + v0;
    constexpr int NX = PX + L2 - 1;
    constexpr int N4 = (NX + SH + 3) / 4;
    float xr[4 * N4];
#pragma unroll
    for (int t4 = 0; t4 < N4; ++t4) {
      const float4 v = *reinterpret_cast<const float4*>(row + 4 * t4);
      xr[4 * t4 + 0] = v.x;
      xr[4 * t4 + 1] = v.y;
      xr[4 * t4 + 2] = v.z;
      xr[4 * t4 + 3] = v.w;
    }
    float x[NX];
#pragma unroll
    for (int t = 0; t < NX; ++t) x[t] = CEN ? xr[t + SH] - c : xr[t + SH];
#pragma unroll
    for (int y = 0; y < PY; ++y) {
      const int ta = a - y;  // tap row of output row y that reads input row a
      if (ta >= 0 && ta < L1) {
        if constexpr (NF % 2 == 0 && F2) {
          // packed fma.rn.f32x2 over filter pairs (g, g+1): a warp-uniform weight pair, the
          // broadcast x value, an accumulator pair -- half the issue slots, same per-lane
          // rounding as two fmaf
#pragma unroll
          for (int b = 0; b < L2; ++b)
#pragma unroll
            for (int j = 0; j < PX; ++j)
#pragma unroll
              for (int g = 0; g < NF; g += 2) {
                const float2 w2 = make_float2(c_taps[(ta * L2 + b) * NF + g], c_taps[(ta * L2 + b) * NF + g + 1]);
                const float2 a2 = __ffma2_rn(w2, make_float2(x[j + b], x[j + b]),
                                             make_float2(acc[y][j][g], acc[y][j][g + 1]));
                acc[y][j][g] = a2.x;
                acc[y][j][g + 1] = a2.y;
              }
        } else {
#pragma unroll
          for (int b = 0; b < L2; ++b)
#pragma unroll
            for (int g = 0; g < NF; ++g)
#pragma unroll
              for (int j = 0; j < PX; ++j)
                acc[y][j][g] = fmaf(c_taps[(ta * L2 + b) * NF + g], x[j + b], acc[y][j][g]);
        }
      }
    }
  };
  if constexpr (L1 * L2 * NF * PX * PY <= CC_FULL_UNROLL) {
    // small bodies: every tap is an immediate constant-bank operand of its FFMA
#pragma unroll
    for (int a = 0; a < L1 + PY - 1; ++a) row_step(a);
  } else {
    // large bodies stay rolled over rows (inside the instruction cache); the taps of
    // a row are warp-uniform constant-bank loads feeding the FFMAs
#pragma unroll 1
    for (int a = 0; a < L1 + PY - 1; ++a) row_step(a);
  }
}

template <int NF, int PX, int PY>
__device__ __forceinline__ unsigned cc_code(const float (&acc)[PY][PX][NF], int y, int j, int count) {
  // filters g >= count have all-zero taps, so their response is +0 and their bit is 0
  unsigned code = 0;
#pragma unroll
  for (int g = 0; g < NF; ++g)
    if (acc[y][j][g] > 0.f) code |= 1u << g;
  return code;
}

// Stage rows [row0, row0 + rows) (padded coordinates) x tile columns [0, Wt) of map m,
// tile column c = image column c - sh - left, zeros outside the map. TMA: thread 0
// issues one box and arms the buffer's mbarrier; else every thread issues 4-byte
// cp.async copies (one commit group per tile).
__device__ __forceinline__ void cc_issue(const CArgs& A, const CUtensorMap* tm, uint64_t* bar, int sh, int64_t m,
                                         int row0, int rows, int Wt, float* buf) {
  if (A.use_tma) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, (unsigned)(rows * Wt * 4));
      tma_load_3d(buf, tm, -(A.left + sh), row0 - A.top, (int)m, bar);
    }
    return;
  }
  const float* img = A.in + m * (int64_t)A.p * A.q;
  for (int r = threadIdx.x >> 5; r < rows; r += blockDim.x / 32) {
    const int i = row0 + r - A.top;
    const bool rok = i >= 0 && i < A.p;
    const float* rowp = img + (int64_t)i * A.q;
    for (int c = threadIdx.x & 31; c < Wt; c += 32) {
      const int j = c - sh - A.left;
      const bool ok = rok && j >= 0 && j < A.q;
      cp_async4c(buf + r * Wt + c, ok ? rowp + j : A.in, ok);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cc_commit_empty(const CArgs& A) {
  if (!A.use_tma) asm volatile("cp.async.commit_group;\n" ::);
}
// Wait until the tile of iteration `it` sits in its buffer.
__device__ __forceinline__ void cc_wait(const CArgs& A, uint64_t* bars, int it) {
  if (A.use_tma) {
    mbar_wait(&bars[it & 1], (unsigned)((it >> 1) & 1));
  } else {
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
  }
}
__device__ __forceinline__ void cc_init_bars(const CArgs& A, uint64_t* bars) {
  if (A.use_tma && threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
}

// Persistent float-response conv (MODE 0): tiles = (map, band of rows_per_tile output rows).
template <int L1, int L2, int NF, int PX, int PY, int SH, int NT>
__global__ void __launch_bounds__(NT, (NT <= 128 ? 3 : 1))
    conv_c_kernel(CArgs A, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t bars[2];
  const int G = (A.ow + PX - 1) / PX;
  const int Wt = cc_tile_width(A.ow, L2, PX, SH);
  const int rows_out = PY * max(1, NT / G);  // output rows per tile (one strip per thread)
  const int rows_in = rows_out + L1 - 1;
  const int bands = (A.oh + rows_out - 1) / rows_out;
  const int64_t total = A.n_maps * bands;
  float* bufs = sm;
  const int belems = cc_buf_elems(rows_in, Wt);
  cc_init_bars(A, bars);
  int64_t t = blockIdx.x;
  if (t < total) cc_issue(A, &tmap, &bars[0], SH, t / bands, (int)(t % bands) * rows_out, rows_in, Wt, bufs);
  const int64_t plane = (int64_t)A.oh * A.ow;
  for (int it = 0; t < total; t += gridDim.x, ++it) {
    const float* cur = bufs + (it & 1) * belems;
    const int64_t tn = t + gridDim.x;
    if (tn < total)
      cc_issue(A, &tmap, &bars[(it + 1) & 1], SH, tn / bands, (int)(tn % bands) * rows_out, rows_in, Wt,
               bufs + ((it + 1) & 1) * belems);
    else
      cc_commit_empty(A);
    cc_wait(A, bars, it);
    const int64_t m = t / bands;
    const int u0 = (int)(t % bands) * rows_out;
    const int r = threadIdx.x / G * PY, gi = threadIdx.x % G;
    if (r < rows_out && u0 + r < A.oh) {
      const int v0 = gi * PX;
      float acc[PY][PX][NF];
      cc_strip<L1, L2, NF, PX, PY, SH, (CC_FFMA2_CONV || NF > 8)>(cur, Wt, r, v0, A.center, acc);
#pragma unroll
      for (int y = 0; y < PY; ++y) {
        const int u = u0 + r + y;
        if (u >= A.oh) break;
        float* o = static_cast<float*>(A.out) + m * A.count * plane + (int64_t)u * A.ow + v0;
        if (v0 + PX <= A.ow && (A.ow & 3) == 0 && PX % 4 == 0) {
#pragma unroll
          for (int g = 0; g < NF; ++g)
            if (g < A.count)
#pragma unroll
              for (int j4 = 0; j4 < PX / 4; ++j4)
                *reinterpret_cast<float4*>(o + g * plane + 4 * j4) = make_float4(
                    acc[y][4 * j4][g], acc[y][4 * j4 + 1][g], acc[y][4 * j4 + 2][g], acc[y][4 * j4 + 3][g]);
        } else {
#pragma unroll
          for (int j = 0; j < PX; ++j)
            if (v0 + j < A.ow)
#pragma unroll
              for (int g = 0; g < NF; ++g)
                if (g < A.count) o[g * plane + j] = acc[y][j][g];
        }
      }
    }
    __syncthreads();
  }
}

// Fused last layer: sign codes of BR block-rows go straight into per-block shared
// bins (packed u16 pairs, CTA-wide atomics); then one warp per block writes the
// counts into the feature row and clears the bins.
// RESP: the input maps are filter responses of a previous layer (zero-mean on average), so
// the float32 shift by a window pixel that keeps image DC out of the sums is skipped.
template <int L1, int L2, int NF, int PX, int PY, int SH, int NT, bool RESP>
__global__ void __launch_bounds__(NT, (NT <= 128 ? 3 : 1))
    conv_hist_kernel(CArgs A, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t bars[2];
  const int cols = A.nbx * A.bw;                 // only pixels inside blocks are needed
  const int G = (cols + PX - 1) / PX;
  const int Wt = cc_tile_width(cols, L2, PX, SH);
  const int rows_out = A.br * A.bh;
  const int rows_in = (rows_out + PY - 1) / PY * PY + L1 - 1;
  const int belems = cc_buf_elems(rows_in, Wt);
  const int bands = (A.nby + A.br - 1) / A.br;
  const int64_t total = A.n_maps * bands;
  const int nbins = 1 << A.nbits;
  const int words = (nbins + 1) / 2;
  const int nwarps = NT / 32;
  float* bufs = sm;                                                // 2 x [rows_in][Wt]
  unsigned* bins = reinterpret_cast<unsigned*>(bufs + 2 * belems);  // [br][nbx][words]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int w = threadIdx.x; w < A.br * A.nbx * words; w += NT) bins[w] = 0u;
  cc_init_bars(A, bars);
  int64_t t = blockIdx.x;
  if (t < total) cc_issue(A, &tmap, &bars[0], SH, t / bands, (int)(t % bands) * rows_out, rows_in, Wt, bufs);
  for (int it = 0; t < total; t += gridDim.x, ++it) {
    const float* cur = bufs + (it & 1) * belems;
    const int64_t tn = t + gridDim.x;
    if (tn < total)
      cc_issue(A, &tmap, &bars[(it + 1) & 1], SH, tn / bands, (int)(tn % bands) * rows_out, rows_in, Wt,
               bufs + ((it + 1) & 1) * belems);
    else
      cc_commit_empty(A);
    cc_wait(A, bars, it);
    const int64_t m = t / bands;
    const int by0 = (int)(t % bands) * A.br;
    const int nbr = min(A.br, A.nby - by0);      // block rows in this band
    // 1) responses -> codes -> bins of the pixel's block
    const int band_rows = nbr * A.bh;
    for (int s = threadIdx.x; s < (band_rows + PY - 1) / PY * G; s += NT) {
      const int r = s / G * PY, v0 = (s % G) * PX;
      float acc[PY][PX][NF];
      cc_strip<L1, L2, NF, PX, PY, SH, CC_FFMA2_HIST, !RESP>(cur, Wt, r, v0, A.center, acc);
      const int bx0 = v0 / A.bw, rem0 = v0 - bx0 * A.bw;
      if (v0 + PX <= cols && rem0 + PX <= A.bw) {
        // whole strip inside one block: no per-pixel bounds or block stepping
#pragma unroll
        for (int y = 0; y < PY; ++y)
          if (r + y < band_rows) {
            unsigned* bb = bins + ((r + y) / A.bh * A.nbx + bx0) * words;
#pragma unroll
            for (int j = 0; j < PX; ++j) {
              const unsigned code = cc_code<NF, PX, PY>(acc, y, j, A.count);
              atomicAdd(&bb[code >> 1], 1u << ((code & 1u) << 4));
            }
          }
        continue;
      }
#pragma unroll
      for (int y = 0; y < PY; ++y)
        if (r + y < band_rows) {
          unsigned* rbins = bins + (r + y) / A.bh * A.nbx * words;
          int bx = bx0, rem = rem0;
#pragma unroll
          for (int j = 0; j < PX; ++j) {
            if (v0 + j < cols) {
              const unsigned code = cc_code<NF, PX, PY>(acc, y, j, A.count);
              atomicAdd(&rbins[bx * words + (code >> 1)], 1u << ((code & 1u) << 4));
            }
            if (++rem == A.bw) {
              rem = 0;
              ++bx;
            }
          }
        }
    }
    __syncthreads();
    // 2) one warp per block: counts out, bins cleared for the next tile
    for (int blk = warp; blk < nbr * A.nbx; blk += nwarps) {
      const int rb = blk / A.nbx, bx = blk - rb * A.nbx;
      unsigned* wb = bins + blk * words;
      const int64_t blk_global = (int64_t)(by0 + rb) * A.nbx + bx;
      const int64_t base = (m / A.gpr) * A.row_stride + (m % A.gpr) * A.group_stride + blk_global * nbins;
      if (A.kind == 2) {
        uint16_t* o = static_cast<uint16_t*>(A.counts) + base;
        for (int b = lane; b < nbins; b += 32) o[b] = (uint16_t)((wb[b >> 1] >> ((b & 1) * 16)) & 0xffffu);
      } else if ((nbins & 7) == 0) {
        // 8 bins (4 words) per lane per store
        uint8_t* o = static_cast<uint8_t*>(A.counts) + base;
        for (int b8 = lane * 8; b8 < nbins; b8 += 256) {
          const uint4 wv = *reinterpret_cast<const uint4*>(wb + (b8 >> 1));
          const unsigned ww[4] = {wv.x, wv.y, wv.z, wv.w};
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            unsigned c = (ww[k >> 1] >> ((k & 1) * 16)) & 0xffffu;
            c = c > 255u ? 255u : c;
            if (k < 4) lo |= c << (8 * k);
            else hi |= c << (8 * (k - 4));
          }
          *reinterpret_cast<uint2*>(o + b8) = make_uint2(lo, hi);
        }
      } else {
        uint8_t* o = static_cast<uint8_t*>(A.counts) + base;
        for (int b = lane; b < nbins; b += 32) {
          const unsigned c = (wb[b >> 1] >> ((b & 1) * 16)) & 0xffffu;
          o[b] = (uint8_t)(c > 255u ? 255u : c);
        }
      }
      __syncwarp();
      for (int w = lane; w < words; w += 32) wb[w] = 0u;
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------------- host side

// One CTA: zero-mean (per-window centering) taps of a device filter pack, padded to nf filters.
__global__ void taps_prep_kernel(const float* __restrict__ pack, int count, int d, int nf, int center, float* out) {
  __shared__ double mean[16];
  if (threadIdx.x < nf) {
    double m = 0.0;
    if (center && (int)threadIdx.x < count) {
      for (int k = 0; k < d; ++k) m += (double)pack[k * count + threadIdx.x];
      m /= d;
    }
    mean[threadIdx.x] = m;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d * nf; e += blockDim.x) {
    const int k = e / nf, g = e - k * nf;
    out[e] = g < count ? (float)((double)pack[k * count + g] - mean[g]) : 0.f;
  }
}

static void zero_mean_taps(const float* pack_host, int count, int d, int nf, bool center, float* out) {
  for (int g = 0; g < nf; ++g) {
    double mean = 0.0;
    if (center && g < count) {
      for (int k = 0; k < d; ++k) mean += (double)pack_host[k * count + g];
      mean /= d;
    }
    for (int k = 0; k < d; ++k)
      out[k * nf + g] = g < count ? (float)((double)pack_host[k * count + g] - mean) : 0.f;
  }
}

// Zero-mean taps of the launch into g_taps_stage (from the device pack, or the host pack)
// and, for the FFMA kernels (to_const), on into the constant bank. Stream-ordered.
static int stage_taps(const float* pack, bool pack_on_device, int count, int d, int nf, bool center, bool to_const,
                      cudaStream_t st) {
  if (d * nf > MAX_TAPS) return fail(DDCCA_ECONFIG, "%d taps exceed the constant tap bank", d * nf);
  if (pack_on_device) {
    float* stage = nullptr;
    if (cudaGetSymbolAddress(reinterpret_cast<void**>(&stage), g_taps_stage) != cudaSuccess)
      return fail(DDCCA_ECUDA, "tap stage symbol");
    taps_prep_kernel<<<1, 256, 0, st>>>(pack, count, d, nf, center ? 1 : 0, stage);
    DDCCA_TRY(check_launch("taps_prep_kernel"));
    if (to_const && cudaMemcpyToSymbolAsync(c_taps, stage, sizeof(float) * d * nf, 0, cudaMemcpyDeviceToDevice, st) !=
                        cudaSuccess)
      return fail(DDCCA_ECUDA, "tap bank copy");
    return DDCCA_OK;
  }
  std::vector<float> w((size_t)d * nf);
  zero_mean_taps(pack, count, d, nf, center, w.data());
  // pageable host source: staged by the driver before the call returns, so w may go away
  const cudaError_t e = to_const ? cudaMemcpyToSymbolAsync(c_taps, w.data(), sizeof(float) * d * nf, 0,
                                                           cudaMemcpyHostToDevice, st)
                                 : cudaMemcpyToSymbolAsync(g_taps_stage, w.data(), sizeof(float) * d * nf, 0,
                                                           cudaMemcpyHostToDevice, st);
  return e == cudaSuccess ? DDCCA_OK : fail(DDCCA_ECUDA, "tap upload: %s", cudaGetErrorString(e));
}

// Grid for a persistent kernel: resident CTAs per SM x SMs, capped by the tile count.
template <typename K>
static int persistent_grid(K kern, size_t smem, int64_t tiles, int threads = CC_THREADS) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (const char* e = getenv("DDCCA_CONV_CTAS_PER_SM")) per_sm = std::min(per_sm, std::max(1, atoi(e)));  // A/B only
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)std::max(1, per_sm) * sms));
  return (int)grid;
}

// TMA staging needs 16 B aligned rows (q % 4 == 0) and a box of at most 256 x 256;
// DDCCA_NO_TMA=1 forces the cp.async path (A/B checks).
static bool cc_tma_map(CArgs& A, int sh, int Wt, int rows_in, CUtensorMap* tm) {
  const char* env = getenv("DDCCA_NO_TMA");
  const bool disabled = env && env[0] == '1';
  memset(tm, 0, sizeof(*tm));
  A.use_tma = 0;
  if (disabled || (A.left + sh) % 4 != 0 || A.q % 4 != 0 || Wt > 256 || rows_in > 256 || (reinterpret_cast<uintptr_t>(A.in) & 15) ||
      A.n_maps > INT32_MAX)
    return false;
  A.use_tma = make_map(tm, A.in, A.n_maps, A.p, A.q, Wt, rows_in, 1) ? 1 : 0;
  return A.use_tma != 0;
}

template <int L1, int L2, int NF, int PX, int PY, int SH, int NT = CC_THREADS>
static int run_conv_c(CArgs A, const float* pack, bool pack_dev, cudaStream_t st) {
  const int G = (A.ow + PX - 1) / PX;
  const int Wt = cc_tile_width(A.ow, L2, PX, SH);
  const int rows_out = PY * std::max(1, NT / G);
  const int rows_in = rows_out + L1 - 1;
  CUtensorMap tm;
  if (SH != 0 && !cc_tma_map(A, SH, Wt, rows_in, &tm)) return DDCCA_ECONFIG;  // caller retries with SH = 0
  if (SH == 0) cc_tma_map(A, SH, Wt, rows_in, &tm);
  const size_t smem = sizeof(float) * 2 * (size_t)cc_buf_elems(rows_in, Wt);
  if (smem > 200 * 1024) return fail(DDCCA_ECONFIG, "conv: map row too wide for shared-memory staging");
  const int64_t tiles = A.n_maps * ((A.oh + rows_out - 1) / rows_out);
  auto kern = conv_c_kernel<L1, L2, NF, PX, PY, SH, NT>;
  const int grid = persistent_grid(kern, smem, tiles, NT);
  DDCCA_TRY(stage_taps(pack, pack_dev, A.count, L1 * L2, NF, A.center, true, st));
  kern<<<grid, NT, smem, st>>>(A, tm);
  return check_launch("conv_c_kernel");
}

template <int L1, int L2, int NF, int PX, int PY, int SH, int NT = CC_THREADS>
static int run_conv_hist(CArgs A, const float* pack, bool pack_dev, cudaStream_t st) {
  const int cols = A.nbx * A.bw;
  const int G = (cols + PX - 1) / PX;
  // block rows per CTA: about one strip per thread, two when a block row alone fills at
  // least half the CTA (amortizes the per-tile staging, barriers and count output)
  const int strips_br = std::max(1, A.bh * G);
  A.br = std::max(1, std::min(A.nby, (strips_br * 2 >= NT ? 2 : 1) * PY * NT / strips_br));
  const int rows_out = A.br * A.bh;
  const int Wt = cc_tile_width(cols, L2, PX, SH);
  const int rows_in = (rows_out + PY - 1) / PY * PY + L1 - 1;
  CUtensorMap tm;
  if (SH != 0 && !cc_tma_map(A, SH, Wt, rows_in, &tm)) return DDCCA_ECONFIG;
  if (SH == 0) cc_tma_map(A, SH, Wt, rows_in, &tm);
  const int nbins = 1 << A.nbits;
  const size_t smem = sizeof(float) * 2 * (size_t)cc_buf_elems(rows_in, Wt) +
                      sizeof(unsigned) * (size_t)A.br * A.nbx * (size_t)((nbins + 1) / 2);
  if (smem > 220 * 1024) return fail(DDCCA_ECONFIG, "conv_hist: band does not fit shared memory");
  const int64_t tiles = A.n_maps * ((A.nby + A.br - 1) / A.br);
  auto kern = A.responses ? conv_hist_kernel<L1, L2, NF, PX, PY, SH, NT, true>
                          : conv_hist_kernel<L1, L2, NF, PX, PY, SH, NT, false>;
  const int grid = persistent_grid(kern, smem, tiles, NT);
  DDCCA_TRY(stage_taps(pack, pack_dev, A.count, L1 * L2, NF, A.center, true, st));
  kern<<<grid, NT, smem, st>>>(A, tm);
  return check_launch("conv_hist_kernel");
}

// Column shift that 16 B aligns the TMA box origin -(left + sh) for "same" padding.
constexpr int same_shift(int l2) { return (4 - ((l2 - 1) / 2) % 4) % 4; }

template <bool HIST, int L, int NF, int PX, int PY, int NT = CC_THREADS>
static int run_shape(const CArgs& A, const float* pack_host, bool pack_dev, cudaStream_t st) {
  constexpr int S = same_shift(L);
  const int want = (4 - A.left % 4) % 4;
  if (S != 0 && want == S) {
    const int rc = HIST ? run_conv_hist<L, L, NF, PX, PY, S, NT>(A, pack_host, pack_dev, st)
                        : run_conv_c<L, L, NF, PX, PY, S, NT>(A, pack_host, pack_dev, st);
    if (rc != DDCCA_ECONFIG) return rc;
  }
  return HIST ? run_conv_hist<L, L, NF, PX, PY, 0, NT>(A, pack_host, pack_dev, st)
              : run_conv_c<L, L, NF, PX, PY, 0, NT>(A, pack_host, pack_dev, st);
}

// Dispatch over the compiled (window, filter-count) shapes; DDCCA_ECONFIG = not covered.
template <bool HIST>
static int dispatch(const CArgs& A, int l1, int l2, const float* pack_host, bool pack_dev, cudaStream_t st) {
  // 8 filters: 16-pixel strips in 128-thread CTAs (3 per SM) halve the tap loads per
  // FFMA; DDCCA_CH8=1 selects the 8-pixel / 256-thread form (A/B)
  const char* ch8 = getenv("DDCCA_CH8");
  if (A.count <= 8 && !(ch8 && ch8[0] == '1')) {
#define DDCCA_CH(L) \
    if (l1 == L && l2 == L) return run_shape<HIST, L, 8, 16, 1, 128>(A, pack_host, pack_dev, st);
    DDCCA_CH(3)
    DDCCA_CH(5)
    DDCCA_CH(7)
    DDCCA_CH(9)
#undef DDCCA_CH
  }
  // 9..16 filters: 8-pixel strips in 128-thread CTAs (the 4-pixel / 256-thread table below
  // spends one tap load per 8 FFMAs)
  // wide histograms (2^n_bits > 256 shared bins per block): 8-pixel strips, 256-thread CTAs
  if (HIST && A.nbits > 8 && A.count > 8 && A.count <= 12 && !(ch8 && ch8[0] == '1')) {
    if (l1 == 7 && l2 == 7) return run_shape<true, 7, 12, 8, 1, 256>(A, pack_host, pack_dev, st);
    if (l1 == 9 && l2 == 9) return run_shape<true, 9, 12, 8, 1, 256>(A, pack_host, pack_dev, st);
  }
  // (not for wide histograms: 2^n_bits shared bins per block would leave one small CTA per SM)
  if (A.count > 8 && A.count <= 16 && !(HIST && A.nbits > 8) && !(ch8 && ch8[0] == '1')) {
#define DDCCA_CH(L, NFV) \
    if (l1 == L && l2 == L && A.count <= NFV && (HIST || NFV <= 12)) \
      return run_shape<HIST, L, NFV, 8, 1, 128>(A, pack_host, pack_dev, st);
    DDCCA_CH(7, 12)
    DDCCA_CH(9, 12)
    DDCCA_CH(3, 16)
    DDCCA_CH(5, 16)
    DDCCA_CH(7, 16)
    DDCCA_CH(9, 16)
#undef DDCCA_CH
  }
#define DDCCA_CC(L, NFV, PXV, PYV) \
  if (l1 == L && l2 == L && A.count <= NFV) return run_shape<HIST, L, NFV, PXV, PYV>(A, pack_host, pack_dev, st);
  DDCCA_CC(3, 8, 8, 1)
  DDCCA_CC(5, 8, 8, 1)
  DDCCA_CC(7, 8, 8, 1)
  DDCCA_CC(9, 8, 8, 1)
  DDCCA_CC(3, 16, 4, 1)
  DDCCA_CC(5, 16, 4, 1)
  DDCCA_CC(7, 12, 4, 1)
  DDCCA_CC(7, 16, 4, 1)
  DDCCA_CC(9, 12, 4, 1)
  DDCCA_CC(9, 16, 4, 1)
#undef DDCCA_CC
  return fail(DDCCA_ECONFIG, "no constant-bank conv instance for %dx%d with %d filters", l1, l2, A.count);
}

}  // namespace ddcca

using namespace ddcca;

namespace {

thread_local int g_last_hist_path = 0;  // 1: the last conv-histogram launch ran on the tensor cores
thread_local int g_last_conv_path = 0;  // 1: the last conv (responses) launch ran on the tensor cores

int conv_entry(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* pack, bool pack_dev, int count,
               int center, float* out, void* stream) {
  Geo g{};
  DDCCA_TRY(make_geo(gg, &g));
  if (g.stride != 1) return fail(DDCCA_ECONFIG, "constant-bank conv needs stride 1");
  if (count < 1 || count > g.d) return fail(DDCCA_ECONFIG, "filter count %d outside [1, %d]", count, g.d);
  if (!pack) return fail(DDCCA_ESHAPE, "null taps");
  if (n_maps == 0) return DDCCA_OK;
  cudaStream_t st = as_stream(stream);
  g_last_conv_path = 0;
  if (g.l1 == g.l2 && g.oh == g.p && g.ow == g.q) {
    // tensor-core kernel (convtc.cu, responses mode): each map shifted by its mean when the
    // windows are centered (zero-mean taps: the responses do not depend on the shift)
    TcHistArgs t{};
    t.in = in; t.n_maps = n_maps; t.p = g.p; t.q = g.q; t.top = g.top; t.left = g.left; t.l = g.l1;
    t.count = count; t.center = center & 1; t.resp = out; t.dc_shift = center & 1; t.nbits = 1;
    if (conv_resp_tc_covers(t)) {
      float* stage = nullptr;
      if (cudaGetSymbolAddress(reinterpret_cast<void**>(&stage), g_taps_stage) != cudaSuccess)
        return fail(DDCCA_ECUDA, "tap stage symbol");
      DDCCA_TRY(stage_taps(pack, pack_dev, count, g.d, TC_FILTERS, center & 1, false, st));
      const int rc = conv_resp_tc(t, stage, st);
      if (rc != DDCCA_ECONFIG) {
        g_last_conv_path = rc == DDCCA_OK ? 1 : 0;
        return rc;
      }
    }
  }
  CArgs A{};
  A.in = in; A.n_maps = n_maps; A.p = g.p; A.q = g.q; A.top = g.top; A.left = g.left; A.oh = g.oh; A.ow = g.ow;
  A.count = count; A.center = center; A.out = out;
  return dispatch<false>(A, g.l1, g.l2, pack, pack_dev, st);
}

int conv_hist_entry(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* pack, bool pack_dev,
                    int count, int center, int block_h, int block_w, void* counts, int count_kind,
                    int64_t groups_per_row, int64_t row_stride, int64_t group_stride, void* stream) {
  Geo g{};
  DDCCA_TRY(make_geo(gg, &g));
  if (g.stride != 1) return fail(DDCCA_ECONFIG, "fused conv-histogram needs stride 1");
  if (count < 1 || count > 16) return fail(DDCCA_ECONFIG, "hash width %d outside the fused path (1..16)", count);
  if (block_h < 1 || block_w < 1 || g.oh < block_h || g.ow < block_w)
    return fail(DDCCA_ESHAPE, "%dx%d blocks do not fit a %dx%d map", block_h, block_w, g.oh, g.ow);
  const int bpc = block_h * block_w;
  if ((count_kind == 0 && bpc > 255) || (count_kind == 1 && bpc > 510) || bpc > 65535)
    return fail(DDCCA_ECONFIG, "count storage cannot hold %d pixels per block", bpc);
  if (!pack) return fail(DDCCA_ESHAPE, "null taps");
  if (n_maps == 0) return DDCCA_OK;
  cudaStream_t st = as_stream(stream);
  g_last_hist_path = 0;
  CArgs A{};
  A.in = in; A.n_maps = n_maps; A.p = g.p; A.q = g.q; A.top = g.top; A.left = g.left; A.oh = g.oh; A.ow = g.ow;
  A.count = count; A.center = center & 1; A.responses = (center & DDCCA_CONV_RESPONSES) ? 1 : 0; A.out = nullptr;
  A.bh = block_h; A.bw = block_w; A.nby = g.oh / block_h; A.nbx = g.ow / block_w; A.kind = count_kind;
  A.nbits = count; A.counts = counts; A.gpr = groups_per_row; A.row_stride = row_stride; A.group_stride = group_stride;
  if ((A.responses || !A.center) && g.l1 == g.l2) {
    // tensor-core kernel (convtc.cu) where no float32 DC shift is needed: filter-response
    // inputs or uncentered taps
    TcHistArgs t{};
    t.in = in; t.n_maps = n_maps; t.p = g.p; t.q = g.q; t.top = g.top; t.left = g.left; t.l = g.l1;
    t.count = count; t.center = A.center; t.bh = A.bh; t.bw = A.bw; t.nby = A.nby; t.nbx = A.nbx;
    t.kind = count_kind; t.nbits = count; t.counts = counts; t.gpr = groups_per_row; t.row_stride = row_stride;
    t.group_stride = group_stride;
    if (conv_hist_tc_covers(t)) {
      float* stage = nullptr;
      if (cudaGetSymbolAddress(reinterpret_cast<void**>(&stage), g_taps_stage) != cudaSuccess)
        return fail(DDCCA_ECUDA, "tap stage symbol");
      DDCCA_TRY(stage_taps(pack, pack_dev, count, g.d, TC_FILTERS, A.center, false, st));
      const int rc = conv_hist_tc(t, stage, st);
      if (rc != DDCCA_ECONFIG) {
        g_last_hist_path = rc == DDCCA_OK ? 1 : 0;
        return rc;
      }
    }
  }
  return dispatch<true>(A, g.l1, g.l2, pack, pack_dev, st);
}

}  // namespace

extern "C" {

int ddcca_conv_hw(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* conv_pack_host, int count,
                  int center, float* out, void* stream) {
  return conv_entry(in, n_maps, gg, conv_pack_host, false, count, center, out, stream);
}

int ddcca_conv_dev(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* conv_pack, int count,
                   int center, float* out, void* stream) {
  return conv_entry(in, n_maps, gg, conv_pack, true, count, center, out, stream);
}

int ddcca_conv_hist_hw(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* conv_pack_host, int count,
                       int center, int block_h, int block_w, void* counts, int count_kind, int64_t groups_per_row,
                       int64_t row_stride, int64_t group_stride, void* stream) {
  return conv_hist_entry(in, n_maps, gg, conv_pack_host, false, count, center, block_h, block_w, counts, count_kind,
                         groups_per_row, row_stride, group_stride, stream);
}

int ddcca_conv_hist_last_path(void) { return g_last_hist_path; }
int ddcca_conv_last_path(void) { return g_last_conv_path; }

int ddcca_conv_hist_dev(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* conv_pack, int count,
                        int center, int block_h, int block_w, void* counts, int count_kind, int64_t groups_per_row,
                        int64_t row_stride, int64_t group_stride, void* stream) {
  return conv_hist_entry(in, n_maps, gg, conv_pack, true, count, center, block_h, block_w, counts, count_kind,
                         groups_per_row, row_stride, group_stride, stream);
}

}  // extern "C"
