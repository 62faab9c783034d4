// K6 / K6-final+K7 / K8 / IQ expansion / explicit im2col.
//
// Reference semantics:
//   apply_filters (cascade.py:108-126): r[m, g, u, v] = W_g . centered patch
//     of map m at grid position (u, v); output filter-minor.
//   binarize + hash_combine (encoder.py:50-68): bit g = (r_g > 0) strictly,
//     code = sum_g bit_g << g (first map of a group is the LSB).
//   iq_block_features (encoder.py:71-99): per block bincount over 2^L bins,
//     -log(count / bpc), zero-bin policy; blocks in row-major scan order.
//
// B200 design: a direct float32 FFMA convolution. With L = 8..16 filters of
// d = 25..81 taps there is no GEMM shape that can feed tcgen05 (N = L is
// tiny and the im2col operand would have to be rebuilt d times per pixel in
// shared memory), so the conv is an FFMA-bound register-blocked stencil:
// each thread owns PX adjacent output pixels x NF filters, the input tile
// (rows + halo, full padded width) is staged once per block in shared
// memory, filter taps are read as float4 broadcasts. Per-window centering
// uses r = sum_k W_k (x_k - c) - sW (m - c) with a per-thread constant c
// taken from the thread's own window, which keeps the float32 sums free of
// the large DC cancellation. The final layer never writes
// its float32 responses: the sign bits are hashed in registers and only the
// code map (u8/u16) is stored; histograms use warp-private shared bins.
#include <algorithm>

#include "common.cuh"

namespace ddcca {

constexpr int CONV_THREADS = 256;

struct ConvArgs {
  const float* in;
  int64_t n_maps;
  int p, q, l1, l2, top, left, oh, ow;
  int count, center;
  const float* pack;  // [d][count]
  void* out;          // float (n_maps, count, oh, ow) or codes (n_maps, oh, ow)
};

// Tile row stride (floats) of the staged input: multiple of 4 so float4 loads stay aligned.
__host__ __device__ inline int conv_tile_width(int ow, int l2, int px) {
  const int G = (ow + px - 1) / px;
  return ((G * px + l2 + 3) + 3) / 4 * 4;
}

// Centered conv as an uncentered conv with zero-mean taps: for every window
//   sum_k W_k (x_k - m) = sum_k (W_k - mean(W)) (x_k - c)   for any constant c,
// so the kernel never forms window means. c is a per-thread constant (a pixel
// of the thread's own windows) that removes the DC part before the float32 sums.
// MODE 0: write float responses; MODE 1: write u8 codes; MODE 2: write u16 codes
__device__ __forceinline__ void cp_async4z(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 4 : 0));
}

// One output strip (PX pixels x NF filters) of one map from a staged tile.
template <int NF, int PX, int L2, int MODE>
__device__ __forceinline__ void conv_strip(const ConvArgs& A, const float* __restrict__ wsm,
                                           const float* __restrict__ tile, int Wt, int64_t m, int u, int v0,
                                           int r0) {
  const int l2 = L2 > 0 ? L2 : A.l2;
  const float c = A.center ? tile[(r0 + (A.l1 - 1) / 2) * Wt + v0 + (l2 - 1) / 2] : 0.f;
  float acc[PX][NF];
#pragma unroll
  for (int j = 0; j < PX; ++j)
#pragma unroll
    for (int g = 0; g < NF; ++g) acc[j][g] = 0.f;
  for (int a = 0; a < A.l1; ++a) {
    const float* row = tile + (r0 + a) * Wt + v0;
    if constexpr (L2 > 0) {
      constexpr int NX = PX + L2 - 1;
      float x[(NX + 3) / 4 * 4];
      if constexpr (PX % 4 == 0) {
#pragma unroll
        for (int t4 = 0; t4 < (NX + 3) / 4; ++t4) {
          const float4 v = *reinterpret_cast<const float4*>(row + 4 * t4);
          x[4 * t4 + 0] = v.x - c;
          x[4 * t4 + 1] = v.y - c;
          x[4 * t4 + 2] = v.z - c;
          x[4 * t4 + 3] = v.w - c;
        }
      } else {
#pragma unroll
        for (int t = 0; t < NX; ++t) x[t] = row[t] - c;
      }
#pragma unroll
      for (int b = 0; b < L2; ++b) {
        const float4* wp = reinterpret_cast<const float4*>(wsm + (a * L2 + b) * NF);
#pragma unroll
        for (int g4 = 0; g4 < NF / 4; ++g4) {
          const float4 w = wp[g4];
#pragma unroll
          for (int j = 0; j < PX; ++j) {
            acc[j][4 * g4 + 0] = fmaf(w.x, x[j + b], acc[j][4 * g4 + 0]);
            acc[j][4 * g4 + 1] = fmaf(w.y, x[j + b], acc[j][4 * g4 + 1]);
            acc[j][4 * g4 + 2] = fmaf(w.z, x[j + b], acc[j][4 * g4 + 2]);
            acc[j][4 * g4 + 3] = fmaf(w.w, x[j + b], acc[j][4 * g4 + 3]);
          }
        }
      }
    } else {
      for (int b = 0; b < l2; ++b) {
        float xv[PX];
#pragma unroll
        for (int j = 0; j < PX; ++j) xv[j] = row[j + b] - c;
        const float4* wp = reinterpret_cast<const float4*>(wsm + (a * l2 + b) * NF);
#pragma unroll
        for (int g4 = 0; g4 < NF / 4; ++g4) {
          const float4 w = wp[g4];
#pragma unroll
          for (int j = 0; j < PX; ++j) {
            acc[j][4 * g4 + 0] = fmaf(w.x, xv[j], acc[j][4 * g4 + 0]);
            acc[j][4 * g4 + 1] = fmaf(w.y, xv[j], acc[j][4 * g4 + 1]);
            acc[j][4 * g4 + 2] = fmaf(w.z, xv[j], acc[j][4 * g4 + 2]);
            acc[j][4 * g4 + 3] = fmaf(w.w, xv[j], acc[j][4 * g4 + 3]);
          }
        }
      }
    }
  }
  const int64_t plane = (int64_t)A.oh * A.ow;
  // full, aligned groups: vector stores (each warp writes contiguous rows per filter)
  if constexpr (PX % 4 == 0) {
    if (v0 + PX <= A.ow && (A.ow & 3) == 0) {
      if constexpr (MODE == 0) {
        float* o = static_cast<float*>(A.out) + (m * A.count) * plane + (int64_t)u * A.ow + v0;
#pragma unroll
        for (int g = 0; g < NF; ++g)
          if (g < A.count) {
#pragma unroll
            for (int j4 = 0; j4 < PX / 4; ++j4)
              *reinterpret_cast<float4*>(o + g * plane + 4 * j4) =
                  make_float4(acc[4 * j4][g], acc[4 * j4 + 1][g], acc[4 * j4 + 2][g], acc[4 * j4 + 3][g]);
          }
      } else if constexpr (MODE == 1) {
        uint32_t wds[PX / 4];
#pragma unroll
        for (int j4 = 0; j4 < PX / 4; ++j4) {
          uint32_t wv = 0;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            unsigned code = 0;
#pragma unroll
            for (int g = 0; g < NF; ++g)
              if (g < A.count && acc[4 * j4 + jj][g] > 0.f) code |= 1u << g;
            wv |= code << (8 * jj);
          }
          wds[j4] = wv;
        }
        uint8_t* o = static_cast<uint8_t*>(A.out) + m * plane + (int64_t)u * A.ow + v0;
        if constexpr (PX == 8)
          *reinterpret_cast<uint2*>(o) = make_uint2(wds[0], wds[1]);
        else
#pragma unroll
          for (int j4 = 0; j4 < PX / 4; ++j4) *reinterpret_cast<uint32_t*>(o + 4 * j4) = wds[j4];
      } else {
#pragma unroll
        for (int j4 = 0; j4 < PX / 4; ++j4) {
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            unsigned code = 0;
#pragma unroll
            for (int g = 0; g < NF; ++g)
              if (g < A.count && acc[4 * j4 + jj][g] > 0.f) code |= 1u << g;
            if (jj < 2) lo |= code << (16 * jj);
            else hi |= code << (16 * (jj - 2));
          }
          *reinterpret_cast<uint2*>(static_cast<uint16_t*>(A.out) + m * plane + (int64_t)u * A.ow + v0 + 4 * j4) =
              make_uint2(lo, hi);
        }
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < PX; ++j) {
    const int v = v0 + j;
    if (v >= A.ow) break;
    if constexpr (MODE == 0) {
      float* o = static_cast<float*>(A.out) + (m * A.count) * plane + (int64_t)u * A.ow + v;
#pragma unroll
      for (int g = 0; g < NF; ++g)
        if (g < A.count) o[g * plane] = acc[j][g];
    } else {
      unsigned code = 0;
#pragma unroll
      for (int g = 0; g < NF; ++g)
        if (g < A.count && acc[j][g] > 0.f) code |= 1u << g;
      if constexpr (MODE == 1)
        static_cast<uint8_t*>(A.out)[m * plane + (int64_t)u * A.ow + v] = (uint8_t)code;
      else
        static_cast<uint16_t*>(A.out)[m * plane + (int64_t)u * A.ow + v] = (uint16_t)code;
    }
  }
}


// Persistent, double-buffered: each block stages its filters once, then walks
// tiles (map, band of output rows) with the next tile's input rows in flight
// (cp.async, zero-filled padding) while the current one is computed.
template <int NF, int PX, int L2, int MODE>
__global__ void __launch_bounds__(CONV_THREADS) conv_s1_kernel(ConvArgs A, int max_rows) {
  extern __shared__ __align__(16) float smf[];
  const int l2 = L2 > 0 ? L2 : A.l2;
  const int d = A.l1 * l2;
  const int Wt = conv_tile_width(A.ow, l2, PX);
  float* wsm = smf;                                // [d][NF] zero-mean taps when centering
  float* bufs = wsm + d * NF;                      // 2 x [max_rows][Wt]
  const int buf_elems = max_rows * Wt;
  const int G = (A.ow + PX - 1) / PX;              // thread groups per output row
  const int64_t per_map = (int64_t)A.oh * G;
  const int blocks_per_map = (int)((per_map + CONV_THREADS - 1) / CONV_THREADS);
  const int64_t total = A.n_maps * blocks_per_map;
  __shared__ float wmean[NF];
  if (threadIdx.x < NF) {
    double s = 0.0;
    if (A.center && (int)threadIdx.x < A.count)
      for (int k = 0; k < d; ++k) s += (double)A.pack[k * A.count + threadIdx.x];
    wmean[threadIdx.x] = (float)(s / d);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d * NF; e += blockDim.x) {
    const int k = e / NF, g = e % NF;
    wsm[e] = g < A.count ? (float)((double)A.pack[k * A.count + g] - (double)wmean[g]) : 0.f;
  }
  auto band = [&](int64_t t, int& u_first, int& rows, int64_t& m, int64_t& i0) {
    m = t / blocks_per_map;
    i0 = (t % blocks_per_map) * (int64_t)CONV_THREADS;
    u_first = (int)(i0 / G);
    const int u_last = (int)((min(per_map, i0 + CONV_THREADS) - 1) / G);
    rows = u_last - u_first + A.l1;
  };
  auto issue = [&](int64_t t, float* buf) {
    int u_first, rows;
    int64_t m, i0;
    band(t, u_first, rows, m, i0);
    const float* img = A.in + m * (int64_t)A.p * A.q;
    for (int r = threadIdx.x >> 5; r < rows; r += CONV_THREADS / 32) {
      const int i = u_first + r - A.top;
      const bool rok = i >= 0 && i < A.p;
      for (int c = threadIdx.x & 31; c < Wt; c += 32) {
        const int j = c - A.left;
        const bool ok = rok && j >= 0 && j < A.q;
        cp_async4z(buf + r * Wt + c, ok ? img + (int64_t)i * A.q + j : A.in, ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  int64_t t = blockIdx.x;
  if (t < total) issue(t, bufs);
  for (int it = 0; t < total; t += gridDim.x, ++it) {
    float* cur = bufs + (it & 1) * buf_elems;
    if (t + gridDim.x < total)
      issue(t + gridDim.x, bufs + ((it + 1) & 1) * buf_elems);
    else
      asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    int u_first, rows;
    int64_t m, i0;
    band(t, u_first, rows, m, i0);
    const int64_t item = i0 + threadIdx.x;
    if (item < per_map) {
      const int u = (int)(item / G);
      const int v0 = (int)(item % G) * PX;
      conv_strip<NF, PX, L2, MODE>(A, wsm, cur, Wt, m, u, v0, u - u_first);
    }
    __syncthreads();
  }
}

// Generic path (any stride): one output pixel per thread, float32 centered dot.
template <int MODE>
__global__ void conv_generic_kernel(ConvArgs A, int stride) {
  const int64_t plane = (int64_t)A.oh * A.ow;
  const int d = A.l1 * A.l2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < A.n_maps * plane;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / plane;
    const int pos = (int)(e % plane);
    const int u = pos / A.ow, v = pos % A.ow;
    const float* img = A.in + m * (int64_t)A.p * A.q;
    float mean = 0.f;
    if (A.center) {
      float s = 0.f;
      for (int k = 0; k < d; ++k) {
        const int i = u * stride - A.top + k / A.l2, j = v * stride - A.left + k % A.l2;
        if (i >= 0 && i < A.p && j >= 0 && j < A.q) s += img[(int64_t)i * A.q + j];
      }
      mean = s / (float)d;
    }
    unsigned code = 0;
    for (int g = 0; g < A.count; ++g) {
      float r = 0.f;
      for (int k = 0; k < d; ++k) {
        const int i = u * stride - A.top + k / A.l2, j = v * stride - A.left + k % A.l2;
        float x = 0.f;
        if (i >= 0 && i < A.p && j >= 0 && j < A.q) x = img[(int64_t)i * A.q + j];
        r = fmaf(A.pack[k * A.count + g], x - mean, r);
      }
      if constexpr (MODE == 0)
        static_cast<float*>(A.out)[(m * A.count + g) * plane + pos] = r;
      else if (r > 0.f)
        code |= 1u << g;
    }
    if constexpr (MODE == 1) static_cast<uint8_t*>(A.out)[m * plane + pos] = (uint8_t)code;
    if constexpr (MODE == 2) static_cast<uint16_t*>(A.out)[m * plane + pos] = (uint16_t)code;
  }
}

// ---------------------------------------------------------------------------
// K8: block histograms, one warp per (group, block), packed u16 shared bins
// ---------------------------------------------------------------------------
struct HistArgs {
  const void* codes;
  int code_bytes;
  int64_t n_groups;
  int oh, ow, nbits, bh, bw, sh, sw, nby, nbx, kind;
  void* counts;
  int64_t gpr, row_stride, group_stride;
};

__global__ void block_hist_kernel(HistArgs H, int warps_per_block) {
  extern __shared__ unsigned int bins_sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbins = 1 << H.nbits;
  const int words = (nbins + 1) / 2;
  unsigned int* bins = bins_sm + (int64_t)warp * words;
  const int nblk = H.nby * H.nbx;
  const int64_t task = (int64_t)blockIdx.x * warps_per_block + warp;
  if (task >= H.n_groups * nblk) return;
  const int64_t grp = task / nblk;
  const int blk = (int)(task % nblk);
  const int by = blk / H.nbx, bx = blk % H.nbx;
  for (int w = lane; w < words; w += 32) bins[w] = 0u;
  __syncwarp();
  const int64_t plane = (int64_t)H.oh * H.ow;
  const int npx = H.bh * H.bw;
  for (int t = lane; t < npx; t += 32) {
    const int i = by * H.sh + t / H.bw, j = bx * H.sw + t % H.bw;
    const int64_t off = grp * plane + (int64_t)i * H.ow + j;
    const unsigned code = H.code_bytes == 1 ? static_cast<const uint8_t*>(H.codes)[off]
                                            : static_cast<const uint16_t*>(H.codes)[off];
    atomicAdd(&bins[code >> 1], 1u << ((code & 1u) * 16));
  }
  __syncwarp();
  const int64_t base = (grp / H.gpr) * H.row_stride + (grp % H.gpr) * H.group_stride + (int64_t)blk * nbins;
  for (int b = lane; b < nbins; b += 32) {
    const unsigned cnt = (bins[b >> 1] >> ((b & 1) * 16)) & 0xffffu;
    if (H.kind == 2)
      static_cast<uint16_t*>(H.counts)[base + b] = (uint16_t)cnt;
    else
      static_cast<uint8_t*>(H.counts)[base + b] = (uint8_t)(cnt > 255u ? 255u : cnt);
  }
}

// counts -> float64 features via LUT; one warp per block histogram
__global__ void iq_expand_kernel(const void* counts, int kind, int64_t n_blocks, int nbins, int bpc,
                                 const double* __restrict__ lut, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t blk = warp; blk < n_blocks; blk += nw) {
    const int64_t base = blk * nbins;
    int extra = 0;
    if (kind == 1) {
      int s = 0;
      for (int b = lane; b < nbins; b += 32) s += static_cast<const uint8_t*>(counts)[base + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      extra = bpc - s;
    }
    for (int b = lane; b < nbins; b += 32) {
      int c = kind == 2 ? static_cast<const uint16_t*>(counts)[base + b] : static_cast<const uint8_t*>(counts)[base + b];
      if (kind == 1 && c == 255) c += extra;
      out[base + b] = lut[c];
    }
  }
}

__global__ void sign_hash_kernel(const float* maps, int64_t n_groups, int nbits, int64_t plane, void* codes) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_groups * plane;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = e / plane, pix = e % plane;
    const float* src = maps + g * nbits * plane + pix;
    unsigned code = 0;
    for (int b = 0; b < nbits; ++b)
      if (src[b * plane] > 0.f) code |= 1u << b;
    if (nbits <= 8)
      static_cast<uint8_t*>(codes)[e] = (uint8_t)code;
    else
      static_cast<uint16_t*>(codes)[e] = (uint16_t)code;
  }
}

// explicit patch matrix (extract_patch_stack): float64 in, float64 out (d x cols)
__global__ void im2col_kernel(const double* maps, int64_t n_maps, Geo g, int center, double* out) {
  const int64_t cpm = (int64_t)g.oh * g.ow;
  const int64_t cols = n_maps * cpm;
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < cols; col += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = col / cpm;
    const int pos = (int)(col % cpm);
    const int u = pos / g.ow, v = pos % g.ow;
    const double* img = maps + m * (int64_t)g.p * g.q;
    double mean = 0.0;
    if (center) {
      double s = 0.0;
      for (int k = 0; k < g.d; ++k) {
        const int i = u * g.stride - g.top + k / g.l2, j = v * g.stride - g.left + k % g.l2;
        if (i >= 0 && i < g.p && j >= 0 && j < g.q) s += img[(int64_t)i * g.q + j];
      }
      mean = s / g.d;
    }
    for (int k = 0; k < g.d; ++k) {
      const int i = u * g.stride - g.top + k / g.l2, j = v * g.stride - g.left + k % g.l2;
      double x = 0.0;
      if (i >= 0 && i < g.p && j >= 0 && j < g.q) x = img[(int64_t)i * g.q + j];
      out[(int64_t)k * cols + col] = x - mean;
    }
  }
}

template <int NF, int PX, int MODE>
static int launch_s1(const ConvArgs& A, cudaStream_t st) {
  const int l2 = A.l2;
  const int G = (A.ow + PX - 1) / PX;
  const int64_t per_map = (int64_t)A.oh * G;
  const int bpm = (int)((per_map + CONV_THREADS - 1) / CONV_THREADS);
  const int max_rows = (CONV_THREADS + G - 1) / G + 1 + A.l1;
  const size_t smem =
      sizeof(float) * ((size_t)A.l1 * l2 * NF + 2 * (size_t)max_rows * conv_tile_width(A.ow, l2, PX));
  const int64_t tiles = (int64_t)bpm * A.n_maps;
  if (smem > 200 * 1024) return fail(DDCCA_ECONFIG, "conv: map row too wide for shared-memory staging");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CONV_THREADS, smem);
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)std::max(1, per_sm) * sms);
    kern<<<(unsigned)grid, CONV_THREADS, smem, st>>>(A, max_rows);
  };
  switch (l2) {
    case 3: go(conv_s1_kernel<NF, PX, 3, MODE>); break;
    case 5: go(conv_s1_kernel<NF, PX, 5, MODE>); break;
    case 7: go(conv_s1_kernel<NF, PX, 7, MODE>); break;
    case 9: go(conv_s1_kernel<NF, PX, 9, MODE>); break;
    default: go(conv_s1_kernel<NF, PX, 0, MODE>);
  }
  return check_launch("conv_s1_kernel");
}

template <int MODE>
static int launch_conv(const ConvArgs& A, int stride, cudaStream_t st) {
  if (A.n_maps == 0) return DDCCA_OK;
  if (stride == 1) {
    if (A.count <= 8) return launch_s1<8, 8, MODE>(A, st);
    if (A.count <= 16) return launch_s1<16, 4, MODE>(A, st);
    if (A.count <= 32) return launch_s1<32, 2, MODE>(A, st);
    if (A.count <= 64 && MODE == 0) return launch_s1<64, 1, MODE>(A, st);
  }
  const int64_t total = A.n_maps * (int64_t)A.oh * A.ow;
  const int blocks = (int)std::min<int64_t>(148 * 64, (total + 255) / 256);
  conv_generic_kernel<MODE><<<blocks, 256, 0, st>>>(A, stride);
  return check_launch("conv_generic_kernel");
}

static int conv_args(const float* in, int64_t n_maps, const ddcca_geom* gg, const float* pack, int count, int center,
                     void* out, ConvArgs* A, int* stride) {
  Geo g{};
  DDCCA_TRY(make_geo(gg, &g));
  if (count < 1 || count > g.d) return fail(DDCCA_ECONFIG, "filter count %d outside [1, %d]", count, g.d);
  if (n_maps < 0) return fail(DDCCA_ESHAPE, "negative map count");
  if (n_maps > 0 && (!in || !pack || !out)) return fail(DDCCA_ESHAPE, "null pointer");
  A->in = in; A->n_maps = n_maps; A->p = g.p; A->q = g.q; A->l1 = g.l1; A->l2 = g.l2; A->top = g.top;
  A->left = g.left; A->oh = g.oh; A->ow = g.ow; A->count = count; A->center = center; A->pack = pack; A->out = out;
  *stride = g.stride;
  return DDCCA_OK;
}

}  // namespace ddcca

using namespace ddcca;

extern "C" {

int ddcca_conv(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack, int count, int center,
               float* out, void* stream) {
  ConvArgs A;
  int stride = 1;
  DDCCA_TRY(conv_args(in, n_maps, g, conv_pack, count, center, out, &A, &stride));
  if (count > 64) return fail(DDCCA_ECONFIG, "conv: at most 64 filters per layer on device");
  return launch_conv<0>(A, stride, as_stream(stream));
}

int ddcca_conv_hash(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack, int count,
                    int center, void* codes, void* stream) {
  ConvArgs A;
  int stride = 1;
  DDCCA_TRY(conv_args(in, n_maps, g, conv_pack, count, center, codes, &A, &stride));
  if (count > 16) return fail(DDCCA_ECONFIG, "hash width %d above the device limit of 16 bits", count);
  if (count <= 8) return launch_conv<1>(A, stride, as_stream(stream));
  return launch_conv<2>(A, stride, as_stream(stream));
}

int ddcca_block_hist(const void* codes, int code_bytes, int64_t n_groups, int oh, int ow, int n_bits, int block_h,
                     int block_w, int step_h, int step_w, void* counts, int count_kind, int64_t groups_per_row,
                     int64_t row_stride, int64_t group_stride, void* stream) {
  if (n_bits < 1 || n_bits > 16) return fail(DDCCA_ECONFIG, "can histogram 1..16 bit codes, got %d", n_bits);
  if (block_h < 1 || block_w < 1 || step_h < 1 || step_w < 1) return fail(DDCCA_ECONFIG, "bad block geometry");
  if (oh < block_h || ow < block_w)
    return fail(DDCCA_ESHAPE, "%dx%d blocks do not fit a %dx%d map", block_h, block_w, oh, ow);
  if (code_bytes != 1 && code_bytes != 2) return fail(DDCCA_ECONFIG, "code width must be 1 or 2 bytes");
  const int bpc = block_h * block_w;
  if (count_kind == 0 && bpc > 255) return fail(DDCCA_ECONFIG, "u8 counts need bpc <= 255");
  if (count_kind == 1 && bpc > 510) return fail(DDCCA_ECONFIG, "saturating u8 counts need bpc <= 510");
  if (bpc > 65535) return fail(DDCCA_ECONFIG, "block of %d pixels too large", bpc);
  if (n_groups == 0) return DDCCA_OK;
  HistArgs H;
  H.codes = codes; H.code_bytes = code_bytes; H.n_groups = n_groups; H.oh = oh; H.ow = ow; H.nbits = n_bits;
  H.bh = block_h; H.bw = block_w; H.sh = step_h; H.sw = step_w;
  H.nby = (oh - block_h) / step_h + 1;
  H.nbx = (ow - block_w) / step_w + 1;
  H.kind = count_kind; H.counts = counts; H.gpr = groups_per_row; H.row_stride = row_stride; H.group_stride = group_stride;
  const size_t words = ((size_t)(1 << n_bits) + 1) / 2;
  int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / (words * 4)));
  const size_t smem = words * 4 * wpb;
  const int64_t tasks = n_groups * H.nby * H.nbx;
  const int64_t blocks = (tasks + wpb - 1) / wpb;
  if (blocks > 0x7fffffffLL) return fail(DDCCA_ECONFIG, "histogram: too many blocks");
  cudaFuncSetAttribute(block_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  block_hist_kernel<<<(unsigned)blocks, 32 * wpb, smem, as_stream(stream)>>>(H, wpb);
  return check_launch("block_hist_kernel");
}

int ddcca_iq_expand(const void* counts, int count_kind, int64_t n_blocks, int n_bits, int bpc, const double* lut,
                    double* out, void* stream) {
  if (n_bits < 1 || n_bits > 16) return fail(DDCCA_ECONFIG, "bad bit width %d", n_bits);
  if (n_blocks == 0) return DDCCA_OK;
  const int blocks = (int)std::min<int64_t>(148 * 16, (n_blocks * 32 + 255) / 256);
  iq_expand_kernel<<<blocks, 256, 0, as_stream(stream)>>>(counts, count_kind, n_blocks, 1 << n_bits, bpc, lut, out);
  return check_launch("iq_expand_kernel");
}

int ddcca_sign_hash(const float* maps, int64_t n_groups, int n_bits, int64_t plane, void* codes, void* stream) {
  if (n_bits < 1 || n_bits > 16) return fail(DDCCA_ECONFIG, "can hash 1..16 bit maps on device, got %d", n_bits);
  const int64_t total = n_groups * plane;
  if (total == 0) return DDCCA_OK;
  const int blocks = (int)std::min<int64_t>(148 * 32, (total + 255) / 256);
  sign_hash_kernel<<<blocks, 256, 0, as_stream(stream)>>>(maps, n_groups, n_bits, plane, codes);
  return check_launch("sign_hash_kernel");
}

int ddcca_im2col(const double* maps, int64_t n_maps, const ddcca_geom* gg, int center, double* out, void* stream) {
  Geo g{};
  DDCCA_TRY(make_geo(gg, &g));
  const int64_t cols = n_maps * (int64_t)g.oh * g.ow;
  if (cols == 0) return DDCCA_OK;
  const int blocks = (int)std::min<int64_t>(148 * 32, (cols + 255) / 256);
  im2col_kernel<<<blocks, 256, 0, as_stream(stream)>>>(maps, n_maps, g, center, out);
  return check_launch("im2col_kernel");
}

}  // extern "C"
