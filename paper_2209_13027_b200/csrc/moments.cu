// K1+K2+K3: per-batch DDCCA moments from image maps, without materializing
// patches.
//
// Reference semantics (cascade.py:155-189, patches.py:97-125,
// moments.py:86-110): for every batch of samples, every stride-1 window of
// every map yields a patch x (d = l1*l2, zero padding counted), centered by
// its own mean when `center`; C11 += x x^T (view 1), C22 += y y^T (view 2),
// class / global column sums, counts.
//
// B200 formulation. For stride 1 the raw Gram is a windowed
// autocorrelation of the padded map P (Hp x Wp):
//   Craw[(a,b),(a+dy,b+dx)] = sum_{y in [a,a+oh), x in [b,b+ow)} P[y,x] P[y+dy,x+dx]
// and centering is the exact projection C = H Craw H, H = I - 11^T/d
// (H kills constants, patch by patch). Each first pixel (y,x) contributes to
// a rectangle of (a,b) that depends only on its row zone / column zone (the
// runs of rows/cols with equal a-range / b-range). So per batch we only need,
// for every lag (dy,dx) and every (row zone, col zone), the sum of
// P[y,x] P[y+dy,x+dx] over that zone: l1*(2*l2-1) lags x ~(2l1-1)(2l2-1)
// zones, instead of d^2/2 products per patch. float32 inputs make every
// product exact in float64; sums are float64, so the result matches the
// reference's float64 Gram to ~1e-15 relative before centering.
//
// Kernels:
//   lag_zone_kernel   one block per (task, split, batch, view): a task is a
//                     row range of one row zone x a 32-column tile; the block
//                     loops over its maps, keeps per-thread float64
//                     accumulators (l1 x KDX lags) and writes one record per
//                     (task, column zone present in the tile).
//   zone_reduce       records -> Z[batch][view][rz][cz][lag] (fixed order).
//   assemble          Z -> Craw -> H Craw H -> payload c11/c22.
//   rect_sums         per-map window sums (class-sum path), centered.
//   batch_epilogue    per-batch class sums / global sums / counts.
//   direct_*          explicit-patch float64 path for stride != 1.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace ddcca {

constexpr int KDX = 3;       // dx lags per thread
constexpr int TILE_X = 32;   // first-pixel columns per block (one per lane)
constexpr bool LAG_F32 = true;  // float32 tiles, convert in the ring (halves shared-memory traffic)
constexpr int STAGE_ROWS = 96;  // staged rows per cp.async stage (all maps of the stage)
constexpr int SLAB_ROWS = 48;   // staged rows of one interior task (slab + halo)
constexpr int MAPS_PER_SPLIT = 128;
constexpr int MAX_LAG_L = 12;  // lag path for windows up to 12 x 12

struct Zones {
  // zone index of each padded row / column and each zone's a-/b-range
  std::vector<int> rz_of_y, cz_of_x;
  std::vector<int> rz_lo, rz_hi, cz_lo, cz_hi;
  int big_cz = -1;  // column zone with >= 2 columns (the interior), or -1
};

static void make_zones(int n, int out, int l, std::vector<int>& zone_of, std::vector<int>& lo,
                       std::vector<int>& hi) {
  zone_of.assign(n, 0);
  lo.clear();
  hi.clear();
  int prev_lo = -1, prev_hi = -1;
  for (int y = 0; y < n; ++y) {
    int a_lo = std::max(0, y - out + 1), a_hi = std::min(y, l - 1);
    if (a_lo != prev_lo || a_hi != prev_hi) {
      lo.push_back(a_lo);
      hi.push_back(a_hi);
      prev_lo = a_lo;
      prev_hi = a_hi;
    }
    zone_of[y] = (int)lo.size() - 1;
  }
}

struct Task {
  int y0, y1, x0, rz;
  int rec0;     // first record index of this task within a (batch, split)
  int nrec;     // records written: [big zone if present] + singleton columns
};

// A record: sum over one task's rows and over the lanes of one column zone.
struct RecInfo {
  int rz, cz;
};

struct Plan {
  Geo g{};
  Zones z;
  int nrz, ncz, G, NDX, NDF, slab;
  std::vector<Task> tasks;
  std::vector<RecInfo> recs;
  std::vector<int> lane_slot;  // per task * 32 + lane -> record offset within task, or -1 (big zone)
  int nrec;
};

static void make_plan(const Geo& g, Plan* P) {
  P->g = g;
  make_zones(g.Hp, g.oh, g.l1, P->z.rz_of_y, P->z.rz_lo, P->z.rz_hi);
  make_zones(g.Wp, g.ow, g.l2, P->z.cz_of_x, P->z.cz_lo, P->z.cz_hi);
  P->nrz = (int)P->z.rz_lo.size();
  P->ncz = (int)P->z.cz_lo.size();
  // column zone with the most columns becomes the warp-reduced "big" zone
  std::vector<int> ccount(P->ncz, 0);
  for (int x = 0; x < g.Wp; ++x) ccount[P->z.cz_of_x[x]]++;
  int best = -1, bestn = 1;
  for (int c = 0; c < P->ncz; ++c)
    if (ccount[c] > bestn) { bestn = ccount[c]; best = c; }
  P->z.big_cz = best;
  P->G = (2 * g.l2 - 1 + KDX - 1) / KDX;
  P->NDX = P->G * KDX;
  P->NDF = g.l1 * P->NDX;
  // one stage stages at most PF_ROWS rows per warp: slab + halo must fit
  P->slab = g.l1 * std::max(1, (SLAB_ROWS - g.l1 + 1) / g.l1);  // whole ring turns
  P->tasks.clear();
  P->recs.clear();
  P->lane_slot.clear();
  int nrec = 0;
  // First pixels outside the image are zero padding: their products vanish, so
  // tasks cover only image rows [top, top+p) and image columns [left, left+q).
  const int yimg_end = g.top + g.p, ximg_end = g.left + g.q;
  int y = g.top;
  while (y < yimg_end) {
    int rz = P->z.rz_of_y[y];
    int y_end = y;
    while (y_end < yimg_end && P->z.rz_of_y[y_end] == rz) ++y_end;
    for (int ys = y; ys < y_end; ys += P->slab) {
      int ye = std::min(y_end, ys + P->slab);
      for (int x0 = g.left; x0 < ximg_end; x0 += TILE_X) {
        Task t;
        t.y0 = ys; t.y1 = ye; t.x0 = x0; t.rz = rz; t.rec0 = nrec; t.nrec = 0;
        bool has_big = false;
        for (int l = 0; l < TILE_X; ++l) {
          int x = x0 + l;
          if (x < ximg_end && P->z.cz_of_x[x] == P->z.big_cz) has_big = true;
        }
        if (has_big) {
          P->recs.push_back({rz, P->z.big_cz});
          t.nrec++;
        }
        for (int l = 0; l < TILE_X; ++l) {
          int x = x0 + l;
          if (x < ximg_end && P->z.cz_of_x[x] != P->z.big_cz) {
            P->lane_slot.push_back(t.nrec);
            P->recs.push_back({rz, P->z.cz_of_x[x]});
            t.nrec++;
          } else {
            P->lane_slot.push_back(-1);
          }
        }
        nrec += t.nrec;
        P->tasks.push_back(t);
      }
    }
    y = y_end;
  }
  P->nrec = nrec;
}

// ----------------------------------------------------------------------------
// lag_zone_kernel
// ----------------------------------------------------------------------------
struct TaskDev {
  int y0, y1, x0, rec0, mb;  // rows [y0, y1), tile column x0, first record, maps per stage
};

struct LagArgs {
  const float* maps[2];
  const TaskDev* tasks;
  const int* lane_slot;     // [task][32]
  const int64_t* batch_off; // device copy of batch map offsets
  double* rec;              // [batch][view][split][nrec][NDF]
  int p, q, top, left, Wp, l2, G, NDX, NDF, nrec, nsplit, nbatch, xend;
  int64_t per_split;        // maps per split: split s of a batch owns its maps [s*per, (s+1)*per)
};

// Sum over rows [0, nrows) of one staged map tile (float64, row stride tc) of
// own * partner for the L1 x KDX lags of this thread. Rows are processed in
// whole ring turns of L1; rows >= nrows are masked through the own value
// (their staged data is still valid partner data for earlier rows). TC > 0
// makes the tile stride a compile-time constant (all smem offsets immediate).
template <int L1, int TC, bool SKIP0, int KK, typename S>
__device__ __forceinline__ void lag_accumulate(const S* __restrict__ t, int tc_rt, int nrows, int cown,
                                               int cpart, double (&acc)[L1][KDX]) {
  const int tc = TC > 0 ? TC : tc_rt;
  double ring[L1][KK];
  const S* pp = t + cpart;
#pragma unroll
  for (int q = 0; q < L1 - 1; ++q)
#pragma unroll
    for (int k = 0; k < KK; ++k) ring[q][k] = (double)pp[q * tc + k];
  pp += (L1 - 1) * tc;
  const S* po = t + cown;
  for (int r0 = 0; r0 < nrows; r0 += L1) {
#pragma unroll
    for (int u = 0; u < L1; ++u) {
      const int snew = (u + L1 - 1) % L1;
#pragma unroll
      for (int k = 0; k < KK; ++k) ring[snew][k] = (double)pp[u * tc + k];
      double own = (double)po[u * tc];
      own = (r0 + u < nrows) ? own : 0.0;
#pragma unroll
      for (int dy = SKIP0 ? 1 : 0; dy < L1; ++dy)
#pragma unroll
        for (int k = 0; k < KK; ++k) acc[dy][k] = fma(own, ring[(u + dy) % L1][k], acc[dy][k]);
    }
    pp += L1 * tc;
    po += L1 * tc;
  }
}

// Tasks shorter than one ring turn (the single border rows): direct partner loads.
template <int L1, int TC, int KK, typename S>
__device__ __forceinline__ void lag_accumulate_short(const S* __restrict__ t, int tc_rt, int nrows, int cown,
                                                     int cpart, bool skip0, double (&acc)[L1][KDX]) {
  const int tc = TC > 0 ? TC : tc_rt;
  for (int r = 0; r < nrows; ++r) {
    const double own = (double)t[r * tc + cown];
    const S* pp = t + r * tc + cpart;
#pragma unroll
    for (int dy = 0; dy < L1; ++dy) {
      if (dy == 0 && skip0) continue;
#pragma unroll
      for (int k = 0; k < KK; ++k) acc[dy][k] = fma(own, (double)pp[dy * tc + k], acc[dy][k]);
    }
  }
}

// One staged map tile through this warp's lag group. kk = live dx lags of the group
// (the last group of 2*l2-1 lags may be partial: its padding lags are not computed).
template <int L1, int TC, typename S>
__device__ __forceinline__ void lag_map(const S* __restrict__ t, int tc, int nrows, int cown, int cpart,
                                        bool short_task, bool skip0, int kk, double (&acc)[L1][KDX]) {
  static_assert(KDX == 3, "lag_map dispatches 1..3 live lags");
  if (short_task) {
    if (kk >= 3) lag_accumulate_short<L1, TC, 3>(t, tc, nrows, cown, cpart, skip0, acc);
    else if (kk == 2) lag_accumulate_short<L1, TC, 2>(t, tc, nrows, cown, cpart, skip0, acc);
    else lag_accumulate_short<L1, TC, 1>(t, tc, nrows, cown, cpart, skip0, acc);
  } else if (skip0) {
    lag_accumulate<L1, TC, true, 3>(t, tc, nrows, cown, cpart, acc);
  } else if (kk >= 3) {
    lag_accumulate<L1, TC, false, 3>(t, tc, nrows, cown, cpart, acc);
  } else if (kk == 2) {
    lag_accumulate<L1, TC, false, 2>(t, tc, nrows, cown, cpart, acc);
  } else {
    lag_accumulate<L1, TC, false, 1>(t, tc, nrows, cown, cpart, acc);
  }
}

// Blocked float32 form (layers whose inputs are filter responses): the products of one
// stage's maps accumulate in float32 (at most mb maps of one slab: <= STAGE_ROWS terms per
// lag) and the stage partial is added to the float64 accumulator. Used only when the caller
// asks for it (DDCCA_MOMENTS_F32_BLOCKS); float64 products are exact, these are not.
// Lags k = 0, 1 run as packed fma.rn.f32x2 (the same per-lane rounding as two fmaf, half the
// issue slots), k = 2 scalar; fa2 holds lags (0, 1), fa1 the scalar lag (k = 2 of three,
// or k = 0 when the group has a single live lag).
template <int L1>
struct F32Partials {
  float2 fa2[L1];
  float fa1[L1];
};

template <int L1, int TC, bool SKIP0, int KK>
__device__ __forceinline__ void lag_accumulate_f32(const float* __restrict__ t, int nrows, int cown, int cpart,
                                                   F32Partials<L1>& f) {
  constexpr bool P2 = KK >= 2;
  constexpr bool S1 = KK != 2;  // a scalar lag: k = 2 of three, or the only one
  constexpr int ks = P2 ? 2 : 0;
  float2 ring2[L1];
  float ring1[L1];
  const float* pp = t + cpart;
#pragma unroll
  for (int q = 0; q < L1 - 1; ++q) {
    if constexpr (P2) ring2[q] = make_float2(pp[q * TC], pp[q * TC + 1]);
    if constexpr (S1) ring1[q] = pp[q * TC + ks];
  }
  pp += (L1 - 1) * TC;
  const float* po = t + cown;
  for (int r0 = 0; r0 < nrows; r0 += L1) {
#pragma unroll
    for (int u = 0; u < L1; ++u) {
      const int snew = (u + L1 - 1) % L1;
      if constexpr (P2) ring2[snew] = make_float2(pp[u * TC], pp[u * TC + 1]);
      if constexpr (S1) ring1[snew] = pp[u * TC + ks];
      float own = po[u * TC];
      own = (r0 + u < nrows) ? own : 0.f;
      const float2 own2 = make_float2(own, own);
#pragma unroll
      for (int dy = SKIP0 ? 1 : 0; dy < L1; ++dy) {
        if constexpr (P2) f.fa2[dy] = __ffma2_rn(own2, ring2[(u + dy) % L1], f.fa2[dy]);
        if constexpr (S1) f.fa1[dy] = fmaf(own, ring1[(u + dy) % L1], f.fa1[dy]);
      }
    }
    pp += L1 * TC;
    po += L1 * TC;
  }
}

// Short tasks (single border rows) in the blocked form: direct partner loads.
template <int L1, int TC, int KK>
__device__ __forceinline__ void lag_accumulate_short_f32(const float* __restrict__ t, int nrows, int cown,
                                                         int cpart, bool skip0, F32Partials<L1>& f) {
  constexpr bool P2 = KK >= 2;
  constexpr bool S1 = KK != 2;
  constexpr int ks = P2 ? 2 : 0;
  for (int r = 0; r < nrows; ++r) {
    const float own = t[r * TC + cown];
    const float2 own2 = make_float2(own, own);
    const float* pp = t + r * TC + cpart;
#pragma unroll
    for (int dy = 0; dy < L1; ++dy) {
      if (dy == 0 && skip0) continue;
      if constexpr (P2) f.fa2[dy] = __ffma2_rn(own2, make_float2(pp[dy * TC], pp[dy * TC + 1]), f.fa2[dy]);
      if constexpr (S1) f.fa1[dy] = fmaf(own, pp[dy * TC + ks], f.fa1[dy]);
    }
  }
}

template <int L1>
__device__ __forceinline__ void f32_zero(F32Partials<L1>& f) {
#pragma unroll
  for (int dy = 0; dy < L1; ++dy) {
    f.fa2[dy] = make_float2(0.f, 0.f);
    f.fa1[dy] = 0.f;
  }
}

// Add the float32 stage partials to the float64 accumulator (and restart them).
template <int L1>
__device__ __forceinline__ void f32_flush(F32Partials<L1>& f, int kk, double (&acc)[L1][KDX]) {
  // static lag indices on every branch: a runtime index into acc would move it to local memory
#pragma unroll
  for (int dy = 0; dy < L1; ++dy) {
    if (kk >= 2) {
      acc[dy][0] += (double)f.fa2[dy].x;
      acc[dy][1] += (double)f.fa2[dy].y;
      if (kk >= 3) acc[dy][2] += (double)f.fa1[dy];
    } else {
      acc[dy][0] += (double)f.fa1[dy];
    }
  }
  f32_zero(f);
}

template <int L1, int TC>
__device__ __forceinline__ void lag_map_f32(const float* __restrict__ t, int nrows, int cown, int cpart,
                                            bool short_task, bool skip0, int kk, F32Partials<L1>& f) {
  if (short_task) {
    if (kk >= 3) lag_accumulate_short_f32<L1, TC, 3>(t, nrows, cown, cpart, skip0, f);
    else if (kk == 2) lag_accumulate_short_f32<L1, TC, 2>(t, nrows, cown, cpart, skip0, f);
    else lag_accumulate_short_f32<L1, TC, 1>(t, nrows, cown, cpart, skip0, f);
  } else if (skip0) {
    lag_accumulate_f32<L1, TC, true, 3>(t, nrows, cown, cpart, f);
  } else if (kk >= 3) {
    lag_accumulate_f32<L1, TC, false, 3>(t, nrows, cown, cpart, f);
  } else if (kk == 2) {
    lag_accumulate_f32<L1, TC, false, 2>(t, nrows, cown, cpart, f);
  } else {
    lag_accumulate_f32<L1, TC, false, 1>(t, nrows, cown, cpart, f);
  }
}

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 4 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(n));
}

// One block = one task (row range x 32-column tile) of one (batch, view, split);
// it walks the split's maps in stages of mb maps. Staging: cp.async float32 copies
// into a per-thread-owned raw buffer (double buffered), each thread converts its
// own elements to float64 into the (double-buffered) compute tile, then a single
// __syncthreads per stage publishes it.
template <int L1, int TC, bool F32>
__global__ void __launch_bounds__(256, (L1 <= 9 ? 2 : 1)) lag_zone_kernel(LagArgs A) {
  extern __shared__ __align__(16) double smem_d[];
  const int task = blockIdx.x;
  const int split = blockIdx.y;
  const int bv = blockIdx.z;  // batch * 2 + view
  const int batch = bv >> 1, view = bv & 1;
  const TaskDev T = A.tasks[task];
  const int lane = threadIdx.x & 31;
  const int grp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int nrows = T.y1 - T.y0;
  const bool short_task = nrows < L1;
  const int nrows_pad = short_task ? nrows : (nrows + L1 - 1) / L1 * L1;
  const int tr = nrows_pad + L1 - 1;                   // staged rows per map (zero beyond the map)
  const int tc = TC > 0 ? TC : TILE_X + A.NDX - 1;     // staged cols: [x0-(l2-1), x0-(l2-1)+tc), tc <= 64
  const int tile_elems = tr * tc;
  const int mb = T.mb;
  const int stage_rows = mb * tr;
  const int stage_elems = stage_rows * tc;
  // F32: three float32 stages, the ring converts on load. Else: two float32 cp.async
  // stages converted by their owners into two float64 compute tiles.
  double* f64 = smem_d;                                                                   // 2 x stage (float64)
  float* raw = F32 ? reinterpret_cast<float*>(smem_d) : reinterpret_cast<float*>(smem_d + 2 * stage_elems);
  const int xs = T.x0 - (A.l2 - 1);
  const int64_t m_begin = A.batch_off[batch];
  const int64_t m_end = A.batch_off[batch + 1];
  const int64_t per = A.per_split;
  const int64_t ma = m_begin + (int64_t)split * per;
  const int64_t mbnd = min(m_end, ma + per);
  const float* src = view == 0 ? A.maps[0] : A.maps[1];
  const int64_t plane = (int64_t)A.p * A.q;
  // this thread's two staging columns
  const int c0 = lane, c1 = lane + 32;
  const int col0 = xs + c0 - A.left, col1 = xs + c1 - A.left;
  const bool cok0 = col0 >= 0 && col0 < A.q;
  const bool cok1 = c1 < tc && col1 >= 0 && col1 < A.q;
  const bool has1 = c1 < tc;

  // staged flat rows fr = j * tr + r owned by warp fr % nwarps (no division: (j, r) advance incrementally)
  auto issue = [&](int64_t ms, float* dst) {
    int j = 0, r = grp;
    while (r >= tr) { r -= tr; ++j; }
    for (int fr = grp; fr < stage_rows; fr += nwarps) {
      const int img_row = T.y0 + r - A.top;
      const bool rok = img_row >= 0 && img_row < A.p && (r < nrows + L1 - 1) && (ms + j < mbnd);
      const float* rowp = src + (ms + j) * plane + (int64_t)img_row * A.q;
      cp_async4(dst + fr * tc + c0, (rok && cok0) ? rowp + col0 : src, rok && cok0);
      if (has1) cp_async4(dst + fr * tc + c1, (rok && cok1) ? rowp + col1 : src, rok && cok1);
      r += nwarps;
      while (r >= tr) { r -= tr; ++j; }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  auto convert = [&](const float* from, double* to) {
    for (int fr = grp; fr < stage_rows; fr += nwarps) {
      to[fr * tc + c0] = (double)from[fr * tc + c0];
      if (has1) to[fr * tc + c1] = (double)from[fr * tc + c1];
    }
  };

  double acc[L1][KDX];
#pragma unroll
  for (int dy = 0; dy < L1; ++dy)
#pragma unroll
    for (int k = 0; k < KDX; ++k) acc[dy][k] = 0.0;

  const int cown = lane + (A.l2 - 1);  // own column inside the tile
  const int cpart = lane + grp * KDX;  // partner column of k = 0
  // groups whose dx are all negative skip the dy = 0 lag (canonical half-plane only)
  const bool skip0 = (grp * KDX + KDX - 1) < (A.l2 - 1);
  const int kk = min(KDX, 2 * A.l2 - 1 - grp * KDX);  // live lags of this group

  if constexpr (F32) {
    if (ma < mbnd) issue(ma, raw); else asm volatile("cp.async.commit_group;\n" ::);
    if (ma + mb < mbnd) issue(ma + mb, raw + stage_elems); else asm volatile("cp.async.commit_group;\n" ::);
    int s = 0;
    for (int64_t ms = ma; ms < mbnd; ms += mb, ++s) {
      asm volatile("cp.async.wait_group 1;\n" ::);
      __syncthreads();  // stage s visible; everybody finished stage s-1 (its buffer is reused below)
      if (ms + 2 * mb < mbnd)
        issue(ms + 2 * mb, raw + ((s + 2) % 3) * stage_elems);
      else
        asm volatile("cp.async.commit_group;\n" ::);
      const float* tile = raw + (s % 3) * stage_elems;
      const int nm = (int)min((int64_t)mb, mbnd - ms);
      for (int j = 0; j < nm; ++j) {
        const float* t = tile + j * tile_elems;
        lag_map<L1, TC>(t, tc, nrows, cown, cpart, short_task, skip0, kk, acc);
      }
    }
  } else {
  if (ma < mbnd) issue(ma, raw);
  int s = 0;
  for (int64_t ms = ma; ms < mbnd; ms += mb, ++s) {
    if (ms + mb < mbnd)
      issue(ms + mb, raw + ((s + 1) & 1) * stage_elems);
    else
      asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    double* tile = f64 + (s & 1) * stage_elems;
    convert(raw + (s & 1) * stage_elems, tile);  // own elements only: no barrier needed before
    __syncthreads();
    const int nm = (int)min((int64_t)mb, mbnd - ms);
    for (int j = 0; j < nm; ++j) {
      const double* t = tile + j * tile_elems;
      lag_map<L1, TC>(t, tc, nrows, cown, cpart, short_task, skip0, kk, acc);
    }
  }
  }
  const int slot = A.lane_slot[task * TILE_X + lane];
  const int x = T.x0 + lane;
  const bool in_big = (slot < 0) && (x < A.xend);
  double* out = A.rec + (((int64_t)batch * 2 + view) * A.nsplit + split) * (int64_t)A.nrec * A.NDF;
  const int any_big = __any_sync(0xffffffffu, in_big);
#pragma unroll
  for (int dy = 0; dy < L1; ++dy)
#pragma unroll
    for (int k = 0; k < KDX; ++k) {
      const int lag = dy * A.NDX + grp * KDX + k;
      double v = in_big ? acc[dy][k] : 0.0;
      v = warp_sum(v);
      if (lane == 0 && any_big) out[(int64_t)T.rec0 * A.NDF + lag] = v;
      if (slot >= 0) out[(int64_t)(T.rec0 + slot) * A.NDF + lag] = acc[dy][k];
    }
}

// ----------------------------------------------------------------------------
// TMA + mbarrier pipeline variant (maps with q % 4 == 0): one elected producer
// thread streams whole stages (mb maps x tr rows x TCB columns, zero-filled
// out of bounds = the zero padding) with a single cp.async.bulk.tensor per
// stage into an NS-deep ring; consumer warps wait on the stage's "full"
// mbarrier and release it through its "empty" mbarrier. No __syncthreads and
// no per-element staging instructions in the steady state.
// ----------------------------------------------------------------------------
constexpr int TMA_NS = 3;  // default ring depth (DDCCA_TMA_STAGES overrides, 2..8)

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

struct TmaBoxes {
  int rows_int, mb_int;      // interior tasks (nrows >= L1)
  int rows_short, mb_short;  // short (single border row) tasks
  int shift;                 // columns the tile starts early so the box origin is 16 B aligned
  int ns;                    // ring depth (stages in flight)
  int f64;                   // consumers convert each stage once into a float64 tile
  int f32blocks;             // float32 products, per-map float32 partials (DDCCA_MOMENTS_F32_BLOCKS)
};

// Named barrier over the consumer warps only (warps 0..G-1; the producer warp is not in it).
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

// One launch per (view, task kind): the single tensor map is used directly from
// the parameter space (no runtime selection of a tensor-map address).
// BLK: the blocked form only, its float64 sums in shared memory instead of registers (~60
// registers: three CTAs per SM instead of two, more warps to cover the stage ring)
template <int L1, int TCB, bool BLK>
__global__ void __launch_bounds__(256, BLK ? 3 : (L1 <= 9 ? 2 : 1))
    lag_tma_kernel(LagArgs A, TmaBoxes bx, const int* __restrict__ task_ids, int view,
                   const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) float stage_mem[];
  const int task = task_ids[blockIdx.x];
  const int split = blockIdx.y;
  const int batch = blockIdx.z;
  const TaskDev T = A.tasks[task];
  const int lane = threadIdx.x & 31;
  const int grp = threadIdx.x >> 5;
  const int nrows = T.y1 - T.y0;
  const bool short_task = nrows < L1;
  const int trb = short_task ? bx.rows_short : bx.rows_int;  // staged rows per map (box height)
  const int mb = short_task ? bx.mb_short : bx.mb_int;
  const int tile_elems = trb * TCB;
  const int stage_elems = mb * tile_elems;
  // stage slots 128-byte aligned: the TMA destination of every slot must be
  const int max_stage = (max(bx.rows_int * bx.mb_int, bx.rows_short * bx.mb_short) * TCB + 31) / 32 * 32;
  const int NS = bx.ns;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_mem + NS * max_stage);
  uint64_t* empty = full + NS;
  const int64_t m_begin = A.batch_off[batch];
  const int64_t m_end = A.batch_off[batch + 1];
  const int64_t per = A.per_split;
  const int64_t ma = m_begin + (int64_t)split * per;
  const int64_t mbnd = min(m_end, ma + per);
  const int nstages = ma < mbnd ? (int)((mbnd - ma + mb - 1) / mb) : 0;
  const int G = A.G;  // consumer warps; warp G is the producer
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], G);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  if (grp >= G) {
    // ---------------- producer (whole warp stays converged; lane 0 issues) ----------------
    // TMA box origins must be 16-byte aligned in the innermost dimension: start the
    // tile bx.shift columns early (consumers offset their columns by the same shift)
    const int x = T.x0 - (A.l2 - 1) - A.left - bx.shift;  // image column of tile column 0
    const int y = T.y0 - A.top;                 // image row of tile row 0
    const unsigned bytes = (unsigned)stage_elems * 4u;
    for (int s = 0; s < nstages; ++s) {
      const int slot = s % NS;
      if (s >= NS) mbar_wait(&empty[slot], (unsigned)((s / NS - 1) & 1));
      if (lane == 0) {
        mbar_expect_tx(&full[slot], bytes);
        tma_load_3d(stage_mem + slot * max_stage, &tmap, x, y, (int)(ma + (int64_t)s * mb), &full[slot]);
      }
      __syncwarp();
    }
  } else if constexpr (BLK) {
    // ---------------- consumers, blocked form, float64 sums in shared memory ----------------
    // accs[(dy * KDX + k) * cth + thread]: consecutive threads on consecutive words
    double* accs = reinterpret_cast<double*>(empty + NS);
    const int ct = threadIdx.x, cth = G * 32;
#pragma unroll
    for (int i = 0; i < L1 * KDX; ++i) accs[i * cth + ct] = 0.0;
    const int cown = lane + (A.l2 - 1) + bx.shift;
    const int cpart = lane + grp * KDX + bx.shift;
    const bool skip0 = (grp * KDX + KDX - 1) < (A.l2 - 1);
    const int kk = min(KDX, 2 * A.l2 - 1 - grp * KDX);
    F32Partials<L1> fp;
    f32_zero(fp);
    for (int s = 0; s < nstages; ++s) {
      const int slot = s % NS;
      mbar_wait(&full[slot], (unsigned)((s / NS) & 1));
      const float* tile = stage_mem + slot * max_stage;
      const int64_t ms = ma + (int64_t)s * mb;
      const int nm = (int)min((int64_t)mb, mbnd - ms);
      for (int j = 0; j < nm; ++j)
        lag_map_f32<L1, TCB>(tile + j * tile_elems, nrows, cown, cpart, short_task, skip0, kk, fp);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      // one float64 flush per stage (static lag indices on every branch)
#pragma unroll
      for (int dy = 0; dy < L1; ++dy) {
        double* a0 = accs + (dy * KDX) * cth + ct;
        if (kk >= 2) {
          a0[0] += (double)fp.fa2[dy].x;
          a0[cth] += (double)fp.fa2[dy].y;
          if (kk >= 3) a0[2 * cth] += (double)fp.fa1[dy];
        } else {
          a0[0] += (double)fp.fa1[dy];
        }
      }
      f32_zero(fp);
    }
    const int rslot = A.lane_slot[task * TILE_X + lane];
    const int xg = T.x0 + lane;
    const bool in_big = (rslot < 0) && (xg < A.xend);
    double* out = A.rec + (((int64_t)batch * 2 + view) * A.nsplit + split) * (int64_t)A.nrec * A.NDF;
    const int any_big = __any_sync(0xffffffffu, in_big);
    for (int dy = 0; dy < L1; ++dy)
      for (int k = 0; k < KDX; ++k) {
        const int lag = dy * A.NDX + grp * KDX + k;
        const double a = accs[(dy * KDX + k) * cth + ct];
        double v = in_big ? a : 0.0;
        v = warp_sum(v);
        if (lane == 0 && any_big) out[(int64_t)T.rec0 * A.NDF + lag] = v;
        if (rslot >= 0) out[(int64_t)(T.rec0 + rslot) * A.NDF + lag] = a;
      }
  } else {
    // ---------------- consumers ----------------
    double acc[L1][KDX];
#pragma unroll
    for (int dy = 0; dy < L1; ++dy)
#pragma unroll
      for (int k = 0; k < KDX; ++k) acc[dy][k] = 0.0;
    const int cown = lane + (A.l2 - 1) + bx.shift;
    const int cpart = lane + grp * KDX + bx.shift;
    const bool skip0 = (grp * KDX + KDX - 1) < (A.l2 - 1);
    const int kk = min(KDX, 2 * A.l2 - 1 - grp * KDX);  // live lags of this group
    if (bx.f32blocks) {
      F32Partials<L1> fp;
      f32_zero(fp);
      for (int s = 0; s < nstages; ++s) {
        const int slot = s % NS;
        mbar_wait(&full[slot], (unsigned)((s / NS) & 1));
        const float* tile = stage_mem + slot * max_stage;
        const int64_t ms = ma + (int64_t)s * mb;
        const int nm = (int)min((int64_t)mb, mbnd - ms);
        for (int j = 0; j < nm; ++j)
          lag_map_f32<L1, TCB>(tile + j * tile_elems, nrows, cown, cpart, short_task, skip0, kk, fp);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        f32_flush(fp, kk, acc);  // one float64 flush per stage of mb maps
      }
    } else if (bx.f64) {
      // convert each landed float32 stage once into a float64 tile shared by all consumer
      // warps (every element is read by ~l2 + 2 threads: one conversion instead of one
      // F2F per read on the FP64 pipe), release the float32 slot, then run the rings on doubles
      // Two float64 tiles: stage s converts into tile s & 1 while no consumer can still be
      // reading it (tile s & 1 last served stage s - 2, and every warp finished that stage's
      // maps before it reached stage s - 1's barrier), so one barrier per stage suffices.
      double* t64b = reinterpret_cast<double*>(empty + NS);  // 16-byte aligned: 2 NS barriers after the stages
      const int ctid = threadIdx.x, cthreads = G * 32;
      for (int s = 0; s < nstages; ++s) {
        const int slot = s % NS;
        double* t64 = t64b + (s & 1) * max_stage;
        mbar_wait(&full[slot], (unsigned)((s / NS) & 1));
        const float* tile = stage_mem + slot * max_stage;
        const int64_t ms = ma + (int64_t)s * mb;
        const int nm = (int)min((int64_t)mb, mbnd - ms);
        const int used = nm * tile_elems;
        for (int e = 4 * ctid; e < used; e += 4 * cthreads) {  // tile_elems is a multiple of 4 (TCB % 4 == 0)
          const float4 v = *reinterpret_cast<const float4*>(tile + e);
          *reinterpret_cast<double2*>(t64 + e) = make_double2(v.x, v.y);
          *reinterpret_cast<double2*>(t64 + e + 2) = make_double2(v.z, v.w);
        }
        consumer_sync(cthreads);
        if (lane == 0) mbar_arrive(&empty[slot]);
        for (int j = 0; j < nm; ++j)
          lag_map<L1, TCB>(t64 + j * tile_elems, TCB, nrows, cown, cpart, short_task, skip0, kk, acc);
      }
    } else {
      for (int s = 0; s < nstages; ++s) {
        const int slot = s % NS;
        mbar_wait(&full[slot], (unsigned)((s / NS) & 1));
        const float* tile = stage_mem + slot * max_stage;
        const int64_t ms = ma + (int64_t)s * mb;
        const int nm = (int)min((int64_t)mb, mbnd - ms);
        for (int j = 0; j < nm; ++j) {
          const float* t = tile + j * tile_elems;
          lag_map<L1, TCB>(t, TCB, nrows, cown, cpart, short_task, skip0, kk, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
    const int rslot = A.lane_slot[task * TILE_X + lane];
    const int xg = T.x0 + lane;
    const bool in_big = (rslot < 0) && (xg < A.xend);
    double* out = A.rec + (((int64_t)batch * 2 + view) * A.nsplit + split) * (int64_t)A.nrec * A.NDF;
    const int any_big = __any_sync(0xffffffffu, in_big);
#pragma unroll
    for (int dy = 0; dy < L1; ++dy)
#pragma unroll
      for (int k = 0; k < KDX; ++k) {
        const int lag = dy * A.NDX + grp * KDX + k;
        double v = in_big ? acc[dy][k] : 0.0;
        v = warp_sum(v);
        if (lane == 0 && any_big) out[(int64_t)T.rec0 * A.NDF + lag] = v;
        if (rslot >= 0) out[(int64_t)(T.rec0 + rslot) * A.NDF + lag] = acc[dy][k];
      }
  }
  __syncthreads();  // every warp (incl. the producer) leaves together, after all copies were consumed
}

// ----------------------------------------------------------------------------
// zone_reduce: Z[batch][view][rz][cz][lag] = sum over splits, records (fixed order)
// ----------------------------------------------------------------------------
__global__ void zone_reduce_kernel(const double* __restrict__ rec, const int* __restrict__ zrec_off,
                                   const int* __restrict__ zrec_list, double* __restrict__ Z, int nzone,
                                   int NDF, int nrec, int nsplit) {
  const int bv = blockIdx.y;
  const int64_t total = (int64_t)nzone * NDF;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int zone = (int)(e / NDF), lag = (int)(e % NDF);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) {
      const double* base = rec + ((int64_t)bv * nsplit + sp) * (int64_t)nrec * NDF;
      for (int t = zrec_off[zone]; t < zrec_off[zone + 1]; ++t) s += base[(int64_t)zrec_list[t] * NDF + lag];
    }
    Z[(int64_t)bv * total + e] = s;
  }
}

// ----------------------------------------------------------------------------
// assemble: Craw (canonical half, mirrored) -> centered -> payload c11 / c22
// ----------------------------------------------------------------------------
struct AsmArgs {
  const double* Z;
  const int* rz_lo; const int* rz_hi; const int* cz_lo; const int* cz_hi;
  double* payload;  // [batch][payload_len]
  int64_t plen;
  int nrz, ncz, NDX, NDF, l1, l2, d, center;
};

__global__ void assemble_kernel(AsmArgs A) {
  extern __shared__ double sm[];
  double* C = sm;                    // d*d raw then centered
  double* rs = sm + A.d * A.d;       // row sums (d)
  const int bv = blockIdx.x;
  const int batch = bv >> 1, view = bv & 1;
  const double* Z = A.Z + (int64_t)bv * A.nrz * A.ncz * A.NDF;
  const int d = A.d;
  // canonical entries: i = (a,b), j = (a+dy, b+dx) with dy > 0, or dy == 0 and dx >= 0
  for (int e = threadIdx.x; e < d * A.l1 * (2 * A.l2 - 1); e += blockDim.x) {
    const int i = e / (A.l1 * (2 * A.l2 - 1));
    const int rem = e % (A.l1 * (2 * A.l2 - 1));
    const int dy = rem / (2 * A.l2 - 1);
    const int dx = rem % (2 * A.l2 - 1) - (A.l2 - 1);
    const int a = i / A.l2, b = i % A.l2;
    const int a2 = a + dy, b2 = b + dx;
    if (a2 >= A.l1 || b2 < 0 || b2 >= A.l2) continue;
    if (dy == 0 && dx < 0) continue;
    const int lag = dy * A.NDX + (dx + A.l2 - 1);
    double s = 0.0;
    for (int rz = 0; rz < A.nrz; ++rz) {
      if (a < A.rz_lo[rz] || a > A.rz_hi[rz]) continue;
      for (int cz = 0; cz < A.ncz; ++cz) {
        if (b < A.cz_lo[cz] || b > A.cz_hi[cz]) continue;
        s += Z[((int64_t)rz * A.ncz + cz) * A.NDF + lag];
      }
    }
    const int j = a2 * A.l2 + b2;
    C[i * d + j] = s;
    C[j * d + i] = s;
  }
  __syncthreads();
  double* out = A.payload + (int64_t)batch * A.plen + (view == 0 ? 0 : (int64_t)d * d);
  if (!A.center) {
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) out[e] = C[e];
    return;
  }
  // H C H with H = I - 11^T/d: C_ij - r_i/d - r_j/d + T/d^2 (C symmetric)
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double r = 0.0;
    for (int j = 0; j < d; ++j) r += C[i * d + j];
    rs[i] = r;
  }
  __syncthreads();
  __shared__ double tot;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < d; ++i) t += rs[i];
    tot = t;
  }
  __syncthreads();
  const double invd = 1.0 / d;
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
    const int i = e / d, j = e % d;
    out[e] = C[e] - rs[i] * invd - rs[j] * invd + tot * invd * invd;
  }
}

// ----------------------------------------------------------------------------
// rect_sums: per-map window sums  sum_{patches} x  (centered if `center`)
// ----------------------------------------------------------------------------
struct RectArgs {
  const float* maps[2];
  double* out;  // [view][map][d]
  const int* rz_y0;  // [nrz + 1] first padded row of each row zone, then Hp
  const int* cz_of_x;
  const int* a_rz;   // [l1][2] first / last row zone covering tap row a
  const int* b_cz;   // [l2][2] first / last column zone covering tap column b
  int64_t n_maps;
  int p, q, top, left, Hp, Wp, nrz, ncz, l1, l2, d, center, big_cz;
};

// Warp per map. Every lane keeps the running sums of its own columns (float4 groups)
// over the rows of the current row zone; at a zone boundary (warp-uniform) the sums go
// either to the column's singleton zone (border columns) or into the warp-reduced
// interior zone. Rows stream in 8-row groups whatever the zones (the boundaries come
// from the rz_y0 table, no per-row lookups). Then R[a][b] = sum of the zone sums
// covering (a, b) (a contiguous zone range per a and per b), centered.
constexpr int RS_WARPS = 4;
constexpr int RS_COLS = 8;  // columns per lane (q <= 256)
constexpr int RS_ROWS = 8;  // rows in flight per warp (narrow form)

// NARROW: q % 4 == 0 and q <= 128 (one float4 per lane per row, 4 lane sums).
template <bool NARROW>
__global__ void __launch_bounds__(RS_WARPS * 32) rect_sums_kernel(RectArgs A) {
  constexpr int NC = NARROW ? 4 : RS_COLS;
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int zsz = A.nrz * A.ncz;
  double* Zp = sm + warp * (zsz + A.d);
  double* R = Zp + zsz;
  const int64_t m = (int64_t)blockIdx.x * RS_WARPS + warp;
  const int view = blockIdx.y;
  if (m >= A.n_maps) return;
  const float* img = (view == 0 ? A.maps[0] : A.maps[1]) + m * (int64_t)A.p * A.q;
  for (int e = lane; e < zsz; e += 32) Zp[e] = 0.0;
  const bool vec = NARROW || (A.q & 3) == 0;
  // lane columns: vec -> 4*lane + 128*g + k ; scalar -> lane + 32*k
  int czc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int col = vec ? (4 * lane + 128 * (k >> 2) + (k & 3)) : (lane + 32 * k);
    czc[k] = col < A.q ? A.cz_of_x[col + A.left] : -1;
  }
  __syncwarp();
  const int big = A.big_cz;
  double acc[NC];
  auto flush = [&](int rz) {
    double s_int = 0.0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (czc[k] >= 0) {
        if (czc[k] == big) s_int += acc[k];
        else Zp[rz * A.ncz + czc[k]] = acc[k];  // singleton column zone: this lane's column only
      }
      acc[k] = 0.0;
    }
    s_int = warp_sum(s_int);
    if (lane == 0 && big >= 0) Zp[rz * A.ncz + big] = s_int;
  };
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = 0.0;
  if constexpr (NARROW) {
    // one float4 per lane per row; RS_ROWS rows' loads in flight before their sums (HBM latency)
    const bool live = 4 * lane < A.q;
    const float* base = img + 4 * lane;
    int rz = 0;
    while (A.rz_y0[rz + 1] <= A.top) ++rz;  // zone of image row 0
    int ynext = A.rz_y0[rz + 1] - A.top;     // first image row of the next zone
    for (int i = 0; i < A.p; i += RS_ROWS) {
      float4 v[RS_ROWS];
#pragma unroll
      for (int u = 0; u < RS_ROWS; ++u)
        v[u] = (live && i + u < A.p) ? __ldg(reinterpret_cast<const float4*>(base + (int64_t)(i + u) * A.q))
                                      : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < RS_ROWS; ++u) {
        if (i + u < A.p) {
          if (i + u >= ynext) {  // warp-uniform: close the zone, move to the one holding row i + u
            flush(rz);
            do { ++rz; } while (A.rz_y0[rz + 1] - A.top <= i + u);
            ynext = A.rz_y0[rz + 1] - A.top;
          }
          acc[0] += (double)v[u].x;
          acc[1] += (double)v[u].y;
          acc[2] += (double)v[u].z;
          acc[3] += (double)v[u].w;
        }
      }
    }
    flush(rz);
  } else {
    for (int rz = 0; rz < A.nrz; ++rz) {
      const int i0 = max(A.rz_y0[rz] - A.top, 0), i1 = min(A.rz_y0[rz + 1] - A.top, A.p);
      if (i0 >= i1) continue;
      for (int i = i0; i < i1; ++i) {
        const float* row = img + (int64_t)i * A.q;
        if (vec) {
#pragma unroll
          for (int g = 0; g < RS_COLS / 4; ++g) {
            const int c0 = 4 * lane + 128 * g;
            if (c0 < A.q) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(row + c0));
              acc[4 * g + 0] += (double)v.x;
              acc[4 * g + 1] += (double)v.y;
              acc[4 * g + 2] += (double)v.z;
              acc[4 * g + 3] += (double)v.w;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < RS_COLS; ++k)
            if (lane + 32 * k < A.q) acc[k] += (double)__ldg(row + lane + 32 * k);
        }
      }
      flush(rz);
    }
  }
  __syncwarp();
  for (int k = lane; k < A.d; k += 32) {
    const int a = k / A.l2, b = k % A.l2;
    const int r0 = A.a_rz[2 * a], r1 = A.a_rz[2 * a + 1], c0 = A.b_cz[2 * b], c1 = A.b_cz[2 * b + 1];
    double s = 0.0;
    for (int rz = r0; rz <= r1; ++rz)
      for (int cz = c0; cz <= c1; ++cz) s += Zp[rz * A.ncz + cz];
    R[k] = s;
  }
  __syncwarp();
  double t = 0.0;
  for (int k = lane; k < A.d; k += 32) t += R[k];
  const double mean = warp_sum(t) / A.d;
  double* o = A.out + ((int64_t)view * A.n_maps + m) * A.d;
  for (int k = lane; k < A.d; k += 32) o[k] = A.center ? R[k] - mean : R[k];
}

// ----------------------------------------------------------------------------
// batch_epilogue: class sums S (d x C), global sums g, counts
// ----------------------------------------------------------------------------
constexpr size_t EPI_SMEM_MAX = 160 * 1024;  // class-sum staging in shared memory up to this size

// Class sums S (d x C, accumulated in shared memory when it fits, else in place), global
// sums g and counts of one (batch, view). Maps of one sample share a label and are
// contiguous, so each thread adds a run of equal labels in registers and touches S
// once per run (the same left-to-right order per element as a per-map update).
__global__ void batch_epilogue_kernel(const double* __restrict__ msum, const int32_t* __restrict__ label,
                                      const int64_t* __restrict__ batch_off, int64_t n_maps, int d, int C,
                                      int64_t plen, double cols_per_map, double* __restrict__ payload) {
  extern __shared__ double sS[];
  const int batch = blockIdx.x;
  const int view = blockIdx.y;
  const PayloadView pv = payload_view(d, C);
  double* P = payload + (int64_t)batch * plen;
  double* S = P + (view == 0 ? pv.s1 : pv.s2);
  double* g = P + (view == 0 ? pv.g1 : pv.g2);
  const bool staged = (size_t)d * C * sizeof(double) <= EPI_SMEM_MAX;
  double* acc = staged ? sS : S;
  const int64_t m0 = batch_off[batch], m1 = batch_off[batch + 1];
  for (int e = threadIdx.x; e < d * C; e += blockDim.x) acc[e] = 0.0;
  __syncthreads();
  const double* src = msum + (int64_t)view * n_maps * d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    double gs = 0.0;
    int lab = -1;
    double run = 0.0;
    for (int64_t m = m0; m < m1; ++m) {
      const double v = src[m * d + k];
      // labels outside [0, C) are a caller error (the Python layer raises ShapeError
      // first); here they only skip the class sums so the public ABI never writes
      // out of bounds
      const int l = ((unsigned)label[m] < (unsigned)C) ? label[m] : -1;
      if (l != lab) {  // close the previous run, continue this label's running sum
        if (lab >= 0) acc[(int64_t)k * C + lab] = run;
        lab = l;
        run = l >= 0 ? acc[(int64_t)k * C + l] : 0.0;
      }
      run += v;
      gs += v;
    }
    if (lab >= 0) acc[(int64_t)k * C + lab] = run;
    g[k] = gs;
  }
  __syncthreads();
  if (staged)
    for (int e = threadIdx.x; e < d * C; e += blockDim.x) S[e] = acc[e];
  if (view == 0) {
    double* cnt = P + pv.ncls;
    for (int c = threadIdx.x; c < C; c += blockDim.x) cnt[c] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int64_t m = m0; m < m1; ++m)
        if ((unsigned)label[m] < (unsigned)C) cnt[label[m]] += cols_per_map;
      P[pv.n] = (double)(m1 - m0) * cols_per_map;
    }
  }
}

// ----------------------------------------------------------------------------
// direct path (any stride / padding): explicit float64 patches per block
// ----------------------------------------------------------------------------
constexpr int DIRECT_K = 64;  // patches staged per step
constexpr int DIRECT_ENT = 8; // Gram entries per thread per pass

__global__ void direct_gram_kernel(const float* maps1, const float* maps2, const int64_t* batch_off, Geo g,
                                   int center, int nsplit, int64_t per_cols,
                                   double* rec /* [batch][view][split][d*d] */) {
  extern __shared__ double stage[];  // [DIRECT_K][d]
  const int split = blockIdx.x;
  const int batch = blockIdx.y;
  const int view = blockIdx.z;
  const float* src = view == 0 ? maps1 : maps2;
  const int d = g.d;
  const int64_t m0 = batch_off[batch], m1 = batch_off[batch + 1];
  const int64_t cols_per_map = (int64_t)g.oh * g.ow;
  const int64_t ncols = (m1 - m0) * cols_per_map;
  const int64_t per = per_cols;  // fixed columns per split (independent of the other batches)
  const int64_t c0 = (int64_t)split * per, c1 = min(ncols, c0 + per);
  const int nent = d * d;
  double* out = rec + (((int64_t)batch * 2 + view) * nsplit + split) * nent;
  // entries are processed in passes of DIRECT_ENT * blockDim; patches are restaged per pass
  for (int e0 = 0; e0 < nent; e0 += DIRECT_ENT * blockDim.x) {
    double acc[DIRECT_ENT];
#pragma unroll
    for (int u = 0; u < DIRECT_ENT; ++u) acc[u] = 0.0;
    for (int64_t cb = c0; cb < c1; cb += DIRECT_K) {
      const int kk = (int)min((int64_t)DIRECT_K, c1 - cb);
      __syncthreads();
      for (int e = threadIdx.x; e < kk * d; e += blockDim.x) {
        const int k = e / d, t = e % d;
        const int64_t col = cb + k;
        const int64_t m = m0 + col / cols_per_map;
        const int pos = (int)(col % cols_per_map);
        const int u = pos / g.ow, v = pos % g.ow;
        const int i = u * g.stride - g.top + t / g.l2, j = v * g.stride - g.left + t % g.l2;
        float x = 0.f;
        if (i >= 0 && i < g.p && j >= 0 && j < g.q) x = src[m * (int64_t)g.p * g.q + (int64_t)i * g.q + j];
        stage[k * d + t] = (double)x;
      }
      __syncthreads();
      if (center) {
        for (int k = threadIdx.x; k < kk; k += blockDim.x) {
          double s = 0.0;
          for (int t = 0; t < d; ++t) s += stage[k * d + t];
          const double mu = s / d;
          for (int t = 0; t < d; ++t) stage[k * d + t] -= mu;
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < DIRECT_ENT; ++u) {
        const int e = e0 + threadIdx.x + u * blockDim.x;
        if (e < nent) {
          const int i = e / d, j = e % d;
          double s = acc[u];
          for (int k = 0; k < kk; ++k) s = fma(stage[k * d + i], stage[k * d + j], s);
          acc[u] = s;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < DIRECT_ENT; ++u) {
      const int e = e0 + threadIdx.x + u * blockDim.x;
      if (e < nent) out[e] = acc[u];
    }
  }
}

__global__ void direct_reduce_kernel(const double* rec, int nsplit, int d, int64_t plen, double* payload) {
  const int bv = blockIdx.x;
  const int batch = bv >> 1, view = bv & 1;
  const int nent = d * d;
  double* out = payload + (int64_t)batch * plen + (view == 0 ? 0 : nent);
  for (int e = threadIdx.x; e < nent; e += blockDim.x) {
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += rec[((int64_t)bv * nsplit + sp) * nent + e];
    out[e] = s;
  }
}

// per-map patch sums for the direct path (any stride): sum over the patch grid
__global__ void direct_map_sums_kernel(const float* maps1, const float* maps2, int64_t n_maps, Geo g, int center,
                                       double* out /* [view][map][d] */) {
  extern __shared__ double R[];
  const int64_t m = blockIdx.x;
  const int view = blockIdx.y;
  const float* img = (view == 0 ? maps1 : maps2) + m * (int64_t)g.p * g.q;
  const int d = g.d;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    const int di = t / g.l2, dj = t % g.l2;
    double s = 0.0;
    for (int u = 0; u < g.oh; ++u) {
      const int i = u * g.stride - g.top + di;
      if (i < 0 || i >= g.p) continue;
      for (int v = 0; v < g.ow; ++v) {
        const int j = v * g.stride - g.left + dj;
        if (j >= 0 && j < g.q) s += (double)img[(int64_t)i * g.q + j];
      }
    }
    R[t] = s;
  }
  __syncthreads();
  __shared__ double mean;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < d; ++k) t += R[k];
    mean = t / d;
  }
  __syncthreads();
  double* o = out + ((int64_t)view * n_maps + m) * d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) o[k] = center ? R[k] - mean : R[k];
}

// ----------------------------------------------------------------------------
// explicit columns (API accumulate_batch): per-block partial Gram + class sums
// ----------------------------------------------------------------------------
constexpr int COLS_PER_BLOCK = 2048;

__global__ void columns_partial_kernel(const double* x, const double* y, const int64_t* labels, int64_t cols, int d,
                                       int C, double* part /* [block][view][d*d + d*C + d] */) {
  extern __shared__ double st[];  // [DIRECT_K][d] x2
  const int64_t c0 = (int64_t)blockIdx.x * COLS_PER_BLOCK;
  const int64_t c1 = min(cols, c0 + COLS_PER_BLOCK);
  const int nent = d * d;
  const int64_t per_view = (int64_t)nent + (int64_t)d * C + d;
  double* outb = part + (int64_t)blockIdx.x * 2 * per_view;
  for (int view = 0; view < 2; ++view) {
    const double* src = view == 0 ? x : y;
    double* o = outb + view * per_view;
    // Gram entries
    for (int e0 = 0; e0 < nent; e0 += blockDim.x) {
      const int e = e0 + threadIdx.x;
      double s = 0.0;
      for (int64_t cb = c0; cb < c1; cb += DIRECT_K) {
        const int kk = (int)min((int64_t)DIRECT_K, c1 - cb);
        __syncthreads();
        for (int t = threadIdx.x; t < kk * d; t += blockDim.x) {
          const int k = t / d, r = t % d;
          st[k * d + r] = src[(int64_t)r * cols + cb + k];
        }
        __syncthreads();
        if (e < nent) {
          const int i = e / d, j = e % d;
          for (int k = 0; k < kk; ++k) s = fma(st[k * d + i], st[k * d + j], s);
        }
      }
      if (e < nent) o[e] = s;
    }
    // class sums and global sums (thread per row, columns in order)
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
      double* S = o + nent;
      for (int c = 0; c < C; ++c) S[(int64_t)k * C + c] = 0.0;
      double gs = 0.0;
      for (int64_t c = c0; c < c1; ++c) {
        const double v = src[(int64_t)k * cols + c];
        if ((uint64_t)labels[c] < (uint64_t)C) S[(int64_t)k * C + labels[c]] += v;  // ABI guard
        gs += v;
      }
      o[nent + (int64_t)d * C + k] = gs;
    }
  }
}

__global__ void columns_reduce_kernel(const double* part, int nblk, const int64_t* labels, int64_t cols, int d,
                                      int C, double* payload) {
  const PayloadView pv = payload_view(d, C);
  const int nent = d * d;
  const int64_t per_view = (int64_t)nent + (int64_t)d * C + d;
  for (int view = 0; view < 2; ++view) {
    for (int64_t e = threadIdx.x; e < per_view; e += blockDim.x) {
      double s = 0.0;
      for (int b = 0; b < nblk; ++b) s += part[((int64_t)b * 2 + view) * per_view + e];
      int64_t dst;
      if (e < nent) dst = (view == 0 ? pv.c11 : pv.c22) + e;
      else if (e < nent + (int64_t)d * C) dst = (view == 0 ? pv.s1 : pv.s2) + (e - nent);
      else dst = (view == 0 ? pv.g1 : pv.g2) + (e - nent - (int64_t)d * C);
      payload[dst] += s;
    }
  }
  if (threadIdx.x == 0) {
    for (int64_t c = 0; c < cols; ++c)
      if ((uint64_t)labels[c] < (uint64_t)C) payload[pv.ncls + labels[c]] += 1.0;
    payload[pv.n] += (double)cols;
  }
}

__global__ void tree_level_kernel(double* parts, int n, int64_t len, int stride_in) {
  // pairs (i, i+1) at positions i = 0, 2, ... in the current level; level entries are
  // spaced `stride_in` payloads apart. Result stored in place of the left element.
  const int npairs = n / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)npairs * len;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int pr = (int)(e / len);
    const int64_t k = e % len;
    double* a = parts + (int64_t)(2 * pr) * stride_in * len;
    const double* b = parts + (int64_t)(2 * pr + 1) * stride_in * len;
    a[k] = a[k] + b[k];
  }
}

}  // namespace ddcca

using namespace ddcca;

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
namespace {

struct LagLayout {
  Plan P;
  int nsplit;
  size_t off_tasks, off_lane, off_boff, off_rec, off_Z, off_zoff, off_zlist, off_zones, off_msum, off_ids, total;
  int nzone_rec;  // total entries of zrec_list
};

// dynamic shared memory of batch_epilogue_kernel (0: class sums accumulated in place)
static size_t epi_smem(int d, int C) {
  const size_t b = (size_t)d * C * sizeof(double);
  if (b > EPI_SMEM_MAX) return 0;
  cudaFuncSetAttribute(batch_epilogue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
  return b;
}

// Maps per split. A batch's split boundaries depend only on the split size (a function of
// the flags alone, never of the other batches of the call), so every batch's partial (and
// the deterministic multi-GPU reduction) is the same whichever call or rank computes it.
// Fine splits (32 maps) for layers with one map per sample (DDCCA_MOMENTS_FINE_SPLITS)
// give the first layer 4x more CTAs.
static int64_t split_maps(int64_t max_maps, int flags) {
  (void)max_maps;
  return (flags & DDCCA_MOMENTS_FINE_SPLITS) ? MAPS_PER_SPLIT / 4 : MAPS_PER_SPLIT;
}

static int nsplit_for(int64_t max_maps, int64_t per) {
  return (int)std::max<int64_t>(1, (max_maps + per - 1) / per);
}

// splits the workspace is sized for (the finer of the two split sizes)
static int nsplit_ws(int64_t max_maps) {
  return nsplit_for(max_maps, split_maps(max_maps, DDCCA_MOMENTS_FINE_SPLITS));
}

static void lag_layout(const Geo& g, int nb, int64_t max_maps, int64_t n_maps, int nsplit, LagLayout* L) {
  make_plan(g, &L->P);
  L->nsplit = nsplit;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L->off_tasks = take(sizeof(TaskDev) * L->P.tasks.size());
  L->off_lane = take(sizeof(int) * L->P.lane_slot.size());
  L->off_boff = take(sizeof(int64_t) * (nb + 1));
  L->off_rec = take(sizeof(double) * (size_t)nb * 2 * L->nsplit * L->P.nrec * L->P.NDF);
  L->off_Z = take(sizeof(double) * (size_t)nb * 2 * L->P.nrz * L->P.ncz * L->P.NDF);
  L->off_zoff = take(sizeof(int) * (L->P.nrz * L->P.ncz + 1));
  L->off_zlist = take(sizeof(int) * L->P.nrec);
  // zone tables + rect_sums helpers: row start of each row zone, covering zone range per tap row / column
  L->off_zones = take(sizeof(int) * (2 * L->P.nrz + 2 * L->P.ncz + g.Hp + g.Wp + (L->P.nrz + 1) + 2 * g.l1 + 2 * g.l2));
  L->off_msum = take(sizeof(double) * 2 * (size_t)n_maps * g.d);
  L->off_ids = take(sizeof(int) * L->P.tasks.size());
  L->total = o;
}

}  // namespace

extern "C" {

int ddcca_version(void) { return 1; }

const char* ddcca_last_error(void) { return err_buf(); }

int64_t ddcca_payload_len(int dim, int class_count) { return payload_len(dim, class_count); }

size_t ddcca_moments_workspace(const ddcca_geom* gg, int n_batches, int64_t max_maps_per_batch, int class_count) {
  (void)class_count;
  Geo g{};
  if (make_geo(gg, &g) != DDCCA_OK) return 0;
  // worst case over the per-batch maps: n_maps <= n_batches * max_maps
  const int64_t n_maps = (int64_t)n_batches * max_maps_per_batch;
  if (g.stride == 1 && g.l1 <= MAX_LAG_L && g.l2 <= MAX_LAG_L) {
    LagLayout L;
    lag_layout(g, n_batches, max_maps_per_batch, n_maps, nsplit_ws(max_maps_per_batch), &L);
    return L.total;
  }
  const int nsplit = nsplit_ws(max_maps_per_batch);
  return align_up(sizeof(double) * (size_t)n_batches * 2 * nsplit * g.d * g.d, 256) +
         align_up(sizeof(int64_t) * (n_batches + 1), 256) + align_up(sizeof(double) * 2 * (size_t)n_maps * g.d, 256);
}

int ddcca_moments_partial(const float* maps1, const float* maps2, const int32_t* map_label,
                          const int64_t* batch_offsets_host, int n_batches, const ddcca_geom* gg, int center,
                          int class_count, double* partials, void* ws, size_t ws_bytes, void* stream) {
  return ddcca_moments_partial_ex(maps1, maps2, map_label, batch_offsets_host, n_batches, gg, center, class_count,
                                  partials, ws, ws_bytes, 0, stream);
}

int ddcca_moments_partial_ex(const float* maps1, const float* maps2, const int32_t* map_label,
                             const int64_t* batch_offsets_host, int n_batches, const ddcca_geom* gg, int center,
                             int class_count, double* partials, void* ws, size_t ws_bytes, int flags,
                             void* stream) {
  if (flags & ~(DDCCA_MOMENTS_F32_BLOCKS | DDCCA_MOMENTS_FINE_SPLITS))
    return fail(DDCCA_ECONFIG, "unknown moments flags 0x%x", flags);
  Geo g{};
  DDCCA_TRY(make_geo(gg, &g));
  if (n_batches < 1) return fail(DDCCA_ECONFIG, "no batches to accumulate");
  if (class_count < 1) return fail(DDCCA_ECONFIG, "invalid class count %d", class_count);
  if (!maps1 || !maps2 || !map_label || !partials || !batch_offsets_host) return fail(DDCCA_ESHAPE, "null pointer");
  int64_t max_maps = 0;
  for (int b = 0; b < n_batches; ++b) {
    const int64_t n = batch_offsets_host[b + 1] - batch_offsets_host[b];
    if (n < 1) return fail(DDCCA_ESHAPE, "batch %d is empty", b);
    max_maps = std::max(max_maps, n);
  }
  const int64_t n_maps = batch_offsets_host[n_batches];
  if (batch_offsets_host[0] != 0) return fail(DDCCA_ESHAPE, "batch offsets must start at 0");
  cudaStream_t st = as_stream(stream);
  const int64_t plen = payload_len(g.d, class_count);
  const double cols_per_map = (double)g.oh * g.ow;
  char* w = static_cast<char*>(ws);

  if (g.stride == 1 && g.l1 <= MAX_LAG_L && g.l2 <= MAX_LAG_L) {
    LagLayout L;
    const int64_t per = split_maps(max_maps, flags);
    lag_layout(g, n_batches, max_maps, n_maps, nsplit_for(max_maps, per), &L);
    if (ws_bytes < L.total) return fail(DDCCA_ECONFIG, "moments workspace too small (%zu < %zu)", ws_bytes, L.total);
    const Plan& P = L.P;
    // upload plan tables (small; pageable H2D copies are staged by the driver)
    std::vector<TaskDev> td(P.tasks.size());
    size_t max_stage = 1;
    for (size_t t = 0; t < P.tasks.size(); ++t) {
      const int nr = P.tasks[t].y1 - P.tasks[t].y0;
      const int tr = (nr < g.l1 ? nr : (nr + g.l1 - 1) / g.l1 * g.l1) + g.l1 - 1;
      const int mb = std::max(1, std::min(8, STAGE_ROWS / tr));
      td[t] = {P.tasks[t].y0, P.tasks[t].y1, P.tasks[t].x0, P.tasks[t].rec0, mb};
      max_stage = std::max(max_stage, (size_t)mb * tr);
    }
    const int nzone = P.nrz * P.ncz;
    std::vector<int> zoff(nzone + 1, 0), zlist(P.nrec);
    for (int r = 0; r < P.nrec; ++r) zoff[P.recs[r].rz * P.ncz + P.recs[r].cz + 1]++;
    for (int z = 0; z < nzone; ++z) zoff[z + 1] += zoff[z];
    {
      std::vector<int> fill(zoff.begin(), zoff.end() - 1);
      for (int r = 0; r < P.nrec; ++r) zlist[fill[P.recs[r].rz * P.ncz + P.recs[r].cz]++] = r;
    }
    std::vector<int> zones;
    zones.insert(zones.end(), P.z.rz_lo.begin(), P.z.rz_lo.end());
    zones.insert(zones.end(), P.z.rz_hi.begin(), P.z.rz_hi.end());
    zones.insert(zones.end(), P.z.cz_lo.begin(), P.z.cz_lo.end());
    zones.insert(zones.end(), P.z.cz_hi.begin(), P.z.cz_hi.end());
    zones.insert(zones.end(), P.z.rz_of_y.begin(), P.z.rz_of_y.end());
    zones.insert(zones.end(), P.z.cz_of_x.begin(), P.z.cz_of_x.end());
    // rect_sums: first padded row of each row zone (+ Hp), and for each tap row a / column b the
    // contiguous range of zones covering it (zones are intervals sorted by position)
    for (int rz = 0, y = 0; rz < P.nrz; ++rz) {
      while (P.z.rz_of_y[y] != rz) ++y;
      zones.push_back(y);
    }
    zones.push_back(g.Hp);
    auto cover = [&](const std::vector<int>& lo, const std::vector<int>& hi, int v) {
      int f = -1, l = -2;
      for (int z = 0; z < (int)lo.size(); ++z)
        if (v >= lo[z] && v <= hi[z]) { if (f < 0) f = z; l = z; }
      zones.push_back(f);
      zones.push_back(l);
    };
    for (int a = 0; a < g.l1; ++a) cover(P.z.rz_lo, P.z.rz_hi, a);
    for (int b = 0; b < g.l2; ++b) cover(P.z.cz_lo, P.z.cz_hi, b);
    {
      const Upload parts[] = {
          {td.data(), sizeof(TaskDev) * td.size(), w + L.off_tasks},
          {P.lane_slot.data(), sizeof(int) * P.lane_slot.size(), w + L.off_lane},
          {batch_offsets_host, sizeof(int64_t) * (n_batches + 1), w + L.off_boff},
          {zoff.data(), sizeof(int) * zoff.size(), w + L.off_zoff},
          {zlist.data(), sizeof(int) * zlist.size(), w + L.off_zlist},
          {zones.data(), sizeof(int) * zones.size(), w + L.off_zones},
      };
      DDCCA_TRY(upload_parts(parts, 6, st));
    }
    DDCCA_TRY(check_launch("moments: plan upload"));
    const int* zd = reinterpret_cast<const int*>(w + L.off_zones);
    const int *rz_lo = zd, *rz_hi = zd + P.nrz, *cz_lo = zd + 2 * P.nrz, *cz_hi = zd + 2 * P.nrz + P.ncz;
    const int* rz_of_y = zd + 2 * P.nrz + 2 * P.ncz;
    const int* cz_of_x = rz_of_y + g.Hp;
    const int* rz_y0 = cz_of_x + g.Wp;
    const int* a_rz = rz_y0 + P.nrz + 1;
    const int* b_cz = a_rz + 2 * g.l1;

    LagArgs A;
    A.maps[0] = maps1;
    A.maps[1] = maps2;
    A.tasks = reinterpret_cast<const TaskDev*>(w + L.off_tasks);
    A.lane_slot = reinterpret_cast<const int*>(w + L.off_lane);
    A.batch_off = reinterpret_cast<const int64_t*>(w + L.off_boff);
    A.rec = reinterpret_cast<double*>(w + L.off_rec);
    A.p = g.p; A.q = g.q; A.top = g.top; A.left = g.left; A.Wp = g.Wp; A.l2 = g.l2;
    A.G = P.G; A.NDX = P.NDX; A.NDF = P.NDF; A.nrec = P.nrec; A.nsplit = L.nsplit; A.per_split = per;
    A.nbatch = n_batches;
    A.xend = g.left + g.q;
    // F32: three float32 stages; else two float64 compute tiles + two float32 cp.async stages
    const size_t smem = (LAG_F32 ? 3 * sizeof(float) : 2 * sizeof(double) + 2 * sizeof(float)) * max_stage *
                        (TILE_X + P.NDX - 1);
    dim3 grid((unsigned)P.tasks.size(), (unsigned)L.nsplit, (unsigned)(n_batches * 2));
    dim3 block(32 * P.G);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      kern<<<grid, block, smem, st>>>(A);
    };
    const int tcv = TILE_X + P.NDX - 1;
    bool launched = false;
    const bool use_tma = getenv("DDCCA_NO_TMA") == nullptr;
    if (use_tma && (g.q % 4) == 0 && (g.l1 == 5 || g.l1 == 7 || g.l1 == 9) && g.l1 == g.l2) {
      // box geometry: interior tasks stage slab+halo rows, short tasks L1 rows; widths padded to 4
      TmaBoxes bx;
      const int stage_rows = env_int("DDCCA_TMA_ROWS", STAGE_ROWS);
      bx.ns = std::max(2, std::min(8, env_int("DDCCA_TMA_STAGES", TMA_NS)));
      bx.rows_int = P.slab + g.l1 - 1;
      bx.mb_int = std::max(1, std::min(8, stage_rows / bx.rows_int));
      bx.rows_short = g.l1;
      for (const Task& t : P.tasks)
        if (t.y1 - t.y0 < g.l1) bx.rows_short = std::max(bx.rows_short, t.y1 - t.y0 + g.l1 - 1);
      // short tasks (single border rows) do little work per map: the blocked form (float32
      // stages, no float64 tiles) takes 16 maps per stage (-2 % layer-2 moments); the exact
      // form keeps 8 (its float64 tiles would cost occupancy)
      const bool blocked = (flags & DDCCA_MOMENTS_F32_BLOCKS) != 0;
      bx.mb_short = blocked ? std::max(1, std::min(16, (stage_rows + 16) / bx.rows_short))
                            : std::max(1, std::min(8, stage_rows / bx.rows_short));
      const int x_first = g.left - (g.l2 - 1) - g.left;  // tile origin column of the first column tile
      bx.shift = ((x_first % 4) + 4) % 4;
      const int tcb = (tcv + bx.shift + 3) / 4 * 4;
      CUtensorMap tm[4];
      bool ok = true;
      for (int v = 0; v < 2 && ok; ++v) {
        const float* base = v == 0 ? maps1 : maps2;
        ok = make_map(&tm[v], base, n_maps, g.p, g.q, tcb, bx.rows_int, bx.mb_int) &&
             make_map(&tm[2 + v], base, n_maps, g.p, g.q, tcb, bx.rows_short, bx.mb_short);
      }
      if (ok) {
        const size_t max_stage =
            ((size_t)std::max(bx.rows_int * bx.mb_int, bx.rows_short * bx.mb_short) * tcb + 31) / 32 * 32;
        bx.f32blocks = (flags & DDCCA_MOMENTS_F32_BLOCKS) ? 1 : 0;
        // float64 compute tiles only for the exact form (the blocked form reads the float32 stages)
        bx.f64 = (env_int("DDCCA_LAG_F32", 0) == 0 && !bx.f32blocks) ? 1 : 0;
        // float64 path: two compute tiles (one barrier per stage) and, by default, two float32
        // TMA stages, so two CTAs still fit one SM
        if (bx.f64 && !bx.f32blocks) bx.ns = std::max(2, std::min(8, env_int("DDCCA_TMA_STAGES", 2)));
        // blocked form: float64 sums in shared memory, two stages (three CTAs per SM fit)
        if (bx.f32blocks) bx.ns = std::max(2, std::min(8, env_int("DDCCA_TMA_STAGES", 2)));
        const size_t tsmem = sizeof(float) * bx.ns * max_stage + (2 * bx.ns + 1) * sizeof(uint64_t) +
                             (bx.f64 ? 2 * sizeof(double) * max_stage : 0) +
                             (bx.f32blocks ? sizeof(double) * (size_t)P.G * 32 * g.l1 * KDX : 0);
        dim3 tblock(32 * (P.G + 1));
        // task ids by kind, uploaded after the plan tables
        std::vector<int> ids_int, ids_short;
        for (size_t t = 0; t < P.tasks.size(); ++t)
          (P.tasks[t].y1 - P.tasks[t].y0 < g.l1 ? ids_short : ids_int).push_back((int)t);
        int* ids_dev = reinterpret_cast<int*>(w + L.off_ids);
        std::vector<int> ids_all(ids_int);
        ids_all.insert(ids_all.end(), ids_short.begin(), ids_short.end());
        {
          const Upload ids_part{ids_all.data(), sizeof(int) * ids_all.size(), ids_dev};
          DDCCA_TRY(upload_parts(&ids_part, 1, st));
        }
        auto tgo = [&](auto kern) {
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
          cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          for (int v = 0; v < 2; ++v) {
            if (!ids_int.empty())
              kern<<<dim3((unsigned)ids_int.size(), (unsigned)L.nsplit, (unsigned)n_batches), tblock, tsmem, st>>>(
                  A, bx, ids_dev, v, tm[v]);
            if (!ids_short.empty())
              kern<<<dim3((unsigned)ids_short.size(), (unsigned)L.nsplit, (unsigned)n_batches), tblock, tsmem, st>>>(
                  A, bx, ids_dev + ids_int.size(), v, tm[2 + v]);
          }
        };
        if (bx.f32blocks) {
          if (g.l1 == 5 && tcb == 40) { tgo(lag_tma_kernel<5, 40, true>); launched = true; }
          else if (g.l1 == 7 && tcb == 48) { tgo(lag_tma_kernel<7, 48, true>); launched = true; }
          else if (g.l1 == 9 && tcb == 52) { tgo(lag_tma_kernel<9, 52, true>); launched = true; }
        } else {
          if (g.l1 == 5 && tcb == 40) { tgo(lag_tma_kernel<5, 40, false>); launched = true; }
          else if (g.l1 == 7 && tcb == 48) { tgo(lag_tma_kernel<7, 48, false>); launched = true; }
          else if (g.l1 == 9 && tcb == 52) { tgo(lag_tma_kernel<9, 52, false>); launched = true; }
        }
      }
    }
    if (launched) {
    } else if (g.l1 == 3 && tcv == 37) go(lag_zone_kernel<3, 37, LAG_F32>);
    else if (g.l1 == 5 && tcv == 40) go(lag_zone_kernel<5, 40, LAG_F32>);
    else if (g.l1 == 7 && tcv == 46) go(lag_zone_kernel<7, 46, LAG_F32>);
    else if (g.l1 == 9 && tcv == 49) go(lag_zone_kernel<9, 49, LAG_F32>);
    else switch (g.l1) {
#define DDCCA_LAG_CASE(N) \
  case N:                 \
    go(lag_zone_kernel<N, 0, LAG_F32>); \
    break;
      DDCCA_LAG_CASE(1) DDCCA_LAG_CASE(2) DDCCA_LAG_CASE(3) DDCCA_LAG_CASE(4) DDCCA_LAG_CASE(5)
      DDCCA_LAG_CASE(6) DDCCA_LAG_CASE(7) DDCCA_LAG_CASE(8) DDCCA_LAG_CASE(9) DDCCA_LAG_CASE(10)
      DDCCA_LAG_CASE(11) DDCCA_LAG_CASE(12)
#undef DDCCA_LAG_CASE
      default:
        return fail(DDCCA_ECONFIG, "unsupported window height %d", g.l1);
    }
    DDCCA_TRY(check_launch("moments: lag_zone_kernel"));
    double* Z = reinterpret_cast<double*>(w + L.off_Z);
    {
      dim3 gz((unsigned)std::min<int64_t>(64, ((int64_t)nzone * P.NDF + 255) / 256), (unsigned)(n_batches * 2));
      zone_reduce_kernel<<<gz, 256, 0, st>>>(A.rec, reinterpret_cast<const int*>(w + L.off_zoff),
                                             reinterpret_cast<const int*>(w + L.off_zlist), Z, nzone, P.NDF, P.nrec,
                                             L.nsplit);
      DDCCA_TRY(check_launch("moments: zone_reduce"));
    }
    {
      AsmArgs S;
      S.Z = Z; S.rz_lo = rz_lo; S.rz_hi = rz_hi; S.cz_lo = cz_lo; S.cz_hi = cz_hi;
      S.payload = partials; S.plen = plen; S.nrz = P.nrz; S.ncz = P.ncz; S.NDX = P.NDX; S.NDF = P.NDF;
      S.l1 = g.l1; S.l2 = g.l2; S.d = g.d; S.center = center;
      const size_t sm = sizeof(double) * ((size_t)g.d * g.d + g.d);
      cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      assemble_kernel<<<n_batches * 2, 256, sm, st>>>(S);
      DDCCA_TRY(check_launch("moments: assemble"));
    }
    {
      RectArgs R;
      R.maps[0] = maps1; R.maps[1] = maps2;
      R.out = reinterpret_cast<double*>(w + L.off_msum);
      R.rz_y0 = rz_y0; R.cz_of_x = cz_of_x; R.a_rz = a_rz; R.b_cz = b_cz;
      R.n_maps = n_maps; R.p = g.p; R.q = g.q; R.top = g.top; R.left = g.left; R.Hp = g.Hp; R.Wp = g.Wp;
      R.nrz = P.nrz; R.ncz = P.ncz; R.l1 = g.l1; R.l2 = g.l2; R.d = g.d; R.center = center;
      R.big_cz = P.z.big_cz;
      if (g.q > 32 * RS_COLS) return fail(DDCCA_ECONFIG, "moments: maps wider than %d columns", 32 * RS_COLS);
      const size_t sm = sizeof(double) * RS_WARPS * ((size_t)P.nrz * P.ncz + g.d);
      const dim3 rgrid((unsigned)((n_maps + RS_WARPS - 1) / RS_WARPS), 2);
      if (g.q % 4 == 0 && g.q <= 128) {
        cudaFuncSetAttribute(rect_sums_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        rect_sums_kernel<true><<<rgrid, RS_WARPS * 32, sm, st>>>(R);
      } else {
        cudaFuncSetAttribute(rect_sums_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        rect_sums_kernel<false><<<rgrid, RS_WARPS * 32, sm, st>>>(R);
      }
      DDCCA_TRY(check_launch("moments: rect_sums"));
      batch_epilogue_kernel<<<dim3(n_batches, 2), 128, epi_smem(g.d, class_count), st>>>(R.out, map_label, A.batch_off, n_maps, g.d,
                                                                 class_count, plen, cols_per_map, partials);
      DDCCA_TRY(check_launch("moments: batch_epilogue"));
    }
    return DDCCA_OK;
  }

  // direct float64 path for stride != 1 (or very tall windows)
  const int64_t per_maps = split_maps(max_maps, flags);
  const int nsplit = nsplit_for(max_maps, per_maps);
  size_t o_rec = 0;
  size_t o_boff = align_up(sizeof(double) * (size_t)n_batches * 2 * nsplit * g.d * g.d, 256);
  size_t o_msum = o_boff + align_up(sizeof(int64_t) * (n_batches + 1), 256);
  size_t need = o_msum + align_up(sizeof(double) * 2 * (size_t)n_maps * g.d, 256);
  if (ws_bytes < need) return fail(DDCCA_ECONFIG, "moments workspace too small (%zu < %zu)", ws_bytes, need);
  double* rec = reinterpret_cast<double*>(w + o_rec);
  int64_t* boff = reinterpret_cast<int64_t*>(w + o_boff);
  double* msum = reinterpret_cast<double*>(w + o_msum);
  {
    const Upload boff_part{batch_offsets_host, sizeof(int64_t) * (n_batches + 1), boff};
    DDCCA_TRY(upload_parts(&boff_part, 1, st));
  }
  const size_t sm = sizeof(double) * DIRECT_K * g.d;
  cudaFuncSetAttribute(direct_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  direct_gram_kernel<<<dim3(nsplit, n_batches, 2), 256, sm, st>>>(maps1, maps2, boff, g, center, nsplit,
                                                                    per_maps * g.oh * g.ow, rec);
  DDCCA_TRY(check_launch("moments: direct_gram"));
  direct_reduce_kernel<<<n_batches * 2, 256, 0, st>>>(rec, nsplit, g.d, plen, partials);
  DDCCA_TRY(check_launch("moments: direct_reduce"));
  direct_map_sums_kernel<<<dim3((unsigned)n_maps, 2), 128, sizeof(double) * g.d, st>>>(maps1, maps2, n_maps, g, center,
                                                                                      msum);
  DDCCA_TRY(check_launch("moments: direct_map_sums"));
  batch_epilogue_kernel<<<dim3(n_batches, 2), 128, epi_smem(g.d, class_count), st>>>(msum, map_label, boff, n_maps, g.d, class_count, plen,
                                                             cols_per_map, partials);
  return check_launch("moments: batch_epilogue");
}

int ddcca_moments_tree(double* parts, int n_parts, int64_t payload_len_, double* out, void* stream) {
  if (n_parts < 1) return fail(DDCCA_ECONFIG, "nothing to merge");
  cudaStream_t st = as_stream(stream);
  // Level k combines entries spaced 2^k apart; an odd tail is carried unchanged,
  // which is exactly the left-to-right tree of pairwise_merge (moments.py:132-144).
  int n = n_parts, stride = 1;
  while (n > 1) {
    const int npairs = n / 2;
    const int64_t work = (int64_t)npairs * payload_len_;
    const int blocks = (int)std::min<int64_t>(4096, (work + 255) / 256);
    tree_level_kernel<<<blocks, 256, 0, st>>>(parts, n, payload_len_, stride);
    DDCCA_TRY(check_launch("moments: tree level"));
    // carried tail: element n-1 (odd) moves to position npairs in the next level,
    // i.e. index (n-1)*stride stays where it is and next level stride doubles;
    // with the in-place scheme next-level entry j lives at j * 2*stride, and the
    // tail at (n-1)*stride == npairs * 2*stride, so nothing needs to move.
    n = (n + 1) / 2;
    stride *= 2;
  }
  if (out != parts)
    cudaMemcpyAsync(out, parts, sizeof(double) * payload_len_, cudaMemcpyDeviceToDevice, st);
  return check_launch("moments: tree copy");
}

int ddcca_accumulate_columns(const double* x, const double* y, const int64_t* labels, int64_t cols, int dim,
                             int class_count, double* payload, void* stream) {
  if (dim < 1 || class_count < 1) return fail(DDCCA_ECONFIG, "invalid accumulator shape dim=%d classes=%d", dim, class_count);
  if (cols < 0) return fail(DDCCA_ESHAPE, "negative column count");
  if (cols == 0) return DDCCA_OK;
  if (dim * dim > 1 << 16) return fail(DDCCA_ECONFIG, "dim %d too large", dim);
  cudaStream_t st = as_stream(stream);
  const int nblk = (int)((cols + COLS_PER_BLOCK - 1) / COLS_PER_BLOCK);
  const int64_t per_view = (int64_t)dim * dim + (int64_t)dim * class_count + dim;
  double* part = nullptr;
  if (cudaMallocAsync(&part, sizeof(double) * (size_t)nblk * 2 * per_view, st) != cudaSuccess)
    return fail(DDCCA_ECUDA, "accumulate_columns: out of memory");
  const size_t sm = sizeof(double) * DIRECT_K * dim;
  cudaFuncSetAttribute(columns_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  columns_partial_kernel<<<nblk, 256, sm, st>>>(x, y, labels, cols, dim, class_count, part);
  int rc = check_launch("accumulate_columns: partial");
  if (rc == DDCCA_OK) {
    columns_reduce_kernel<<<1, 256, 0, st>>>(part, nblk, labels, cols, dim, class_count, payload);
    rc = check_launch("accumulate_columns: reduce");
  }
  cudaFreeAsync(part, st);
  return rc;
}

}  // extern "C"
