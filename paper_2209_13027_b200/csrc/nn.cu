// Nearest-neighbour classifier (classify.py:109-143 of the reference): for every
// query row, the training row at the smallest squared euclidean distance
// (q2 + t2 - 2 q.t, classify.py:113-115) or cosine distance (1 - q.t/(|q||t|),
// 0 similarity when a norm is zero, classify.py:116-120); ties go to the lowest
// class id (classify.py:136-138).
//
// B200 form: a float64 DFMA GEMM that never materializes the distance matrix.
// Rows are float64 feature vectors, or the integer block counts the transform
// keeps in HBM, expanded through the IQ LUT while a tile is staged (u8/u16 in
// HBM, float64 only in shared memory). Each CTA owns a 64 x 64 (query x train)
// tile over the full feature dimension and reduces its rows to a (distance,
// label) candidate per query; a second kernel takes the lexicographic minimum
// over the train tiles, which is exactly "lowest label among the rows at the
// minimum distance", independent of tile order.
#include <algorithm>
#include <cfloat>

#include "common.cuh"

namespace ddcca {

constexpr int NN_T = 128;       // query / train rows per tile
constexpr int NN_K = 16;        // features per stage
constexpr int NN_THREADS = 256; // 16 x 16 threads, 8 x 8 outputs each

template <int KIND>
__device__ __forceinline__ double nn_elem(const void* rows, int64_t idx, const double* lut) {
  if (KIND == 0) return lut[static_cast<const uint8_t*>(rows)[idx]];
  if (KIND == 2) return lut[static_cast<const uint16_t*>(rows)[idx]];
  return static_cast<const double*>(rows)[idx];
}

// Row norms: sq[i] = sum f^2 (euclidean) or sqrt of it (cosine).
template <int KIND>
__global__ void nn_norms_kernel(const void* rows, int64_t n, int64_t dim, const double* __restrict__ lut_g, int lut_len,
                                int take_sqrt, double* __restrict__ out) {
  extern __shared__ double lut[];
  if (KIND != 3)
    for (int i = threadIdx.x; i < lut_len; i += blockDim.x) lut[i] = lut_g[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + warp; r < n; r += (int64_t)gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int64_t f = lane; f < dim; f += 32) {
      const double v = nn_elem<KIND>(rows, r * dim + f, lut);
      s = fma(v, v, s);
    }
    s = warp_sum(s);
    if (lane == 0) out[r] = take_sqrt ? sqrt(s) : s;
  }
}

struct NnCand {
  double dist;
  int64_t label;
};

__device__ __forceinline__ bool nn_better(double d, int64_t l, double bd, int64_t bl) {
  return d < bd || (d == bd && l < bl);
}

// One row's NN_K features [k0, k0 + NN_K) held in registers between stages:
// integer counts for KIND 0 / 2, float64 values for KIND 3; zeros outside the matrix.
template <int KIND>
struct NnRaw {
  unsigned c[KIND == 3 ? 1 : NN_K];
  double d[KIND == 3 ? NN_K : 1];
};

template <int KIND>
__device__ __forceinline__ void nn_fetch(const void* rows, int64_t n, int64_t dim, int64_t row, int64_t k0,
                                         NnRaw<KIND>& raw) {
  constexpr int ES = KIND == 0 ? 1 : (KIND == 2 ? 2 : 8);
  const bool full = row < n && k0 + NN_K <= dim && ((dim * ES) & 15) == 0;
  const char* base = static_cast<const char*>(rows) + (row * dim + k0) * ES;
  if (full) {
    const uint4* src = reinterpret_cast<const uint4*>(base);
    if (KIND == 0) {
      const uint4 v = __ldg(src);
      const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < NN_K; ++k) raw.c[k] = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
    } else if (KIND == 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 v = __ldg(src + h);
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) raw.c[8 * h + k] = (w[k >> 1] >> (16 * (k & 1))) & 0xffffu;
      }
    } else {
#pragma unroll
      for (int k = 0; k < NN_K; ++k) raw.d[k] = __ldg(reinterpret_cast<const double*>(base) + k);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < NN_K; ++k) {
    const bool in = row < n && k0 + k < dim;
    if (KIND == 0) raw.c[k] = in ? static_cast<const uint8_t*>(rows)[row * dim + k0 + k] : 0u;
    else if (KIND == 2) raw.c[k] = in ? static_cast<const uint16_t*>(rows)[row * dim + k0 + k] : 0u;
    else raw.d[k] = in ? static_cast<const double*>(rows)[row * dim + k0 + k] : 0.0;
  }
}

template <int KIND>
__device__ __forceinline__ void nn_store(const NnRaw<KIND>& raw, const double* lut, double (*dst)[NN_T + 2], int r,
                                         bool live, int64_t kvalid) {
  // out-of-range rows / features hold count 0 -> lut[0]; force exact zeros for them
#pragma unroll
  for (int k = 0; k < NN_K; ++k) {
    double v;
    if (KIND == 0) v = lut[raw.c[k]];
    else if (KIND == 2) v = __ldg(lut + raw.c[k]);
    else v = raw.d[k];
    dst[k][r] = (live && k < kvalid) ? v : 0.0;
  }
}

// One CTA = NN_T queries x NN_T training rows over the whole feature dimension,
// 8 x 8 outputs per thread (rows ty*2 + {0,1} + 32 i, columns tx*2 + {0,1} + 32 j),
// double-buffered shared tiles filled from registers fetched one stage ahead.
template <int KIND>
__global__ void __launch_bounds__(NN_THREADS, 1)
    nn_tile_kernel(const void* query, int64_t nq, const void* train, int64_t nt, int64_t dim,
                   const double* __restrict__ lut_g, int lut_len, const double* __restrict__ qn,
                   const double* __restrict__ tn, const int64_t* __restrict__ labels, int metric,
                   NnCand* __restrict__ cand) {
  extern __shared__ __align__(16) double nn_sm[];
  double (*As)[NN_T + 2] = reinterpret_cast<double (*)[NN_T + 2]>(nn_sm);                  // [2][NN_K][NN_T+2]
  double (*Bs)[NN_T + 2] = reinterpret_cast<double (*)[NN_T + 2]>(nn_sm + 2 * NN_K * (NN_T + 2));
  double* lut = nn_sm + 4 * NN_K * (NN_T + 2);
  const double* L = lut_g;
  if (KIND == 0) {
    for (int i = threadIdx.x; i < lut_len; i += NN_THREADS) lut[i] = lut_g[i];
    L = lut;
  }
  const int64_t q0 = (int64_t)blockIdx.y * NN_T, t0 = (int64_t)blockIdx.x * NN_T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  // staging roles: threads 0..127 fetch query rows, 128..255 training rows
  const bool stage_q = threadIdx.x < NN_T;
  const int srow = threadIdx.x & (NN_T - 1);
  const void* src = stage_q ? query : train;
  const int64_t sn = stage_q ? nq : nt, sr = (stage_q ? q0 : t0) + srow;
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  NnRaw<KIND> raw;
  nn_fetch<KIND>(src, sn, dim, sr, 0, raw);
  __syncthreads();  // LUT in shared memory
  nn_store<KIND>(raw, L, (stage_q ? As : Bs), srow, sr < sn, dim);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < dim; k0 += NN_K) {
    const bool more = k0 + NN_K < dim;
    if (more) nn_fetch<KIND>(src, sn, dim, sr, k0 + NN_K, raw);  // next stage, in flight during the math
    const double (*A)[NN_T + 2] = As + buf * NN_K;
    const double (*B)[NN_T + 2] = Bs + buf * NN_K;
#pragma unroll 4
    for (int k = 0; k < NN_K; ++k) {
      double a[8], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 va = *reinterpret_cast<const double2*>(&A[k][ty * 2 + 32 * i]);
        const double2 vb = *reinterpret_cast<const double2*>(&B[k][tx * 2 + 32 * i]);
        a[2 * i] = va.x;
        a[2 * i + 1] = va.y;
        b[2 * i] = vb.x;
        b[2 * i + 1] = vb.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (more) nn_store<KIND>(raw, L, (stage_q ? As : Bs) + (buf ^ 1) * NN_K, srow, sr < sn, dim - (k0 + NN_K));
    __syncthreads();
    buf ^= 1;
  }
  // distances and the per-row candidate of this tile
  NnCand* red = reinterpret_cast<NnCand*>(nn_sm);  // [NN_T][16], aliases the staging tiles
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rl = ty * 2 + (i & 1) + 32 * (i >> 1);
    const int64_t qi = q0 + rl;
    double bd = DBL_MAX;
    int64_t bl = INT64_MAX;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t tj = t0 + tx * 2 + (j & 1) + 32 * (j >> 1);
      if (qi >= nq || tj >= nt) continue;
      double d;
      if (metric == 0) {
        d = (qn[qi] + tn[tj]) - 2.0 * acc[i][j];
      } else if (metric == 2) {
        d = -(acc[i][j] + tn[tj]);  // linear scores (ridge): tn = bias, best = largest score
      } else {
        const double den = qn[qi] * tn[tj];
        d = 1.0 - (den > 0.0 ? acc[i][j] / den : 0.0);
      }
      const int64_t l = labels[tj];
      if (nn_better(d, l, bd, bl)) { bd = d; bl = l; }
    }
    red[rl * 16 + tx] = {bd, bl};
  }
  __syncthreads();
  if (threadIdx.x < NN_T) {
    const int r = threadIdx.x;
    double bd = DBL_MAX;
    int64_t bl = INT64_MAX;
    for (int c = 0; c < 16; ++c) {
      const NnCand x = red[r * 16 + c];
      if (nn_better(x.dist, x.label, bd, bl)) { bd = x.dist; bl = x.label; }
    }
    if (q0 + r < nq) cand[(q0 + r) * gridDim.x + blockIdx.x] = {bd, bl};
  }
}

static size_t nn_smem(int kind, int lut_len) {
  return sizeof(double) * (4 * (size_t)NN_K * (NN_T + 2) + (kind == 0 ? (size_t)lut_len : 0));
}

__global__ void nn_reduce_kernel(const NnCand* __restrict__ cand, int64_t nq, int ntiles, int64_t* __restrict__ pred) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    double bd = DBL_MAX;
    int64_t bl = INT64_MAX;
    for (int t = 0; t < ntiles; ++t) {
      const NnCand c = cand[q * ntiles + t];
      if (nn_better(c.dist, c.label, bd, bl)) { bd = c.dist; bl = c.label; }
    }
    pred[q] = bl;
  }
}

// Saturating-u8 block counts -> exact u16 (the 255 sentinel is the block remainder).
__global__ void counts_u16_kernel(const uint8_t* __restrict__ in, int64_t n_blocks, int bins, int bpc,
                                  uint16_t* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + warp; b < n_blocks;
       b += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const uint8_t* src = in + b * bins;
    int s = 0;
    for (int k = lane; k < bins; k += 32) s += src[k];
    s = (int)warp_sum((double)s);
    for (int k = lane; k < bins; k += 32) {
      const int c = src[k];
      out[b * bins + k] = (uint16_t)(c == 255 ? 255 + (bpc - s) : c);
    }
  }
}

static size_t nn_cand_bytes(int64_t nq, int64_t nt) {
  return sizeof(NnCand) * (size_t)nq * (size_t)((nt + NN_T - 1) / NN_T);
}

template <int KIND>
static int nn_run(const void* q, int64_t nq, const void* t, int64_t nt, int64_t dim, const double* lut, int lut_len,
                  const int64_t* labels, int metric, int64_t* pred, void* ws, cudaStream_t st,
                  const double* bias = nullptr) {
  double* qn = static_cast<double*>(ws);
  double* tn = qn + nq;
  NnCand* cand = reinterpret_cast<NnCand*>(tn + nt + (((nq + nt) & 1) ? 1 : 0));
  const size_t lsm = KIND == 3 ? 0 : sizeof(double) * (size_t)lut_len;
  const int nb = (int)std::min<int64_t>((std::max(nq, nt) + 7) / 8, 148 * 8);
  if (metric == 2) {
    cudaMemcpyAsync(tn, bias, sizeof(double) * nt, cudaMemcpyDeviceToDevice, st);
  } else {
    nn_norms_kernel<KIND><<<nb, 256, lsm, st>>>(q, nq, dim, lut, lut_len, metric == 1, qn);
    nn_norms_kernel<KIND><<<nb, 256, lsm, st>>>(t, nt, dim, lut, lut_len, metric == 1, tn);
  }
  DDCCA_TRY(check_launch("nn_norms"));
  const int ntiles = (int)((nt + NN_T - 1) / NN_T);
  const int64_t qtiles = (nq + NN_T - 1) / NN_T;
  if (qtiles > 65535) return fail(DDCCA_ECONFIG, "nn: %lld query rows exceed one launch", (long long)nq);
  const size_t sm = nn_smem(KIND, lut_len);
  cudaFuncSetAttribute(nn_tile_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  nn_tile_kernel<KIND><<<dim3(ntiles, (unsigned)qtiles), NN_THREADS, sm, st>>>(q, nq, t, nt, dim, lut, lut_len, qn,
                                                                              tn, labels, metric, cand);
  DDCCA_TRY(check_launch("nn_tile"));
  nn_reduce_kernel<<<(int)std::min<int64_t>((nq + 255) / 256, 4096), 256, 0, st>>>(cand, nq, ntiles, pred);
  return check_launch("nn_reduce");
}

}  // namespace ddcca

using namespace ddcca;

extern "C" {

size_t ddcca_nn_workspace(int64_t n_query, int64_t n_train) {
  return sizeof(double) * (size_t)(n_query + n_train + 1) + nn_cand_bytes(n_query, n_train) + 64;
}

int ddcca_nn_classify(const void* query, int64_t n_query, const void* train, int64_t n_train, int64_t dim,
                      int row_kind, const double* lut, int lut_len, const int64_t* train_labels, int metric,
                      int64_t* pred, void* workspace, size_t ws_bytes, void* stream) {
  if (n_query < 0 || n_train < 1 || dim < 1) return fail(DDCCA_ESHAPE, "nn: empty training set or feature dim");
  if (metric != 0 && metric != 1) return fail(DDCCA_ECONFIG, "nn: metric %d not euclidean(0)/cosine(1)", metric);
  if (n_query == 0) return DDCCA_OK;
  if (ws_bytes < ddcca_nn_workspace(n_query, n_train)) return fail(DDCCA_ESHAPE, "nn: workspace too small");
  cudaStream_t st = as_stream(stream);
  switch (row_kind) {
    case 0:
      if (!lut || lut_len < 1 || lut_len > 256) return fail(DDCCA_ESHAPE, "nn: u8 rows need a LUT of <= 256 values");
      return nn_run<0>(query, n_query, train, n_train, dim, lut, lut_len, train_labels, metric, pred, workspace, st);
    case 2:
      if (!lut || lut_len < 1) return fail(DDCCA_ESHAPE, "nn: u16 rows need a LUT");
      return nn_run<2>(query, n_query, train, n_train, dim, lut, lut_len, train_labels, metric, pred, workspace, st);
    case 3:
      return nn_run<3>(query, n_query, train, n_train, dim, nullptr, 0, train_labels, metric, pred, workspace, st);
    default:
      return fail(DDCCA_ECONFIG, "nn: row kind %d not u8(0)/u16(2)/f64(3)", row_kind);
  }
}

// Linear one-vs-all prediction (classify.py:140-142): pred = argmax_c (x . w_c + b_c), the
// first maximum on ties -> the lowest class id, as (-score, class) minima through the same
// tiled float64 GEMM. query (nq x dim) and weights (n_class x dim) are float64 rows.
int ddcca_linear_classify(const double* query, int64_t n_query, const double* weights, int64_t n_class, int64_t dim,
                          const double* bias, const int64_t* class_ids, int64_t* pred, void* workspace,
                          size_t ws_bytes, void* stream) {
  if (n_query < 0 || n_class < 1 || dim < 1) return fail(DDCCA_ESHAPE, "linear: empty weights or feature dim");
  if (!weights || !bias || !class_ids) return fail(DDCCA_ESHAPE, "linear: null pointer");
  if (n_query == 0) return DDCCA_OK;
  if (ws_bytes < ddcca_nn_workspace(n_query, n_class)) return fail(DDCCA_ESHAPE, "linear: workspace too small");
  return nn_run<3>(query, n_query, weights, n_class, dim, nullptr, 0, class_ids, 2, pred, workspace, as_stream(stream),
                   bias);
}

int ddcca_counts_to_u16(const uint8_t* counts, int64_t n_blocks, int bins, int bpc, uint16_t* out, void* stream) {
  if (n_blocks < 0 || bins < 1 || bpc < 1 || bpc > 65535) return fail(DDCCA_ESHAPE, "counts_to_u16: bad shape");
  if (n_blocks == 0) return DDCCA_OK;
  const int grid = (int)std::min<int64_t>((n_blocks + 7) / 8, 148 * 16);
  counts_u16_kernel<<<grid, 256, 0, as_stream(stream)>>>(counts, n_blocks, bins, bpc, out);
  return check_launch("counts_to_u16");
}

}  // extern "C"
