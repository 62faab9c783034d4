// Shared helpers for the ddcca CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstdarg>
#include <cstring>

#include "../../include/ddcca.h"

namespace ddcca {

// Thread-local last-error message (ddcca_last_error).
inline char* err_buf() {
  static thread_local char buf[512];
  return buf;
}

inline int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err_buf(), 512, fmt, ap);
  va_end(ap);
  return code;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DDCCA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return DDCCA_OK;
}

#define DDCCA_TRY(expr)            \
  do {                             \
    int _rc = (expr);              \
    if (_rc != DDCCA_OK) return _rc; \
  } while (0)

struct Geo {
  int p, q, l1, l2, stride, zero_same;
  int oh, ow, top, bottom, left, right;
  int Hp, Wp;  // padded domain
  int d;
};

// Restates PatchGeometry.out_shape / pad_amounts (patches.py:41-65).
inline int make_geo(const ddcca_geom* g, Geo* o) {
  if (!g) return fail(DDCCA_ECONFIG, "null geometry");
  if (g->l1 < 1 || g->l2 < 1) return fail(DDCCA_ECONFIG, "patch size %dx%d must be at least 1x1", g->l1, g->l2);
  if (g->stride < 1) return fail(DDCCA_ECONFIG, "stride %d must be >= 1", g->stride);
  if (g->p < 1 || g->q < 1) return fail(DDCCA_ESHAPE, "empty map %dx%d", g->p, g->q);
  o->p = g->p; o->q = g->q; o->l1 = g->l1; o->l2 = g->l2; o->stride = g->stride; o->zero_same = g->zero_same;
  o->d = g->l1 * g->l2;
  if (g->zero_same) {
    o->oh = (g->p + g->stride - 1) / g->stride;
    o->ow = (g->q + g->stride - 1) / g->stride;
    o->top = (g->l1 - 1) / 2;
    o->left = (g->l2 - 1) / 2;
    int b = (o->oh - 1) * g->stride + g->l1 - g->p - o->top;
    int r = (o->ow - 1) * g->stride + g->l2 - g->q - o->left;
    o->bottom = b > 0 ? b : 0;
    o->right = r > 0 ? r : 0;
  } else {
    if (g->p < g->l1 || g->q < g->l2)
      return fail(DDCCA_ESHAPE, "%dx%d window does not fit a %dx%d map without padding", g->l1, g->l2, g->p, g->q);
    o->oh = (g->p - g->l1) / g->stride + 1;
    o->ow = (g->q - g->l2) / g->stride + 1;
    o->top = o->bottom = o->left = o->right = 0;
  }
  o->Hp = g->p + o->top + o->bottom;
  o->Wp = g->q + o->left + o->right;
  return DDCCA_OK;
}

__host__ __device__ inline int64_t payload_len(int d, int C) { return 2LL * d * d + 2LL * d * C + 2LL * d + 1 + C; }

struct PayloadView {
  int64_t c11, c22, s1, s2, g1, g2, n, ncls, len;
};
__host__ __device__ inline PayloadView payload_view(int d, int C) {
  PayloadView v;
  v.c11 = 0;
  v.c22 = (int64_t)d * d;
  v.s1 = 2LL * d * d;
  v.s2 = v.s1 + (int64_t)d * C;
  v.g1 = v.s2 + (int64_t)d * C;
  v.g2 = v.g1 + d;
  v.n = v.g2 + d;
  v.ncls = v.n + 1;
  v.len = v.ncls + C;
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Host -> device upload of a call's small plan tables (tens of KB). Deliberately from
// pageable memory: the driver sends copies this small inline through the stream's own
// channel, while a pinned-memory copy is a copy-engine DMA that queues behind whatever
// bulk transfer is in flight (the image upload of an end-to-end run: measured 334 vs
// 348 ms per Caltech e2e step with a pinned staging ring).
struct Upload {
  const void* src;
  size_t bytes;
  void* dst;
};
inline int upload_parts(const Upload* parts, int n, cudaStream_t st) {
  for (int i = 0; i < n; ++i)
    if (parts[i].bytes) cudaMemcpyAsync(parts[i].dst, parts[i].src, parts[i].bytes, cudaMemcpyHostToDevice, st);
  return check_launch("plan upload");
}

}  // namespace ddcca
