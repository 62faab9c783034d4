// K4+K5: finalize + DCCA filter solve on device, one CTA, float64.
//
// Restates moments.finalize (moments.py:168-193) and solver.solve_dcca /
// sym_eig / inv_sqrt / reshape_filters (solver.py:32-272) including the
// reference's ordering semantics: cyclic Jacobi with the round-robin pair
// schedule (solver.py:32-46), unit-Frobenius pre-scaling, 1e-12 off-diagonal
// stop, 100-sweep cap, stable descending sort, largest-|entry|-positive sign
// rule (solver.py:49-57), lexicographic order inside near-degenerate runs
// (solver.py:60-79), and null-space completion for sigma <= 1e-12 sigma_1
// (solver.py:238-247). The problem is d x d with d = l1*l2 <= ~100, so one
// CTA with the Jacobi matrices in shared memory is the right shape: the
// solve is latency-bound (a few hundred rotation rounds), not FLOP-bound.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace ddcca {

constexpr int SOLVE_THREADS = 1024;  // latency-bound rounds: more warps per rotation pass

#ifdef DDCCA_SOLVE_PROF  // diagnostic build only (tools/microbench/jacobi_probe.cu)
__device__ unsigned long long g_solve_prof[8];
#define PROF_MARK(t) const long long t = clock64()
#define PROF_ADD(k, t0) do { if (threadIdx.x == 0) g_solve_prof[k] += clock64() - (t0); } while (0)
#define PROF_COUNT_SWEEP() do { if (threadIdx.x == 0) g_solve_prof[7] += 1; } while (0)
#else
#define PROF_MARK(t)
#define PROF_ADD(k, t0)
#define PROF_COUNT_SWEEP()
#endif
constexpr int SMEM_JACOBI_MAX_N = 110;  // 2*n*n doubles in shared memory

struct Blk {
  double* red;   // reduction scratch, SOLVE_THREADS doubles (shared)
  int* flag;     // shared error flag
  int* iscr;     // shared int scratch, >= 2*n ints
};

__device__ double block_sum(double v, Blk& B) {
  const int t = threadIdx.x;
  v = warp_sum(v);
  __syncthreads();
  if ((t & 31) == 0) B.red[t >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (t < 32) {
    s = (t < (int)(blockDim.x >> 5)) ? B.red[t] : 0.0;
    s = warp_sum(s);
    if (t == 0) B.red[0] = s;
  }
  __syncthreads();
  s = B.red[0];
  __syncthreads();
  return s;
}

__device__ double block_max(double v, Blk& B) {
  const int t = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((t & 31) == 0) B.red[t >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (t < 32) {
    s = (t < (int)(blockDim.x >> 5)) ? B.red[t] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (t == 0) B.red[0] = s;
  }
  __syncthreads();
  s = B.red[0];
  __syncthreads();
  return s;
}

__device__ double offdiag_norm(const double* a, int n, Blk& B) {
  double s = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    if (i != j) s += a[e] * a[e];
  }
  return sqrt(block_sum(s, B));
}

// seat of position k in round r of the round-robin tournament (solver.py:32-46)
__device__ __forceinline__ int rr_seat(int k, int r, int m) {
  if (k == 0) return 0;
  int v = (k - 1 - r) % (m - 1);
  if (v < 0) v += m - 1;
  return v + 1;
}

// argsort(-w, kind="stable"): rank of element i
__device__ __forceinline__ int desc_rank(const double* w, int n, int i) {
  const double wi = w[i];
  int r = 0;
  for (int j = 0; j < n; ++j) {
    const double wj = w[j];
    if (wj > wi || (wj == wi && j < i)) ++r;
  }
  return r;
}

// Sign per column: largest |entry| (first on ties) made positive (solver.py:49-57).
__device__ void col_signs(const double* v, int n, int ncols, int ld, double* sgn) {
  for (int j = threadIdx.x; j < ncols; j += blockDim.x) {
    int best = 0;
    double bv = fabs(v[j]);
    for (int i = 1; i < n; ++i) {
      const double x = fabs(v[i * ld + j]);
      if (x > bv) { bv = x; best = i; }
    }
    const double e = v[best * ld + j];
    sgn[j] = e > 0.0 ? 1.0 : (e < 0.0 ? -1.0 : 1.0);
  }
}

// Lexicographic comparison of columns i and j of v (n rows, leading dim ld).
__device__ __forceinline__ int lex_cmp(const double* v, int n, int ld, int i, int j) {
  for (int k = 0; k < n; ++k) {
    const double a = v[k * ld + i], b = v[k * ld + j];
    if (a < b) return -1;
    if (a > b) return 1;
  }
  return 0;
}

// Stable descending sort of eigenvalues wtmp (unsorted, final scale) with their eigenvector
// columns va, the sign rule (solver.py:49-57) and the lexicographic order inside degenerate
// runs (solver.py:60-79) -> w, v. tmp: n x n scratch. Shared by every eigensolver form.
__device__ void eig_order(int n, double* wtmp, const double* va, double* w, double* v, double* tmp, Blk& B) {
  const int nn = n * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = desc_rank(wtmp, n, i);
    w[r] = wtmp[i];
    for (int k = 0; k < n; ++k) tmp[k * n + r] = va[k * n + i];
  }
  __syncthreads();
  // sign rule
  col_signs(tmp, n, n, n, wtmp);
  __syncthreads();
  for (int e = threadIdx.x; e < nn; e += blockDim.x) tmp[e] *= wtmp[e % n];
  __syncthreads();
  // degenerate runs: |w[k] - w[start]| <= 1e-10 * max|w|, sorted lexicographically
  int* run_start = B.iscr;  // n ints
  if (threadIdx.x == 0) {
    double sc = 0.0;
    for (int i = 0; i < n; ++i) sc = fmax(sc, fabs(w[i]));
    const double tol = 1e-10 * sc;
    int start = 0;
    for (int k = 1; k <= n; ++k) {
      if (k < n && fabs(w[k] - w[start]) <= tol) continue;
      for (int i = start; i < k; ++i) run_start[i] = start;
      start = k;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int st = run_start[i];
    int en = i + 1;
    while (en < n && run_start[en] == st) ++en;
    int r = st;
    for (int j = st; j < en; ++j) {
      if (j == i) continue;
      const int c = lex_cmp(tmp, n, n, j, i);
      if (c < 0 || (c == 0 && j < i)) ++r;
    }
    wtmp[r] = w[i];
    for (int k = 0; k < n; ++k) v[k * n + r] = tmp[k * n + i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = wtmp[i];
  __syncthreads();
}

// C = op(A) * op(B) for n x n row-major matrices (ta/tb: use transpose)
__device__ void matmul(const double* A, bool ta, const double* Bm, bool tb, double* C, int n, int kdim, int mcols) {
  // C (n x mcols) = A' (n x kdim) * B' (kdim x mcols)
  for (int e = threadIdx.x; e < n * mcols; e += blockDim.x) {
    const int i = e / mcols, j = e - i * mcols;
    double s = 0.0;
    for (int k = 0; k < kdim; ++k) {
      const double x = ta ? A[k * n + i] : A[i * kdim + k];
      const double y = tb ? Bm[j * kdim + k] : Bm[k * mcols + j];
      s += x * y;
    }
    C[e] = s;
  }
  __syncthreads();
}


// Symmetric eigensolver (solver.py:90-158). s: input n x n. Results: w (n),
// v (n x n row-major, column j = eigenvector j). The rotation working set
// (a, the accumulated rotations va, and the per-round (c, s) table cs) lives in
// shared memory; tmp / wtmp are global scratch for the final ordering.
// Returns a DDCCA_* status (uniform across the block).
__device__ int sym_eig_dev(const double* s, int n, double* w, double* v, double* a, double* va, double* cs,
                           double* tmp, double* wtmp, Blk& B) {
  const int nn = n * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double mx = 0.0;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) mx = fmax(mx, fabs(s[e]));
  mx = block_max(mx, B);
  if (n == 1 || mx == 0.0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) wtmp[i] = s[i * n + i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int r = desc_rank(wtmp, n, i);
      w[r] = wtmp[i];
      for (int k = 0; k < n; ++k) v[k * n + r] = (k == i) ? 1.0 : 0.0;
    }
    __syncthreads();
    return DDCCA_OK;
  }
  // unit-scaled copy, its Frobenius norm and the symmetry test
  double fs = 0.0, as = 0.0;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    const double u = s[e] / mx, ut = s[j * n + i] / mx;
    fs += u * u;
    as += (u - ut) * (u - ut);
  }
  const double fro_u = sqrt(block_sum(fs, B));
  const double asym = sqrt(block_sum(as, B));
  if (asym > 1e-10 * fro_u) return DDCCA_ESHAPE;
  const double norm = mx * fro_u;
  const double f = mx / norm;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    a[e] = 0.5 * (s[e] / mx + s[j * n + i] / mx) * f;
    va[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int m = n + (n & 1);
  const int npair = m / 2;
  int* pp = B.iscr;          // p of pair t
  int* qq = B.iscr + npair;  // q of pair t (or -1 if inactive / dummy)
  bool converged = false;
  PROF_MARK(t_start);
  for (int sweep = 0; sweep < 100; ++sweep) {
    PROF_MARK(t_off);
    if (offdiag_norm(a, n, B) <= 1e-12) { converged = true; break; }
    PROF_ADD(0, t_off);
    PROF_COUNT_SWEEP();
    // this thread's pair seats, advanced one seat per round (no integer modulo on the
    // round's critical path): rr_seat(k, r + 1) = rr_seat(k, r) - 1, wrapping 1 -> m - 1
    const bool own = (int)threadIdx.x < npair;
    int su = own ? rr_seat(threadIdx.x, 0, m) : 0, sx = own ? rr_seat(m - 1 - threadIdx.x, 0, m) : 0;
    for (int r = 0; r < m - 1; ++r) {
      PROF_MARK(t_round);
      for (int t = threadIdx.x; t < npair; t += blockDim.x) {
        const bool mine = t == (int)threadIdx.x;
        const int u = mine ? su : rr_seat(t, r, m), x = mine ? sx : rr_seat(m - 1 - t, r, m);
        int p = min(u, x), q = max(u, x);
        double c = 1.0, sn = 0.0;
        if (q < n) {
          const double apq = a[p * n + q];
          if (apq != 0.0) {
            // theta = (a_qq - a_pp) / (2 a_pq), t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)),
            // c = 1 / sqrt(t^2 + 1), s = t c (solver.py:32-46), i.e. the rotation by the smaller
            // angle phi with cos 2phi = |d| / rho, rho = sqrt(d^2 + (2 a_pq)^2). Evaluated as
            // c = sqrt(h), h = (1 + |d| / rho) / 2, s = sgn(theta) |2 a_pq| / (2 rho c): two
            // reciprocal square roots on the round's critical path, no division (no cancellation:
            // h is in [1/2, 1]).
            double dlt = a[q * n + q] - a[p * n + p];
            double two = 2.0 * apq;
            // h and s depend only on the ratio dlt : two; an exact power-of-two rescale keeps
            // dlt^2 + two^2 from underflowing when both are tiny (the reference's theta form
            // is scale-invariant). Never taken for entries above 2^-500: bits unchanged there.
            if (fmax(fabs(dlt), fabs(two)) < 0x1p-500) {
              dlt *= 0x1p+600;
              two *= 0x1p+600;
            }
            const double sg = ((dlt >= 0.0) == (two > 0.0)) || dlt == 0.0 ? 1.0 : -1.0;
            const double ri = rsqrt(fma(dlt, dlt, two * two));  // 1 / rho
            const double h = fma(0.5 * fabs(dlt), ri, 0.5);
            const double ci = rsqrt(h);                          // 1 / c
            c = h * ci;
            sn = sg * (0.5 * fabs(two)) * ri * ci;
          } else {
            q = -1;
          }
        } else {
          q = -1;
        }
        pp[t] = p;
        qq[t] = q;
        cs[2 * t] = c;
        cs[2 * t + 1] = sn;
      }
      if (own) {
        if (su != 0) su = su > 1 ? su - 1 : m - 1;  // seat 0 (k = 0) is fixed
        sx = sx > 1 ? sx - 1 : m - 1;
      }
      __syncthreads();
      PROF_ADD(1, t_round);
      PROF_MARK(t_upd);
      // rows: B = J^T a   (warp per pair, lanes over columns)
      for (int t = warp; t < npair; t += nwarps) {
        const int q = qq[t];
        if (q < 0) continue;
        const int p = pp[t];
        const double c = cs[2 * t], sn = cs[2 * t + 1];
        for (int j = lane; j < n; j += 32) {
          const double ap = a[p * n + j], aq = a[q * n + j];
          a[p * n + j] = c * ap - sn * aq;
          a[q * n + j] = sn * ap + c * aq;
        }
      }
      __syncthreads();
      // columns: a = B J, va = va J
      for (int t = warp; t < npair; t += nwarps) {
        const int q = qq[t];
        if (q < 0) continue;
        const int p = pp[t];
        const double c = cs[2 * t], sn = cs[2 * t + 1];
        for (int i = lane; i < n; i += 32) {
          const double bp = a[i * n + p], bq = a[i * n + q];
          a[i * n + p] = c * bp - sn * bq;
          a[i * n + q] = sn * bp + c * bq;
          const double vp = va[i * n + p], vq = va[i * n + q];
          va[i * n + p] = c * vp - sn * vq;
          va[i * n + q] = sn * vp + c * vq;
        }
      }
      __syncthreads();
      PROF_ADD(2, t_upd);
    }
    // a = (a + a^T) / 2
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      if (i < j) {
        const double x = 0.5 * (a[e] + a[j * n + i]);
        a[e] = x;
        a[j * n + i] = x;
      }
    }
    __syncthreads();
  }
  PROF_ADD(3, t_start);
  PROF_MARK(t_post);
  // written as !(x <= tol) so a NaN off-diagonal norm is reported, never returned as converged
  if (!converged && !(offdiag_norm(a, n, B) <= 1e-12)) return DDCCA_ENUMERICAL;
  // eigenvalues, stable descending order, sign rule, degenerate-run order
  for (int i = threadIdx.x; i < n; i += blockDim.x) wtmp[i] = a[i * n + i] * norm;
  __syncthreads();
  eig_order(n, wtmp, va, w, v, tmp, B);
  PROF_ADD(4, t_post);
  return DDCCA_OK;
}


// C = A B for dp x dp row-major matrices in shared memory (dp % 8 == 0), on the FP64 tensor
// path: one warp per 8 x 8 output tile, mma.sync m8n8k4 f64 over K (each product and sum in
// float64, like the FFMA form, at the DMMA pipe's rate instead of one load per DFMA).
__device__ void gemm_dmma(const double* __restrict__ A, const double* __restrict__ Bm, double* __restrict__ C,
                          int dp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = dp >> 3, r = lane >> 2, c4 = lane & 3;
  for (int t = warp; t < nt * nt; t += blockDim.x >> 5) {
    const int ti = t / nt, tj = t - ti * nt;
    // two independent accumulator pairs (k = 0, 8, .. and k = 4, 12, ..) halve the
    // dependent DMMA chain; dp % 8 == 0
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
    const double* arow = A + (ti * 8 + r) * dp + c4;  // A[8 ti + r][k + c4]
    const double* bcol = Bm + c4 * dp + tj * 8 + r;   // B[k + c4][8 tj + r]
#pragma unroll 2
    for (int k = 0; k < dp; k += 8) {
      const double a0 = arow[k], a1 = arow[k + 4];
      const double b0 = bcol[k * dp], b1 = bcol[(k + 4) * dp];
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
          : "+d"(d0), "+d"(d1)
          : "d"(a0), "d"(b0));
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
          : "+d"(e0), "+d"(e1)
          : "d"(a1), "d"(b1));
    }
    double* o = C + (ti * 8 + r) * dp + tj * 8 + 2 * c4;
    o[0] = d0 + e0;
    o[1] = d1 + e1;
  }
  __syncthreads();
}

constexpr int NS_MAX_DP = 64;    // coupled Newton-Schulz in shared memory up to 64 x 64 (padded)
constexpr int NS_MAX_ITERS = 100;

__host__ __device__ inline int ns_dp(int n) { return (n + 7) & ~7; }
__host__ __device__ inline size_t ns_smem_doubles(int n) {
  const size_t dp = (size_t)ns_dp(n);
  return dp <= (size_t)NS_MAX_DP ? 4 * dp * dp : 0;
}

// Symmetric inverse square root of an SPD matrix by the coupled Newton-Schulz iteration
// (Y0 = A / ||A||_F, Z0 = I; T = (3 I - Z Y) / 2, Y <- Y T, Z <- T Z; Z -> (A / ||A||_F)^-1/2),
// padded with an identity block to a multiple of 8 for the DMMA tiles. The result is the
// same matrix the reference's V diag(w^-1/2) V' (solver.py:161-170) computes, to rounding;
// returns false (the caller then runs the Jacobi form, which also reports non-PD input) when
// the iteration does not converge: not positive definite, or too ill-conditioned.
__device__ bool ns_inv_sqrt(const double* c, int n, double* r, double* buf, Blk& B) {
  const int dp = ns_dp(n), np = dp * dp;
  double *Y = buf, *Z = buf + np, *T = buf + 2 * np, *W = buf + 3 * np;
  double fro = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) fro += c[e] * c[e];
  fro = sqrt(block_sum(fro, B));
  if (!(fro > 0.0) || !isfinite(fro)) return false;
  const double inv = 1.0 / fro;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    const int i = e / dp, j = e - i * dp;
    Y[e] = (i < n && j < n) ? 0.5 * (c[i * n + j] + c[j * n + i]) * inv : (i == j ? 1.0 : 0.0);
    Z[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  int settled = 0;
  for (int it = 0; it < NS_MAX_ITERS; ++it) {
    gemm_dmma(Z, Y, T, dp);
    double err = 0.0;
    for (int e = threadIdx.x; e < np; e += blockDim.x) {
      const int i = e / dp, j = e - i * dp;
      const double t = (i == j ? 1.5 : 0.0) - 0.5 * T[e];
      T[e] = t;
      err = fmax(err, fabs(t - (i == j ? 1.0 : 0.0)));
    }
    err = block_max(err, B);  // includes the barrier before T is read
    gemm_dmma(Y, T, W, dp);
    double* x = Y; Y = W; W = x;
    gemm_dmma(T, Z, W, dp);
    x = Z; Z = W; W = x;
    if (!(err < 1e30)) return false;  // diverging: not positive definite
    // quadratic convergence: two more sweeps once the residual is small reach rounding level
    if (err < 1e-11 && ++settled >= 3) {
      const double s = rsqrt(fro);
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        r[e] = 0.5 * (Z[i * dp + j] + Z[j * dp + i]) * s;
      }
      __syncthreads();
      return true;
    }
  }
  return false;
}

// inv_sqrt (solver.py:161-170) into r; eigen scratch from the caller. nsbuf (shared memory,
// ns_smem_doubles(n)) enables the Newton-Schulz form; Jacobi otherwise or as its fallback.
__device__ int inv_sqrt_dev(const double* c, int n, double* r, double* w, double* v, double* a, double* va, double* cs,
                            double* tmp, double* wtmp, Blk& B, double* nsbuf = nullptr) {
  if (nsbuf != nullptr && ns_inv_sqrt(c, n, r, nsbuf, B)) return DDCCA_OK;
  int rc = sym_eig_dev(c, n, w, v, a, va, cs, tmp, wtmp, B);
  if (rc != DDCCA_OK) return rc;
  if (!(w[n - 1] > 0.0)) return DDCCA_ENUMERICAL;
  // w^-1/2 once per eigenvalue (the same pow values the per-term form would use)
  for (int k = threadIdx.x; k < n; k += blockDim.x) wtmp[k] = pow(w[k], -0.5);
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += (v[i * n + k] * wtmp[k]) * v[j * n + k];
    tmp[e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    r[e] = 0.5 * (tmp[e] + tmp[j * n + i]);
  }
  __syncthreads();
  return DDCCA_OK;
}

// finalize (moments.py:168-193): Cw = S1 S2^T, Cb = g1 g2^T - Cw, Ct = Cw - Cb,
// C11 = sym(C11) + eps * tr/d * I (same for C22). Returns false on an empty
// accumulator (NumericalError in the reference).
// Entries e0, e0 + es, ... of the d x d outputs are this thread's (one CTA: threadIdx.x /
// blockDim.x; the grid form spreads the C-term dot products over several CTAs). Every
// CTA evaluates the traces the same way, so the ridge terms do not depend on the grid.
__device__ bool finalize_dev(const double* P, int n, int C, double eps, double* fin, Blk& B, int e0, int es) {
  const PayloadView pv = payload_view(n, C);
  const int nn = n * n;
  double* c11 = fin;
  double* c22 = fin + nn;
  double* cw = fin + 2 * nn;
  double* cb = fin + 3 * nn;
  double* ct = fin + 4 * nn;
  if (!(P[pv.n] >= 1.0)) return false;
  for (int e = e0; e < nn; e += es) {
    const int i = e / n, j = e - i * n;
    const double* r1 = P + pv.s1 + (int64_t)i * C;
    const double* r2 = P + pv.s2 + (int64_t)j * C;
    double s = 0.0;
#pragma unroll 8
    for (int c = 0; c < C; ++c) s += r1[c] * r2[c];
    const double b = P[pv.g1 + i] * P[pv.g2 + j] - s;
    cw[e] = s;
    cb[e] = b;
    ct[e] = s - b;
  }
  double tr1 = 0.0, tr2 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    tr1 += 0.5 * (P[pv.c11 + i * n + i] + P[pv.c11 + i * n + i]);
    tr2 += 0.5 * (P[pv.c22 + i * n + i] + P[pv.c22 + i * n + i]);
  }
  tr1 = block_sum(tr1, B);
  tr2 = block_sum(tr2, B);
  const double rid1 = eps * (tr1 / n), rid2 = eps * (tr2 / n);
  for (int e = e0; e < nn; e += es) {
    const int i = e / n, j = e - i * n;
    c11[e] = 0.5 * (P[pv.c11 + e] + P[pv.c11 + j * n + i]) + (i == j ? rid1 : 0.0);
    c22[e] = 0.5 * (P[pv.c22 + e] + P[pv.c22 + j * n + i]) + (i == j ? rid2 : 0.0);
  }
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(SOLVE_THREADS) finalize_kernel(const double* P, int n, int C, double eps, double* fin,
                                                                 int32_t* status) {
  __shared__ double red[SOLVE_THREADS / 32 + 1];
  __shared__ int flag;
  __shared__ int iscr[2];
  Blk B{red, &flag, iscr};
  const bool ok = finalize_dev(P, n, C, eps, fin, B, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) *status = ok ? DDCCA_OK : DDCCA_ENUMERICAL;
}

// One output entry per thread: the C-term dot products are latency-bound chains.
static int finalize_grid(int n) { return (n * n + SOLVE_THREADS - 1) / SOLVE_THREADS; }

struct SolveArgs {
  const double* payload;
  int d, C, count;
  double eps;
  double *fin, *w1, *w2, *rho;
  float *pack1, *pack2;
  int32_t* status;
  double* ws;  // global scratch
  int jacobi_in_smem;
  int prewhitened;  // R1, R2 already computed by whiten_kernel (status checked first)
};

// Global scratch of one solve: [main Jacobi a/va (if not in smem)] [jtmp] R1 R2 T Gm U V NB ev
// lam wsc sig flip lam2, then per whitening CTA b in {0,1}: [a/va] jtmp ev lam wsc.
struct SolveLayout {
  double *ja, *jva, *jtmp, *R1, *R2, *T, *Gm, *U, *V, *NB, *ev, *lam, *wsc, *sig, *flip, *lam2;
  double* side;  // start of the whitening CTAs' scratch
};

__device__ __forceinline__ SolveLayout solve_layout(double* g, int n, bool in_smem, double* smem_base) {
  const int nn = n * n;
  SolveLayout L;
  if (in_smem) {
    L.ja = smem_base;
    L.jva = smem_base + nn;
  } else {
    L.ja = g;
    L.jva = g + nn;
  }
  g += 2 * nn;  // reserved either way so the layout does not depend on in_smem
  L.jtmp = g; g += nn;
  L.R1 = g; g += nn;
  L.R2 = g; g += nn;
  L.T = g; g += nn;
  L.Gm = g; g += nn;
  L.U = g; g += nn;
  L.V = g; g += nn;   // right vectors (n x L used)
  L.NB = g; g += nn;  // null basis
  L.ev = g; g += nn;  // eigvec scratch
  L.lam = g; g += n;
  L.wsc = g; g += 2 * n + 2;
  L.sig = g; g += n;
  L.flip = g; g += n;
  L.lam2 = g; g += n;
  L.side = g;
  return L;
}
__host__ __device__ inline size_t solve_side_doubles(int n) { return 4 * (size_t)n * n + 3 * (size_t)n + 2; }

// Whitening (solver.py:227-229) of both views in parallel: CTA b computes
// inv_sqrt(C_bb) into R1 / R2 with its own Jacobi scratch.
__global__ void __launch_bounds__(SOLVE_THREADS) whiten_kernel(SolveArgs S) {
  extern __shared__ double sm[];
  __shared__ double red[SOLVE_THREADS / 32 + 1];
  __shared__ int flag;
  if (*S.status != 0) return;  // finalize failed
  const int n = S.d, nn = n * n;
  const int b = blockIdx.x;
  int* iscr = reinterpret_cast<int*>(sm);
  double* cs = sm + (2 * n + 2 + 1) / 2 + 1;
  double* base = cs + 2 * n + 2;
  SolveLayout L = solve_layout(S.ws, n, false, nullptr);
  double* g = L.side + (size_t)b * solve_side_doubles(n);
  double *ja, *jva;
  if (S.jacobi_in_smem) {
    ja = base;
    jva = base + nn;
  } else {
    ja = g;
    jva = g + nn;
  }
  g += 2 * nn;
  double* jtmp = g; g += nn;
  double* ev = g; g += nn;
  double* lam = g; g += n;
  double* wsc = g;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  Blk B{red, &flag, iscr};
  const double* c = S.fin + (b == 0 ? 0 : nn);
  double* nsbuf = ns_smem_doubles(n) ? base + (S.jacobi_in_smem ? 2 * nn : 0) : nullptr;
  const int rc = inv_sqrt_dev(c, n, b == 0 ? L.R1 : L.R2, lam, ev, ja, jva, cs, jtmp, wsc, B, nsbuf);
  if (rc != DDCCA_OK && threadIdx.x == 0) atomicCAS(reinterpret_cast<int*>(S.status), 0, rc);
}

// ---- after the whitening: T = R1 C~ R2, G1 = T T', G2 = T' T (solver.py:230-247) --------------
// dp x dp shared-memory tiles (zero padding is exact for these products) on the DMMA path; the
// plain per-entry form above NS_MAX_DP.
__device__ void load_padded(const double* src, int n, double* dst, int dp, bool transpose) {
  for (int e = threadIdx.x; e < dp * dp; e += blockDim.x) {
    const int i = e / dp, j = e - i * dp;
    dst[e] = (i < n && j < n) ? (transpose ? src[j * n + i] : src[i * n + j]) : 0.0;
  }
}

__global__ void __launch_bounds__(SOLVE_THREADS) gram_kernel(SolveArgs S) {
  extern __shared__ double sm[];
  if (*S.status != 0) return;
  const int n = S.d, nn = n * n;
  const SolveLayout Y = solve_layout(S.ws, n, false, nullptr);
  double* ct = S.fin + 4 * nn;
  const int dp = ns_dp(n);
  if (dp <= NS_MAX_DP) {
    const int np = dp * dp;
    double *a = sm, *b = sm + np, *c = sm + 2 * np, *t = sm + 3 * np, *tt = sm + 4 * np;
    load_padded(Y.R1, n, a, dp, false);
    load_padded(ct, n, b, dp, false);
    __syncthreads();
    gemm_dmma(a, b, c, dp);               // R1 C~
    load_padded(Y.R2, n, a, dp, false);
    __syncthreads();
    gemm_dmma(c, a, t, dp);               // T = R1 C~ R2
    for (int e = threadIdx.x; e < np; e += blockDim.x) {
      const int i = e / dp, j = e - i * dp;
      tt[e] = t[j * dp + i];
    }
    __syncthreads();
    gemm_dmma(t, tt, a, dp);              // T T'
    gemm_dmma(tt, t, b, dp);              // T' T
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      Y.T[e] = t[i * dp + j];
      Y.ev[e] = 0.5 * (a[i * dp + j] + a[j * dp + i]);  // symmetrized eig inputs (solver.py:232, :240)
      Y.Gm[e] = 0.5 * (b[i * dp + j] + b[j * dp + i]);
    }
    return;
  }
  matmul(Y.R1, false, ct, false, Y.NB, n, n, n);   // R1 C~
  matmul(Y.NB, false, Y.R2, false, Y.T, n, n, n);  // T
  matmul(Y.T, false, Y.T, true, Y.U, n, n, n);     // T T'
  matmul(Y.T, true, Y.T, false, Y.V, n, n, n);     // T' T
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    Y.ev[e] = 0.5 * (Y.U[e] + Y.U[j * n + i]);
    Y.Gm[e] = 0.5 * (Y.V[e] + Y.V[j * n + i]);
  }
}

// eig(T T') (CTA 0: lam, U) and eig(T' T) (CTA 1: lam2, NB -- the null-space completion
// basis, used only when a requested sigma vanishes) in parallel.
__global__ void __launch_bounds__(SOLVE_THREADS) eig2_kernel(SolveArgs S) {
  extern __shared__ double sm[];
  __shared__ double red[SOLVE_THREADS / 32 + 1];
  __shared__ int flag;
  if (*S.status != 0) return;
  const int n = S.d, nn = n * n;
  const int b = blockIdx.x;
  int* iscr = reinterpret_cast<int*>(sm);
  double* cs = sm + (2 * n + 2 + 1) / 2 + 1;
  double* base = cs + 2 * n + 2;
  const SolveLayout Y = solve_layout(S.ws, n, false, nullptr);
  double *ja, *jva, *jtmp, *wsc;
  if (b == 0) {
    ja = Y.ja; jva = Y.jva; jtmp = Y.jtmp; wsc = Y.wsc;
  } else {
    double* g = Y.side + solve_side_doubles(n);  // the second whitening CTA's scratch (free now)
    ja = g; jva = g + nn; g += 2 * nn;
    jtmp = g; g += nn;
    g += nn + n;  // ev, lam of that layout (unused here)
    wsc = g;
  }
  if (S.jacobi_in_smem) {
    ja = base;
    jva = base + nn;
  }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  Blk B{red, &flag, iscr};
  const int rc = b == 0 ? sym_eig_dev(Y.ev, n, Y.lam, Y.U, ja, jva, cs, jtmp, wsc, B)
                        : sym_eig_dev(Y.Gm, n, Y.lam2, Y.NB, ja, jva, cs, jtmp, wsc, B);
  if (rc != DDCCA_OK && threadIdx.x == 0) atomicCAS(reinterpret_cast<int*>(S.status), 0, rc);
}

// sigma, right vectors with null-space completion, W1 = R1 U, W2 = R2 V, the shared sign
// flips and the float32 conv packs (solver.py:233-257, :260-272).
__global__ void __launch_bounds__(SOLVE_THREADS) finish_kernel(SolveArgs S) {
  if (*S.status != 0) return;
  const int n = S.d, L = S.count;
  const SolveLayout Y = solve_layout(S.ws, n, false, nullptr);
  double *R1 = Y.R1, *R2 = Y.R2, *T = Y.T, *U = Y.U, *V = Y.V, *NB = Y.NB, *lam = Y.lam, *sig = Y.sig,
         *flip = Y.flip;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sig[i] = sqrt(fmax(lam[i], 0.0));
  __syncthreads();
  // column k of V (n x L row-major)
  __shared__ int null_src[64];
  if (threadIdx.x == 0) {
    const double thr = 1e-12 * fmax(sig[0], 1e-300);
    int nxt = n - 1;
    for (int k = 0; k < L; ++k) {
      if (sig[k] > thr) {
        null_src[k] = -1;
      } else {
        sig[k] = 0.0;
        null_src[k] = nxt--;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * L; e += blockDim.x) {
    const int i = e / L, k = e - i * L;
    double val;
    if (null_src[k] < 0) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += T[j * n + i] * U[j * n + k];
      val = s / sig[k];
    } else {
      val = NB[i * n + null_src[k]];
    }
    V[e] = val;
  }
  __syncthreads();
  // W1 = R1 U[:, :L], W2 = R2 V
  for (int e = threadIdx.x; e < n * L; e += blockDim.x) {
    const int i = e / L, k = e - i * L;
    double s1 = 0.0, s2 = 0.0;
    for (int j = 0; j < n; ++j) {
      s1 += R1[i * n + j] * U[j * n + k];
      s2 += R2[i * n + j] * V[j * L + k];
    }
    S.w1[e] = s1;
    S.w2[e] = s2;
  }
  __syncthreads();
  col_signs(S.w1, n, L, L, flip);
  __syncthreads();
  for (int e = threadIdx.x; e < n * L; e += blockDim.x) {
    const int k = e % L;
    S.w1[e] *= flip[k];
    S.w2[e] *= flip[k];
  }
  __syncthreads();
  // zero-correlation columns of W2 re-signed independently (solver.py:254-256)
  col_signs(S.w2, n, L, L, flip);
  __syncthreads();
  for (int e = threadIdx.x; e < n * L; e += blockDim.x) {
    const int k = e % L;
    if (sig[k] == 0.0) S.w2[e] *= flip[k];
  }
  for (int k = threadIdx.x; k < L; k += blockDim.x) S.rho[k] = sig[k];
  __syncthreads();
  // conv-ready float32 packs: [tap][filter] == W row-major (reshape_filters, solver.py:260-272)
  for (int e = threadIdx.x; e < n * L; e += blockDim.x) {
    if (S.pack1) S.pack1[e] = (float)S.w1[e];
    if (S.pack2) S.pack2[e] = (float)S.w2[e];
  }
}

struct EigArgs {
  const double* s;
  int n, mode;
  double *w, *v;
  int32_t* status;
  double* ws;
  int jacobi_in_smem;
};

__global__ void __launch_bounds__(SOLVE_THREADS) sym_eig_kernel(EigArgs E) {
  extern __shared__ double sm[];
  __shared__ double red[SOLVE_THREADS / 32 + 1];
  __shared__ int flag;
  const int n = E.n, nn = n * n;
  int* iscr = reinterpret_cast<int*>(sm);
  double* cs = sm + (2 * n + 2 + 1) / 2 + 1;
  double* base = cs + 2 * n + 2;
  double* g = E.ws;
  double *ja, *jva;
  if (E.jacobi_in_smem) {
    ja = base;
    jva = base + nn;
  } else {
    ja = g;
    jva = g + nn;
    g += 2 * nn;
  }
  double* jtmp = g; g += nn;
  double* vv = g; g += nn;
  double* wsc = g; g += 2 * n + 2;
  Blk B{red, &flag, iscr};
  int rc;
  if (E.mode == 0) {
    rc = sym_eig_dev(E.s, n, E.w, E.v, ja, jva, cs, jtmp, wsc, B);
  } else {
    double* nsbuf = ns_smem_doubles(n) ? base + (E.jacobi_in_smem ? 2 * nn : 0) : nullptr;
    rc = inv_sqrt_dev(E.s, n, E.v, E.w, vv, ja, jva, cs, jtmp, wsc, B, nsbuf);
  }
  if (threadIdx.x == 0) *E.status = rc;
}

__global__ void pack_kernel(const double* f, int n, float* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) out[e] = (float)f[e];
}

static size_t jacobi_smem(int n, bool in_smem) {
  size_t ints = sizeof(double) * ((2 * n + 2 + 1) / 2 + 1 + 2 * n + 2);
  return ints + (in_smem ? sizeof(double) * 2 * (size_t)n * n : 0);
}
// whitening / inv_sqrt kernels: the Jacobi area plus the Newton-Schulz buffers
static size_t whiten_smem(int n, bool in_smem) { return jacobi_smem(n, in_smem) + sizeof(double) * ns_smem_doubles(n); }

}  // namespace ddcca

using namespace ddcca;

extern "C" {

size_t ddcca_solve_workspace(int dim) {
  const size_t nn = (size_t)dim * dim;
  return sizeof(double) * (14 * nn + 8 * (size_t)dim + 16 + 2 * solve_side_doubles(dim));
}

int ddcca_solve(const double* payload, int dim, int class_count, double epsilon, int count, double* fin, double* w1,
                double* w2, double* rho, float* conv_pack1, float* conv_pack2, int32_t* status, void* ws,
                size_t ws_bytes, void* stream) {
  if (dim < 1 || class_count < 1) return fail(DDCCA_ECONFIG, "invalid accumulator shape dim=%d classes=%d", dim, class_count);
  if (count < 1 || count > dim) return fail(DDCCA_ECONFIG, "filter count %d outside [1, %d]", count, dim);
  if (count > 64) return fail(DDCCA_ECONFIG, "filter count %d above the device limit 64", count);
  if (epsilon < 0) return fail(DDCCA_ECONFIG, "ridge coefficient %g must be >= 0", epsilon);
  if (ws_bytes < ddcca_solve_workspace(dim)) return fail(DDCCA_ECONFIG, "solve workspace too small");
  if (!fin || !w1 || !w2 || !rho || !status || !ws) return fail(DDCCA_ESHAPE, "null pointer");
  const bool in_smem = dim <= SMEM_JACOBI_MAX_N;
  const size_t sm = jacobi_smem(dim, in_smem);
  SolveArgs S{payload, dim, class_count, count, epsilon, fin, w1, w2, rho, conv_pack1, conv_pack2, status,
              static_cast<double*>(ws), in_smem ? 1 : 0, 1};
  cudaStream_t st = as_stream(stream);
  // finalize -> both whitenings in parallel (two CTAs) -> T, eig(T T^T), filters
  if (payload != nullptr) {
    finalize_kernel<<<finalize_grid(dim), SOLVE_THREADS, 0, st>>>(payload, dim, class_count, epsilon, fin, status);
  } else {
    cudaMemsetAsync(status, 0, sizeof(int32_t), st);
  }
  const size_t smw = whiten_smem(dim, in_smem);
  cudaFuncSetAttribute(whiten_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
  whiten_kernel<<<2, SOLVE_THREADS, smw, st>>>(S);
  // T and both Grams (DMMA), then eig(T T') and eig(T' T) in parallel CTAs, then the filters
  const size_t smg = ns_dp(dim) <= NS_MAX_DP ? sizeof(double) * 5 * (size_t)ns_dp(dim) * ns_dp(dim) : 0;
  cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smg);
  gram_kernel<<<1, SOLVE_THREADS, smg, st>>>(S);
  cudaFuncSetAttribute(eig2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  eig2_kernel<<<2, SOLVE_THREADS, sm, st>>>(S);
  finish_kernel<<<1, SOLVE_THREADS, 0, st>>>(S);
  return check_launch("solve_kernel");
}

int ddcca_finalize(const double* payload, int dim, int class_count, double epsilon, double* fin, int32_t* status,
                   void* stream) {
  if (dim < 1 || class_count < 1) return fail(DDCCA_ECONFIG, "invalid accumulator shape dim=%d classes=%d", dim, class_count);
  if (epsilon < 0) return fail(DDCCA_ECONFIG, "ridge coefficient %g must be >= 0", epsilon);
  finalize_kernel<<<finalize_grid(dim), SOLVE_THREADS, 0, as_stream(stream)>>>(payload, dim, class_count, epsilon, fin, status);
  return check_launch("finalize_kernel");
}

int ddcca_sym_eig(const double* s, int n, int mode, double* w, double* v, int32_t* status, void* ws, size_t ws_bytes,
                  void* stream) {
  if (n < 1) return fail(DDCCA_ESHAPE, "expected a square matrix");
  if (ws_bytes < ddcca_solve_workspace(n)) return fail(DDCCA_ECONFIG, "eig workspace too small");
  const bool in_smem = n <= SMEM_JACOBI_MAX_N;
  const size_t sm = mode == 1 ? whiten_smem(n, in_smem) : jacobi_smem(n, in_smem);
  EigArgs E{s, n, mode, w, v, status, static_cast<double*>(ws), in_smem ? 1 : 0};
  cudaFuncSetAttribute(sym_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  sym_eig_kernel<<<1, SOLVE_THREADS, sm, as_stream(stream)>>>(E);
  return check_launch("sym_eig_kernel");
}

int ddcca_pack_filters(const double* filters, int count, int dim, float* conv_pack, void* stream) {
  if (count < 1 || dim < 1) return fail(DDCCA_ECONFIG, "invalid filter bank %d x %d", count, dim);
  pack_kernel<<<(count * dim + 255) / 256, 256, 0, as_stream(stream)>>>(filters, count * dim, conv_pack);
  return check_launch("pack_filters");
}

}  // extern "C"
