// Phase timing of the device Jacobi eigensolver (diagnostic build of solve.cu with
// DDCCA_SOLVE_PROF): clock64 totals of thread 0 for the off-diagonal norm, the
// rotation-parameter phase, the update phase, the whole sweep loop and the
// ordering epilogue, plus the sweep count, for a few matrix orders.
#define DDCCA_SOLVE_PROF 1
#include "../../paper_2209_13027_b200/csrc/solve.cu"

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

int main() {
  for (int n : {25, 49, 81}) {
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> x((size_t)n * n), s((size_t)n * n, 0.0);
    for (auto& v : x) v = nd(rng);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double acc = 0;
        for (int k = 0; k < n; ++k) acc += x[i * n + k] * x[j * n + k];
        s[i * n + j] = acc;
      }
    double *ds, *w, *v, *ws;
    int32_t* st;
    const size_t wsb = ddcca_solve_workspace(n);
    cudaMalloc(&ds, 8 * n * n); cudaMalloc(&w, 8 * n); cudaMalloc(&v, 8 * n * n); cudaMalloc(&ws, wsb);
    cudaMalloc(&st, 4);
    cudaMemcpy(ds, s.data(), 8 * n * n, cudaMemcpyHostToDevice);
    unsigned long long zero[8] = {0};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpyToSymbol(g_solve_prof, zero, sizeof(zero));
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      ddcca_sym_eig(ds, n, 0, w, v, st, ws, wsb, nullptr);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      unsigned long long pr[8];
      cudaMemcpyFromSymbol(pr, g_solve_prof, sizeof(pr));
      printf("n=%d %.3f ms sweeps %llu | cycles: offnorm %llu params %llu update %llu loop %llu post %llu | per round params %.0f update %.0f\n",
             n, ms, pr[7], pr[0], pr[1], pr[2], pr[3], pr[4], (double)pr[1] / (pr[7] * (n + (n & 1) - 1)),
             (double)pr[2] / (pr[7] * (n + (n & 1) - 1)));
    }
  }
  return 0;
}
