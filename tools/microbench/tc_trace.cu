// Pipeline timeline of the tensor-core conv-histogram kernel (CTA 0): clock64 at each
// hand-off (MMA warp: A full / accumulator empty / issued; epilogue: accumulator full /
// read; producer: A slot free / written). Build from the repo root:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench/_bin/tc_trace \
//     tools/microbench/tc_trace.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#define DDCCA_TC_TRACE 1
#include "../../paper_2209_13027_b200/csrc/convtc.cu"

int main(int argc, char** argv) {
  using namespace ddcca;
  const int n = argc > 1 ? atoi(argv[1]) : 2048, p = 128, q = 128, l = 7;
  const bool resp = argc > 2 && argv[2][0] == 'r';  // responses mode (ddcca_conv) instead of histograms
  std::vector<float> h((size_t)n * p * q), taps(l * l * TC_FILTERS);
  srand(1);
  for (auto& v : h) v = (float)rand() / RAND_MAX - 0.5f;
  for (auto& v : taps) v = (float)rand() / RAND_MAX - 0.5f;
  float *din, *dtaps;
  uint8_t* dcounts;
  const int nby = 8, nbx = 8;
  cudaMalloc(&din, h.size() * 4);
  cudaMalloc(&dtaps, taps.size() * 4);
  cudaMalloc(&dcounts, (size_t)n * nby * nbx * 256);
  float* dresp = nullptr;
  if (resp) cudaMalloc(&dresp, (size_t)n * 8 * p * q * 4);
  cudaMemcpy(din, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dtaps, taps.data(), taps.size() * 4, cudaMemcpyHostToDevice);
  TcHistArgs a{};
  a.in = din; a.n_maps = n; a.p = p; a.q = q; a.top = 3; a.left = 3; a.l = l;
  a.count = 8; a.center = 1; a.bh = 16; a.bw = 16; a.nby = nby; a.nbx = nbx; a.kind = 0; a.nbits = 8;
  a.counts = dcounts; a.gpr = 1; a.row_stride = (int64_t)nby * nbx * 256; a.group_stride = 0;
  a.resp = dresp; a.dc_shift = 1;
  auto launch = [&]() { return resp ? conv_resp_tc(a, dtaps, 0) : conv_hist_tc(a, dtaps, 0); };
  for (int it = 0; it < 2; ++it) printf("rc %d\n", launch());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%d maps: %.3f ms (%s)\n", n, ms, cudaGetErrorString(cudaDeviceSynchronize()));
  long long t[12][256];
  cudaMemcpyFromSymbol(t, tc::g_tc_trace, sizeof(t));
  const long long t0 = t[5][0];
  printf("blk  prodTfree prodFull | mmaFull mmaEmpty mmaIssued | epiFull epiRead\n");
  for (int b = 0; b < 80; ++b)
    printf("%3d %9lld %9lld | %9lld %9lld %9lld | %9lld %9lld\n", b, t[5][b] - t0, t[6][b] - t0, t[0][b] - t0,
           t[1][b] - t0, t[2][b] - t0, t[3][b] - t0, t[4][b] - t0);
  printf("map  flushStart flushEnd\n");
  for (int i = 0; i < 6; ++i) printf("%3d %9lld %9lld\n", i, t[7][2 * i] - t0, t[7][2 * i + 1] - t0);
  return 0;
}
