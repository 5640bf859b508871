// Phase timing of the CG loop of ols_large_kernel (C3's shape: d = 1024, H a
// sketched Gram with m = 8 d): builds ols_large.cu with IHS_CG_TIMING and
// prints cycles per CG step by phase (CTA 0, thread 0).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//     -Ipaper_1910_14166_b200/csrc -o tools/probe/cg_timing tools/probe/cg_timing.cu
#define IHS_CG_TIMING 1
#include "../../paper_1910_14166_b200/csrc/ols_large.cu"

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char **argv) {
  const int d = argc > 1 ? atoi(argv[1]) : 1024, m = 8 * d;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::mt19937_64 rng(11);
  std::normal_distribution<double> nd;
  // H = SA^T SA / m with SA Gaussian (m x d), formed on the host in blocks
  std::vector<double> SA((size_t)m * d), H((size_t)d * d, 0.0), g(d), x(d, 0.0);
  for (auto &v : SA) v = nd(rng);
  for (int k = 0; k < m; ++k) {
    const double *r = &SA[(size_t)k * d];
    for (int i = 0; i < d; ++i) {
      const double ri = r[i] / m;
      double *hi = &H[(size_t)i * d];
      for (int j = 0; j < d; ++j) hi[j] += ri * r[j];
    }
  }
  for (auto &v : g) v = nd(rng);
  double *dH, *dg, *dx, *dxn, *scr;
  int *dst;
  cudaMalloc(&dH, sizeof(double) * d * d);
  cudaMalloc(&dg, sizeof(double) * d);
  cudaMalloc(&dx, sizeof(double) * d);
  cudaMalloc(&dxn, sizeof(double) * d);
  cudaMalloc(&scr, ihs::ols_large_scratch_bytes(d));
  cudaMalloc(&dst, sizeof(int));
  cudaMemcpy(dH, H.data(), sizeof(double) * d * d, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, g.data(), sizeof(double) * d, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), sizeof(double) * d, cudaMemcpyHostToDevice);
  cudaMemset(dst, 0, sizeof(int));
  ihs::LaunchCounter lc;
  for (int rep = 0; rep < 4; ++rep) {
    long long z[8] = {0};
    cudaMemcpyToSymbol(ihs::g_cg_timing, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = ihs::launch_ols_large(dH, dg, d, dx, dxn, scr, dst, sms, 0, 0, lc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, ihs::g_cg_timing, sizeof(z));
    const double k = z[5] > 0 ? (double)z[5] : 1.0;
    printf("d=%d: %lld CG steps, %.4f ms (%.3f us/step incl. launch); cycles/step: matvec %.0f  barrier %.0f  "
           "q read+pq %.0f  updates %.0f  total %.0f  (%s / %s)\n",
           d, z[5], ms, 1e3 * ms / k, z[0] / k, z[1] / k, z[2] / k, z[3] / k, z[4] / k, cudaGetErrorString(e),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
