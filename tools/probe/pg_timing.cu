// Phase timing of the PG inner loop (pg_warp_kernel, l1 ball and LASSO) at
// d = 256 on a sketched Gram: builds pg.cu with IHS_PG_TIMING (per-phase
// clock64 sums of cluster rank 0, thread 0), runs one update with the step
// bound given (L_in, as in the look-ahead schedule) and prints cycles per
// inner step by phase.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//     -Ipaper_1910_14166_b200/csrc -o tools/probe/pg_timing tools/probe/pg_timing.cu
#ifdef PG_OLD  // the committed pg.cu before the st.async exchange (A/B of the step time only)
#include "pg_old.cuh"
#else
#define IHS_PG_TIMING 1
#include "../../paper_1910_14166_b200/csrc/pg.cu"
#endif

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char **argv) {
  const int d = argc > 1 ? atoi(argv[1]) : 256, m = 8 * d;
  const int cl = argc > 2 ? atoi(argv[2]) : 0;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::vector<double> SA((size_t)m * d), H((size_t)d * d, 0.0), g(d), x(d, 0.0);
  for (auto &v : SA) v = nd(rng);
  for (int k = 0; k < m; ++k)
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) H[(size_t)i * d + j] += SA[(size_t)k * d + i] * SA[(size_t)k * d + j] / m;
  for (auto &v : g) v = 5.0 * nd(rng);
  double *dH, *dg, *dx, *dxn, *dL, *dsc;
  int32_t *dit;
  int *dst;
  cudaMalloc(&dH, sizeof(double) * d * d);
  cudaMalloc(&dg, sizeof(double) * d);
  cudaMalloc(&dx, sizeof(double) * d);
  cudaMalloc(&dxn, sizeof(double) * d);
  cudaMalloc(&dL, sizeof(double));
  cudaMalloc(&dsc, sizeof(double) * d);
  cudaMalloc(&dit, sizeof(int32_t));
  cudaMalloc(&dst, sizeof(int));
  cudaMemcpy(dH, H.data(), sizeof(double) * d * d, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, g.data(), sizeof(double) * d, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), sizeof(double) * d, cudaMemcpyHostToDevice);
  cudaMemset(dst, 0, sizeof(int));
  ihs::LaunchCounter lc;
  // the step bound first (power-only launch), then the timed updates
  ihs::launch_l1ball_update(dH, dg, d, dx, 3.0, 20000, 50, 12, 1e-14, 1.05, dxn, dit, dsc, dst, 0, lc, false, 0,
                            nullptr, dL, cl);
  for (int prox = 0; prox < 2; ++prox) {
    for (int rep = 0; rep < 3; ++rep) {
      long long z[8] = {0};
#ifndef PG_OLD
      cudaMemcpyToSymbol(ihs::g_pg_timing, z, sizeof(z));
#endif
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      ihs::launch_l1ball_update(dH, dg, d, dx, prox ? 2.0 : 3.0, 20000, 50, 12, 1e-14, 1.05, dxn, dit, dsc, dst, 0,
                                lc, false, prox, dL, nullptr, cl);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      int it = 0;
      cudaMemcpy(&it, dit, sizeof(int), cudaMemcpyDeviceToHost);
#ifndef PG_OLD
      cudaMemcpyFromSymbol(z, ihs::g_pg_timing, sizeof(z));
#endif
      const double k = it > 0 ? it : 1;
      printf("%s d=%d cluster=%d: %d inner steps, %.4f ms launch (%.3f us/step incl. launch); cycles/step: "
             "gemv+send %.0f  wait %.0f  projection %.0f  norms+update %.0f [elementwise %.0f, shuffles %.0f]  total %.0f  (%s)\n",
             prox ? "lasso " : "l1ball", d, cl, it, ms, 1e3 * ms / k, z[0] / k - z[1] / k, z[1] / k, z[2] / k,
             z[3] / k, z[5] / k, z[6] / k, z[4] / k, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
