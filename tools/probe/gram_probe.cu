// Stream-K Gram at C3's shape (SA 8192 x 1024): CTAs per SM 2 vs 3 (the plan's
// persistent grid), device time per launch.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//     -Ipaper_1910_14166_b200/csrc -o tools/probe/gram_probe tools/probe/gram_probe.cu
#include "../../paper_1910_14166_b200/csrc/gram.cu"

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char **argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 8192, d = argc > 2 ? atoll(argv[2]) : 1024;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> h((size_t)m * d);
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  for (auto &v : h) v = nd(rng);
  double *SA, *H, *part;
  cudaMalloc(&SA, sizeof(double) * m * d);
  cudaMalloc(&H, sizeof(double) * d * d);
  cudaMemcpy(SA, h.data(), sizeof(double) * m * d, cudaMemcpyHostToDevice);
  cudaMalloc(&part, (size_t)512 << 20);
  ihs::LaunchCounter lc;
  std::vector<double> ref((size_t)d * d), out((size_t)d * d);
  for (int cps : {2, 3, 4, 2}) {
    ihs::GramPlan p = ihs::gram_plan(m, d, sms, cps);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) ihs::launch_gram(p, SA, 1.0, part, H, 0, lc);
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) ihs::launch_gram(p, SA, 1.0, part, H, 0, lc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(out.data(), H, sizeof(double) * d * d, cudaMemcpyDeviceToHost);
    if (cps == 2 && ref[0] == 0.0) ref = out;
    double md = 0;
    for (size_t i = 0; i < out.size(); ++i) md = std::max(md, std::abs(out[i] - ref[i]));
    const double fl = (double)p.ntri * 64 * 64 * m * 2;
    printf("ctas/SM %d: ncta %d kch %d ipc %d: %.4f ms per Gram (gram + reduce), %.2f TF/s (upper tiles), max|dH| vs 2/SM %.3g (%s)\n",
           cps, p.ncta, p.kch, p.ipc, ms / reps, fl / (ms / reps * 1e-3) / 1e12, md, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
