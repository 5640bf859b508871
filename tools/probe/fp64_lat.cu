// fp64 / shuffle latency probe (one warp, clock64): dependent DFMA chain,
// dependent DADD chain, 8 interleaved DFMA chains, dependent 64-bit SHFL+DADD
// (the warp-reduction step), MUFU-based sqrt and divide.
#include <cstdio>

__global__ void lat(double *out, long long *cyc, int n, double a, double b) {
  double x = a, y = b, v[8];
  for (int i = 0; i < 8; ++i) v[i] = a + i;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = y + a;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fma(v[k], a, b);
  long long t3 = clock64();
  double s = x;
  for (int i = 0; i < n; ++i) s += __shfl_xor_sync(0xffffffffu, s, 1 + (i & 15));
  long long t4 = clock64();
  double q = y;
  for (int i = 0; i < n; ++i) q = sqrt(q + 1.0);
  long long t5 = clock64();
  double r = y;
  for (int i = 0; i < n; ++i) r = a / (r + 1.0);
  long long t6 = clock64();
  double acc = x + y + s + q + r;
  for (int k = 0; k < 8; ++k) acc += v[k];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}

int main() {
  double *o;
  long long *c, h[6];
  cudaMalloc(&o, 1024 * 8);
  cudaMalloc(&c, 6 * 8);
  const int n = 1024;
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 32>>>(o, c, n, 0.999, 1e-3);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  }
  printf("per op (cycles): DFMA dep %.1f  DADD dep %.1f  8xDFMA indep (per 8) %.1f  SHFL64+DADD dep %.1f  sqrt dep %.1f  div dep %.1f\n",
         h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  for (int w : {4, 8, 16}) {
    lat<<<1, 32 * w>>>(o, c, n, 0.999, 1e-3);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%2d warps/CTA: DFMA dep %.1f  DADD dep %.1f  8xDFMA %.1f  SHFL64+DADD %.1f  sqrt %.1f  div %.1f\n", w,
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  }
  return 0;
}
