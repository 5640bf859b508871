// Microbenchmarks for design decisions (not product code):
//  1. streaming read bandwidth (LDG.128, grid-stride)
//  2. gather of 1 KiB rows in random order, warp-per-row-list with U rows in flight
//  3. DMMA m8n8k4 f64 throughput
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void rd_stream(const double2* __restrict__ a, size_t n2, double* out) {
  double2 acc = {0,0};
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  #pragma unroll 8
  for (; i < n2; i += stride) { double2 v; asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a+i)); acc.x += v.x; acc.y += v.y; }
  if (acc.x == 12345.0) out[0] = acc.y;
}

template <int U, int NV>
__global__ void gather_rows(const double* __restrict__ A, const int* __restrict__ perm, const int* __restrict__ off, int m, int d, double* out) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; int lane = threadIdx.x & 31;
  if (w >= m) return;
  int beg = off[w], end = off[w+1];
  double acc[NV]; for (int k=0;k<NV;k++) acc[k]=0;
  for (int base = beg; base < end; base += 32) {
    int pe = base + lane < end ? perm[base+lane] : 0;
    int cnt = min(32, end-base);
    for (int u0 = 0; u0 < cnt; u0 += U) {
      double v[U][NV];
      #pragma unroll
      for (int u=0;u<U;u++){ int r = __shfl_sync(0xffffffff, pe, u0+u); const double* p = A + (size_t)r*d;
        #pragma unroll
        for (int k=0;k<NV;k++){ double t=0; if (u0+u<cnt) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(t) : "l"(p+lane+32*k)); v[u][k]=t; } }
      #pragma unroll
      for (int u=0;u<U;u++) for (int k=0;k<NV;k++) acc[k]+=v[u][k];
    }
  }
  for (int k=0;k<NV;k++) out[(size_t)w*d+lane+32*k]=acc[k];
}

// L2-resident re-reads: each CTA streams the same small buffer reps times
__global__ void rd_l2(const double2* __restrict__ a, size_t n2, int reps, double* out) {
  double2 acc = {0,0};
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x + (size_t)r * 7919 * 32) % n2;
    #pragma unroll 8
    for (size_t k = 0; k < n2 / stride; ++k) { double2 v = a[(i + k * stride) % n2]; acc.x += v.x; acc.y += v.y; }
  }
  if (acc.x == 12345.0) out[0] = acc.y;
}
// smem fp64 read-modify-write throughput: conflict-free (lane-contiguous) vs random rows
__global__ void smem_rmw(int iters, int random, double* out) {
  extern __shared__ double tile[];
  const int n = 16384;  // 128 KB
  for (int e = threadIdx.x; e < n; e += blockDim.x) tile[e] = 0.0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < iters; ++i) {
    int idx;
    if (random) { x = x * 1664525u + 1013904223u; idx = ((x >> 8) % (n / 4)) * 4 + (lane & 3); }
    else idx = ((i * 16 + warp) * 32 + lane) % n;
    tile[idx] += 1.0;
  }
  __syncthreads();
  if (tile[threadIdx.x] == 12345.0) out[0] = 1;
}

// fp64 RED.ADD throughput into a large array (random 8-byte addresses), the
// CSR sketch's bound
__global__ void red_random(double* buf, size_t n, int iters) {
  unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    size_t idx = ((size_t)x * 2654435761ull) % n;
    atomicAdd(buf + idx, 1.0);
  }
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[4]={0,0,0,0}, c1[4]={0,0,0,0};
  for (int i=0;i<iters;i++){
    #pragma unroll
    for (int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0[j]), "+d"(c1[j]) : "d"(a), "d"(b));
  }
  double s=0; for(int j=0;j<4;j++) s+=c0[j]+c1[j];
  if (s == 1234.5) out[0]=s;
}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("gpu %s sms %d l2 %d MB smemPerBlockOptin %zu\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20, p.sharedMemPerBlockOptin);
  size_t bytes = (size_t)4<<30; double* A; CK(cudaMalloc(&A, bytes)); CK(cudaMemset(A, 0, bytes));
  double* out; CK(cudaMalloc(&out, 64<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int bl : {148*4, 148*8, 148*16}) {
    for (int r=0;r<3;r++){ cudaEventRecord(e0); rd_stream<<<bl,256>>>((const double2*)A, bytes/16, out); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("stream read grid=%d: %.3f ms  %.1f GB/s\n", bl, ms, bytes/ms/1e6);
  }
  // gather: n=4M rows, d=128, m=1024
  int n = 1<<22, d = 128, m = 1024;
  std::vector<int> h(n), perm(n), off(m+1,0);
  std::mt19937_64 rng(1); for (int i=0;i<n;i++){ h[i]=rng()%m; off[h[i]+1]++; }
  for (int b=0;b<m;b++) off[b+1]+=off[b];
  { std::vector<int> c(off.begin(), off.end()-1); for (int i=0;i<n;i++) perm[c[h[i]]++]=i; }
  int *dp,*doff; CK(cudaMalloc(&dp,n*4)); CK(cudaMalloc(&doff,(m+1)*4));
  cudaMemcpy(dp,perm.data(),n*4,cudaMemcpyHostToDevice); cudaMemcpy(doff,off.data(),(m+1)*4,cudaMemcpyHostToDevice);
  #define G(U) for(int r=0;r<3;r++){cudaEventRecord(e0); gather_rows<U,4><<<m*32/64,64>>>(A,dp,doff,m,d,out); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1); printf("gather U=%d warp/bucket: %.3f ms %.1f GB/s\n", U, ms, (double)n*d*8/ms/1e6);
  G(4) G(8) G(16)
  // contiguous: bucket b = rows [b*n/m, (b+1)*n/m)
  { std::vector<int> id(n), of2(m+1); for (int i=0;i<n;i++) id[i]=i; for (int b=0;b<=m;b++) of2[b]=(int)((long)b*n/m);
    cudaMemcpy(dp,id.data(),n*4,cudaMemcpyHostToDevice); cudaMemcpy(doff,of2.data(),(m+1)*4,cudaMemcpyHostToDevice); }
  printf("contiguous:\n"); G(8) G(16)
  // interleaved: bucket b = rows b, b+m, b+2m, ... (the band pattern of sorted buckets, perfectly in sync)
  { std::vector<int> id(n), of2(m+1); int k=0; for (int b=0;b<m;b++){ of2[b]=k; for (int i=b;i<n;i+=m) id[k++]=i; } of2[m]=n;
    cudaMemcpy(dp,id.data(),n*4,cudaMemcpyHostToDevice); cudaMemcpy(doff,of2.data(),(m+1)*4,cudaMemcpyHostToDevice); }
  printf("strided b+k*m:\n"); G(8) G(16)
  CK(cudaGetLastError());
  for (size_t mb : {32, 64, 96}) {
    size_t nb = mb << 20;
    for (int r=0;r<3;r++){ cudaEventRecord(e0); rd_l2<<<148*8,256>>>((const double2*)A, nb/16, 20, out); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("L2 re-read %zu MB x20: %.3f ms  %.1f GB/s\n", mb, ms, 20.0*nb/ms/1e6);
  }
  cudaFuncSetAttribute(smem_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int rnd : {0, 1}) {
    int it = 4096;
    for (int r=0;r<2;r++){ cudaEventRecord(e0); smem_rmw<<<148,512,131072>>>(it, rnd, out); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    double upd = 148.0*512*it;
    printf("smem fp64 RMW %s: %.3f ms  %.2f G upd/s  (%.2f upd/clk/SM at 1.965 GHz)\n", rnd ? "random 32B rows" : "contiguous", ms, upd/ms/1e6, upd/ms/1e-3/148/1.965e9);
  }
  for (size_t mb : {64, 512}) {
    size_t nel = (mb << 20) / 8;
    int it = 256;
    for (int r=0;r<2;r++){ cudaEventRecord(e0); red_random<<<148*8,256>>>(A, nel, it); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    double ops = 148.0*8*256*it;
    printf("RED.ADD.F64 random over %zu MB: %.3f ms  %.1f G red/s\n", mb, ms, ops/ms/1e6);
  }
  CK(cudaGetLastError());
  // dmma
  for (int r=0;r<2;r++){ cudaEventRecord(e0); dmma_loop<<<148*4,256>>>(out, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
  double fl = 148.0*4*8*4096*4*2*8*8*4; printf("dmma: %.3f ms %.2f TFLOP/s\n", ms, fl/ms/1e9);
  CK(cudaGetLastError());
  return 0;
}
