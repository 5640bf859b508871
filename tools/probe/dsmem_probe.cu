// Microbenchmark (not product code): distributed-shared-memory read bandwidth
// inside a thread-block cluster (each CTA streams peer CTAs' shared memory).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void dsmem_read(int iters, double *out) {
  extern __shared__ double buf[];  // 8192 doubles = 64 KB
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), cs = cl.num_blocks();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = rank + i * 1e-9;
  cl.sync();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int peer = (rank + 1 + it % (cs - 1)) % cs;
    const double2 *p = reinterpret_cast<const double2 *>(cl.map_shared_rank(buf, peer));
#pragma unroll 4
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
      double2 v = p[i];
      acc += v.x + v.y;
    }
  }
  cl.sync();
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  double *out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(dsmem_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(dsmem_read, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    for (int threads : {256, 512, 1024}) {
      cudaLaunchConfig_t cfg = {};
      int nclusters = 148 / cs;
      cfg.gridDim = dim3(nclusters * cs);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = 65536;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int iters = 200;
      float ms = 0;
      for (int r = 0; r < 2; ++r) {
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, dsmem_read, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)nclusters * cs * iters * 65536.0;
      printf("cluster %2d threads %4d: %.3f ms, %.1f GB/s total, %.1f GB/s per SM (%.1f B/clk at 1.965 GHz) %s\n", cs,
             threads, ms, bytes / ms / 1e6, bytes / ms / 1e6 / (nclusters * cs),
             bytes / ms / 1e6 / (nclusters * cs) / 1.965, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
