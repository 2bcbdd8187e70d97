// Microbenchmark: barrier.cluster round trip and DSMEM load latency vs cluster size (sm_100a).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void bar_kernel(long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int x[32];
  if (threadIdx.x < 32) x[threadIdx.x] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  // remote load latency: dependent chain through the next CTA's smem
  int* rx = cl.map_shared_rank(x, (cl.block_rank() + 1) % cl.num_blocks());
  int v = 0;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) v = rx[(v + i) & 31];
  long long t3 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t3 - t2) / iters + (v == 12345);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int cs : {2, 4, 8, 16}) {
    for (int threads : {64, 256, 512}) {
      cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(threads);
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cs;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, bar_kernel, d, 2000);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("cluster=%d threads=%d barrier_cycles=%lld dsmem_load_cycles=%lld (%s)\n", cs, threads, h[0], h[1],
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
