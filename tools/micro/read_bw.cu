// Read-bandwidth microbenchmark: what does the SRHT access pattern (one warp per
// 8 KiB block, 32 x LDG.64 per lane, persistent warps) reach vs. a plain
// grid-stride vectorised read?  2 GiB input (configs[1] A).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void warp_block_read(const double* __restrict__ a, long total_blocks, long per, double* out) {
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  long it = warp * per, end = it + per;
  if (end > total_blocks) end = total_blocks;
  double s = 0;
  for (; it < end; ++it) {
    const double* p = a + it * 1024 + lane;
    double x[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) x[t] = __ldcs(p + 32 * t);
#pragma unroll
    for (int t = 0; t < 32; ++t) s += x[t];
  }
  if (s == 1.2345) out[0] = s;
}
__global__ void grid_read(const double2* __restrict__ a, long n4, double* out) {
  double s = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i);
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  const long n = 1L << 28;  // 2 GiB of doubles
  double *a, *o;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int wps : {4, 8, 12, 16}) {
    int ctas_per_sm = wps / 4;
    long warps = 148L * wps, blocks = n / 1024, per = (blocks + warps - 1) / warps;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      warp_block_read<<<148 * ctas_per_sm, 128>>>(a, blocks, per, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("warp-block read, %2d warps/SM: %.1f GB/s\n", wps, n * 8 / (ms * 1e-3) / 1e9);
  }
  for (int cps : {2, 4, 8, 16, 32}) {  // the read-only ceiling: plain grid-stride 16-byte loads
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      grid_read<<<148 * cps, 256>>>((const double2*)a, n / 2, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid-stride 16-byte read, %2d CTAs of 256 per SM: %.1f GB/s\n", cps, n * 8 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
