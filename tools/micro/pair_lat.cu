// Microbenchmark: cycles per jacobi_pair() call (one warp per pair, 8 warps, columns in SMEM).
#include <cstdio>
#include "../../paper_2206_00975_b200/csrc/jacobi_pair.cuh"

template <int NW>
__global__ void bench(double* out, long long* cyc, int n, int iters) {
  extern __shared__ double sm[];
  const int ld = 2 * n, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 2 * NW * ld; e += blockDim.x) sm[e] = 1.0 + ((e * 37) % 101) * 0.01;
  __syncthreads();
  double* xp = sm + (2 * warp) * ld;
  double* xq = sm + (2 * warp + 1) * ld;
  int rot = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    rot += nsk::jacobi_pair<1>(xp, xq, n, ld, lane, 1e-60);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / iters;
    cyc[1] = rot;
  }
  out[threadIdx.x] = xp[lane];
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 16);
  for (int n : {64, 128, 256}) {
    const int smem = 2 * 8 * 2 * n * 8;
    cudaFuncSetAttribute(bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<8><<<1, 256, smem>>>(o, c, n, 2000);
    long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("n=%d: %lld cycles per pair step (8 warps), rotations %lld (%s)\n", n, h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
