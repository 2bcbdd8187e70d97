// Microbenchmark: where the cycles of one one-sided Jacobi pair step go
// (8 warps, one pair each, columns in shared memory, ld = n as in the
// preconditioned cluster path).  mode 0: jacobi_pair(); 1: dot products +
// butterfly reductions; 2: + rotation angle; 3: rotation only; 4: jacobi_pair_reg.
#include <cstdio>

#include "../../paper_2206_00975_b200/csrc/jacobi_pair.cuh"

template <int MODE>
__global__ void bench(double* out, long long* cyc, int n, int iters) {
  extern __shared__ double sm[];
  const int ld = n, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 16 * ld; e += blockDim.x) sm[e] = 1.0 + ((e * 37) % 101) * 0.01;
  __syncthreads();
  double* xp = sm + (2 * warp) * ld;
  double* xq = sm + (2 * warp + 1) * ld;
  double sink = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      sink += nsk::jacobi_pair<1>(xp, xq, n, ld, lane, 1e-60);
    } else if (MODE == 4) {
      sink += nsk::jacobi_pair_reg<1, 8>(xp, xq, n, ld, lane, 1e-60);
    } else if (MODE == 3) {
      nsk::rotate_cols<1>(xp, xq, ld, lane, 0.8, 0.6, 1.0, 0.0);
    } else {
      double a = 0, bb = 0, cr = 0;
      int row = lane;
      for (; row + 96 < n; row += 128) {
        double up[4], uq[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          up[k] = xp[row + 32 * k];
          uq[k] = xq[row + 32 * k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a = fma(up[k], up[k], a);
          bb = fma(uq[k], uq[k], bb);
          cr = fma(up[k], uq[k], cr);
        }
      }
      for (; row < n; row += 32) {
        const double up = xp[row], uq = xq[row];
        a = fma(up, up, a);
        bb = fma(uq, uq, bb);
        cr = fma(up, uq, cr);
      }
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        bb += __shfl_xor_sync(0xffffffffu, bb, o);
        cr += __shfl_xor_sync(0xffffffffu, cr, o);
      }
      if (MODE == 1) {
        sink += a + bb + cr;
      } else {
        const double zeta = (bb - a) / (2.0 * cr);
        const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double cs = rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
        sink += cs + sn;
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  out[threadIdx.x] = xp[lane] + sink;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 4096 * 8);
  cudaMalloc(&c, 16);
  for (int n : {64, 128, 256}) {
    const int smem = 16 * n * 8;
    long long h[5];
    auto run = [&](auto kern, int idx) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<1, 256, smem>>>(o, c, n, 2000);
      cudaMemcpy(&h[idx], c, 8, cudaMemcpyDeviceToHost);
    };
    run(bench<0>, 0);
    run(bench<1>, 1);
    run(bench<2>, 2);
    run(bench<3>, 3);
    run(bench<4>, 4);
    printf("n=%d cycles/step: full %lld | dots+reduce %lld | +angle %lld | rotate only %lld | register step %lld (%s)\n",
           n, h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
