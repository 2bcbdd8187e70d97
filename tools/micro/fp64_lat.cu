// Microbenchmark: dependent-chain latency (cycles) of FP64 ops on sm_100a.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, int iters, double x) {
  double a = x, b = x * 0.5 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-300);
  long long t1 = clock64();
  double d = x + 3.0;
  for (int i = 0; i < iters; ++i) d = 1.0 / (d + 1.0);
  long long t2 = clock64();
  double s = x + 2.0;
  for (int i = 0; i < iters; ++i) s = sqrt(s + 1.0);
  long long t3 = clock64();
  double r = x + 2.0;
  for (int i = 0; i < iters; ++i) r = rsqrt(r + 1.0);
  long long t4 = clock64();
  double h = x;
  for (int i = 0; i < iters; ++i) h += __shfl_xor_sync(0xffffffffu, h, 1);
  long long t5 = clock64();
  double q = x + 1.0;
  for (int i = 0; i < iters; ++i) q = q + 1e-300;
  long long t6 = clock64();
  out[threadIdx.x] = a + d + s + r + h + q;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters;
    cyc[3] = (t4 - t3) / iters; cyc[4] = (t5 - t4) / iters; cyc[5] = (t6 - t5) / iters;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  lat<<<1, 32>>>(o, c, 1000, 0.3);
  lat<<<1, 32>>>(o, c, 4000, 0.3);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DFMA %lld  DDIV(1/x) %lld  DSQRT %lld  DRSQRT %lld  SHFL64+DADD %lld  DADD %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
