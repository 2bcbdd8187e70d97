// DRAM efficiency of the srft / srdct access pattern: a column of m = 2^20 doubles is read as
// 1024 rows (stride P = 1024 doubles = 8 KiB) of G contiguous 128-byte lines per visit, one visit
// per "tile group"; 148 x 2 CTAs walk different (column, group) ranges as the transform kernels do.
// G = 1 is what the kernels' per-tile L2 prefetch issues today.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void strided_lines(const double* __restrict__ a, long lda, long n, int G, long groups_per_col,
                              long per, double* out) {
  const long total = n * groups_per_col;
  long u = blockIdx.x * per, u1 = u + per < total ? u + per : total;
  double s = 0;
  for (; u < u1; ++u) {
    const long c = u / groups_per_col, g = u % groups_per_col;
    const double* base = a + c * lda + g * (16L * G);
    // 1024 rows x G lines of 16 doubles; thread t: row = (t + 256 j) / (G), line = ... coalesce 16 B per thread
    const int per_row = 8 * G;  // double2 per row visit
    for (int e = threadIdx.x; e < 1024 * per_row; e += blockDim.x) {
      const int row = e / per_row, k = e % per_row;
      const double2 v = __ldcg(reinterpret_cast<const double2*>(base + 1024L * row) + k);
      s += v.x + v.y;
    }
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  const long m = 1L << 20, n = 256;
  double *a, *o;
  cudaMalloc(&a, m * n * 8);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, m * n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int ctas : {148, 296, 592})
    for (int G : {1, 2, 4, 8}) {
      const long groups = 1024 / (16 * G), total = n * groups, per = (total + ctas - 1) / ctas;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        strided_lines<<<ctas, 256>>>(a, m, n, G, groups, per, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%d CTAs, %d line(s) of 128 B per row visit (stride 8 KiB): %.1f GB/s\n", ctas, G,
             m * n * 8 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
