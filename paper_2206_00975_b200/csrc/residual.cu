// residual.cu -- ||A W||_F in one streaming pass over A.
//
// Reference: residual_certificate (/root/reference/proj/src/nullspace.cpp:55-62),
// frobenius_norm(matmul(A, W)).  Opt-in, O(mnk); used for parity checks.
// Each thread owns one row of A and forms up to 8 entries of (A W)(row, :)
// per pass; the sum of squares is reduced per CTA and then across CTAs in
// fixed order (deterministic).
#include "nsk_internal.hpp"

namespace nsk {
namespace {

constexpr int RT = 256;
constexpr int KB = 8;

template <int NC>
__global__ void residual_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                const double* __restrict__ W, int64_t ldw, int64_t k,
                                double* __restrict__ partial) {
  extern __shared__ double sw[];  // W block: n x KB (x NC)
  __shared__ double red[RT / 32];
  double acc = 0.0;
  for (int64_t t0 = 0; t0 < k; t0 += KB) {
    const int kb = static_cast<int>((k - t0) < KB ? (k - t0) : KB);
    __syncthreads();
    for (int64_t e = threadIdx.x; e < n * KB; e += RT) {
      const int64_t c = e / KB, t = e % KB;
      if (NC == 1) {
        sw[e] = t < kb ? W[c + (t0 + t) * ldw] : 0.0;
      } else {
        sw[2 * e] = t < kb ? W[2 * (c + (t0 + t) * ldw)] : 0.0;
        sw[2 * e + 1] = t < kb ? W[2 * (c + (t0 + t) * ldw) + 1] : 0.0;
      }
    }
    __syncthreads();
    for (int64_t row = blockIdx.x * static_cast<int64_t>(RT) + threadIdx.x; row < m;
         row += static_cast<int64_t>(gridDim.x) * RT) {
      double yr[KB], yi[KB];
#pragma unroll
      for (int t = 0; t < KB; ++t) yr[t] = yi[t] = 0.0;
      for (int64_t c = 0; c < n; ++c) {
        if (NC == 1) {
          const double a = A[row + c * lda];
#pragma unroll
          for (int t = 0; t < KB; ++t) yr[t] = fma(a, sw[c * KB + t], yr[t]);
        } else {
          const double ar = A[2 * (row + c * lda)], ai = A[2 * (row + c * lda) + 1];
#pragma unroll
          for (int t = 0; t < KB; ++t) {
            const double wr = sw[2 * (c * KB + t)], wi = sw[2 * (c * KB + t) + 1];
            yr[t] += ar * wr - ai * wi;
            yi[t] += ar * wi + ai * wr;
          }
        }
      }
#pragma unroll
      for (int t = 0; t < KB; ++t) acc += yr[t] * yr[t] + yi[t] * yi[t];
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RT / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void sum_partials(const double* __restrict__ partial, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < nb; ++i) t += partial[i];
    out[0] = sqrt(t);
  }
}

}  // namespace

int residual_fro(int ncomp, int64_t m, int64_t n, const double* A, int64_t lda, int64_t k, const double* W,
                 int64_t ldw, double* out_host, cudaStream_t st) {
  if (k == 0 || m == 0) {
    *out_host = 0.0;
    return OK;
  }
  int64_t blocks = (m + RT - 1) / RT;
  if (blocks > 4L * sm_count()) blocks = 4L * sm_count();
  Scratch ws;
  NSK_CUDA_OK(ws.alloc(sizeof(double) * (blocks + 1), st));
  const size_t smem = sizeof(double) * n * KB * ncomp;
  if (smem > 200 * 1024) return fail(EINVAL_, "residual_certificate: n too large for this build");
  if (ncomp == 1) {
    NSK_CUDA_OK(cudaFuncSetAttribute(residual_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    residual_kernel<1><<<static_cast<unsigned>(blocks), RT, smem, st>>>(A, lda, m, n, W, ldw, k, ws.as<double>());
  } else {
    NSK_CUDA_OK(cudaFuncSetAttribute(residual_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    residual_kernel<2><<<static_cast<unsigned>(blocks), RT, smem, st>>>(A, lda, m, n, W, ldw, k, ws.as<double>());
  }
  NSK_CUDA_OK(cudaGetLastError());
  sum_partials<<<1, 32, 0, st>>>(ws.as<double>(), static_cast<int>(blocks), ws.as<double>() + blocks);
  count_launch(2);
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaMemcpyAsync(out_host, ws.as<double>() + blocks, sizeof(double), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return OK;
}

}  // namespace nsk
