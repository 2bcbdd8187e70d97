// tall_qr.cu -- R factor of a tall [A | B] on the device: shifted
// CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020), the
// "exact" baseline behind tls_solve_exact (tls.cpp:83-95: thin QR of [A|B],
// then SVDs of the small triangle).
//
// The reference factors [A|B] with Householder QR on one core.  On a B200
// the O(m N^2) work has to run on the FP64 tensor pipe, and Householder's
// panel is latency-bound, so the factor comes from Gram matrices instead:
//
//   G1 = C^H C + s I   (s = 11 (m N + N (N + 1)) u ||C||_F^2)   R1 = chol(G1)   Q1 = C R1^{-1}
//   G2 = Q1^H Q1                                               R2 = chol(G2)   Q2 = Q1 R2^{-1}
//   G3 = Q2^H Q2                                               R3 = chol(G3)   R = R3 R2 R1
//
// The shift makes the first Cholesky succeed for any kappa(C) < u^{-1}; it
// leaves kappa(Q1) ~ sqrt(kappa), and two unshifted passes restore
// orthogonality: backward stable like Householder (||C - Q R|| = O(u ||C||)).
// C is never concatenated: the Gram blocks of A and B are formed separately
// and Q1 is written once.  The Gram products and triangular solves are plain
// cuBLAS level-3 calls (batched GEMM, SYRK/HERK, TRSM, TRMM); the Cholesky diagonal
// blocks are a one-CTA shared-memory kernel.  O(m N^2): 3 Gram passes + 2
// solves, ~5 m N^2 flops -- a baseline, not the sketched hot path.
#include <cublas_v2.h>

#include <cmath>
#include <mutex>
#include <vector>

#include "nsk_internal.hpp"

namespace nsk {

namespace {

constexpr int cblock(int nc) { return nc == 1 ? 64 : 32; }  // Cholesky block (32 KiB of shared memory)

struct HandleSlot {
  int device;
  cublasHandle_t h;
};

std::mutex g_cublas_mu;
std::vector<HandleSlot> g_cublas;

cublasHandle_t cublas_for(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_cublas_mu);
  cublasHandle_t h = nullptr;
  for (auto& s : g_cublas)
    if (s.device == dev) h = s.h;
  if (!h) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    g_cublas.push_back({dev, h});
  }
  cublasSetStream(h, st);
  cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST);
  return h;
}

#define NSK_CUBLAS_OK(expr)                                                         \
  do {                                                                              \
    cublasStatus_t s_ = (expr);                                                     \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                \
      return fail(ECUDA, std::string("cuBLAS error ") + std::to_string(int(s_)) + \
                             " in " #expr);                                         \
  } while (0)

// Adds s = 11 (m N + N (N + 1)) u tr(G) to the diagonal (G = C^H C, so tr G = ||C||_F^2).
__global__ void add_shift_kernel(double* G, int64_t N, int nc, double coef) {
  __shared__ double red[32];
  double t = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) t += G[(i + i * N) * nc];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double shift = coef * red[0];
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) G[(i + i * N) * nc] += shift;
}

// In-place upper Cholesky (G = R^H R) of the b x b diagonal block at (j0, j0)
// of the N x N matrix G (ld N), in shared memory.  *bad is raised on a
// non-positive or non-finite pivot.
template <int NC>
__global__ void __launch_bounds__(256) chol_block_kernel(double* G, int64_t N, int64_t j0, int b, int* bad) {
  __shared__ double T[cblock(NC) * cblock(NC) * NC];  // column-major b x b
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int r = e % b, c = e / b;
    for (int q = 0; q < NC; ++q) T[(r + c * b) * NC + q] = G[((j0 + r) + (j0 + c) * N) * NC + q];
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    const double d = T[(j + j * b) * NC];
    if (!(d > 0.0) || !isfinite(d)) {
      if (threadIdx.x == 0) atomicExch(bad, 1);
      return;
    }
    const double rjj = sqrt(d), inv = 1.0 / rjj;
    __syncthreads();
    // row j to the right of the diagonal: R[j][c] = T[j][c] / r_jj
    for (int c = j + 1 + threadIdx.x; c < b; c += blockDim.x)
      for (int q = 0; q < NC; ++q) T[(j + c * b) * NC + q] *= inv;
    if (threadIdx.x == 0) {
      T[(j + j * b) * NC] = rjj;
      if (NC == 2) T[(j + j * b) * NC + 1] = 0.0;
    }
    __syncthreads();
    // trailing upper triangle: T[r][c] -= conj(R[j][r]) R[j][c], j < r <= c
    const int w = b - j - 1;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int r = j + 1 + e % w, c = j + 1 + e / w;
      if (r > c) continue;
      if (NC == 1) {
        T[r + c * b] -= T[j + r * b] * T[j + c * b];
      } else {
        const double ar = T[2 * (j + r * b)], ai = T[2 * (j + r * b) + 1];
        const double br = T[2 * (j + c * b)], bi = T[2 * (j + c * b) + 1];
        T[2 * (r + c * b)] -= ar * br + ai * bi;  // conj(a) b
        T[2 * (r + c * b) + 1] -= ar * bi - ai * br;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int r = e % b, c = e / b;
    for (int q = 0; q < NC; ++q) G[((j0 + r) + (j0 + c) * N) * NC + q] = r <= c ? T[(r + c * b) * NC + q] : 0.0;
  }
}

// Zero the strictly lower triangle of an N x N matrix (ld N).
__global__ void zero_lower_kernel(double* R, int64_t N, int nc) {
  const int64_t total = N * N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e % N, c = e / N;
    if (r > c)
      for (int q = 0; q < nc; ++q) R[e * nc + q] = 0.0;
  }
}

// Blocked upper Cholesky of G (N x N, ld N) in place; the strictly lower part is zeroed.
int cholesky_upper(cublasHandle_t h, int nc, double* G, int64_t N, int* bad, cudaStream_t st) {
  const int CB = cblock(nc);
  for (int64_t j0 = 0; j0 < N; j0 += CB) {
    const int b = static_cast<int>(N - j0 < CB ? N - j0 : CB);
    if (nc == 1)
      chol_block_kernel<1><<<1, 256, 0, st>>>(G, N, j0, b, bad);
    else
      chol_block_kernel<2><<<1, 256, 0, st>>>(G, N, j0, b, bad);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    const int64_t rest = N - j0 - b;
    if (rest <= 0) continue;
    double* Rjj = G + (j0 + j0 * N) * nc;
    double* Rjr = G + (j0 + (j0 + b) * N) * nc;      // b x rest panel right of the block
    double* Grr = G + ((j0 + b) + (j0 + b) * N) * nc;  // trailing rest x rest
    if (nc == 1) {
      const double one = 1.0, mone = -1.0;
      NSK_CUBLAS_OK(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, b,
                                static_cast<int>(rest), &one, Rjj, static_cast<int>(N), Rjr, static_cast<int>(N)));
      NSK_CUBLAS_OK(cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, static_cast<int>(rest), b, &mone, Rjr,
                                static_cast<int>(N), &one, Grr, static_cast<int>(N)));
    } else {
      const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
      const double rone = 1.0, rmone = -1.0;
      NSK_CUBLAS_OK(cublasZtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, b,
                                static_cast<int>(rest), &one, reinterpret_cast<cuDoubleComplex*>(Rjj),
                                static_cast<int>(N), reinterpret_cast<cuDoubleComplex*>(Rjr), static_cast<int>(N)));
      NSK_CUBLAS_OK(cublasZherk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, static_cast<int>(rest), b, &rmone,
                                reinterpret_cast<cuDoubleComplex*>(Rjr), static_cast<int>(N), &rone,
                                reinterpret_cast<cuDoubleComplex*>(Grr), static_cast<int>(N)));
    }
  }
  int64_t blocks = (N * N + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  zero_lower_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(G, N, nc);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

// G[e] = sum_b P[b][e] (fixed order), e < N * N * nc.
__global__ void sum_partials_kernel(const double* __restrict__ P, int64_t elems, int batch, double* __restrict__ G) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < elems;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < batch; ++b) v += P[b * elems + e];
    G[e] = v;
  }
}

// G = Q^H Q, Q m x N (ld m).  The reduction dimension m is huge and N small,
// so a single SYRK/GEMM has only (N / tile)^2 CTAs each walking all m rows;
// instead the rows are split into chunks (a strided-batched GEMM, one
// product per chunk) and the partial Grams are summed in fixed order.
int gram(cublasHandle_t h, int nc, const double* Q, int64_t m, int64_t N, double* G, cudaStream_t st) {
  int batch = static_cast<int>(m / (8 * N));
  if (batch > 64) batch = 64;
  if (batch < 1) batch = 1;
  const int64_t chunk = m / batch, tail = m - chunk * batch;
  const int64_t elems = N * N * nc;
  Scratch ps;
  NSK_CUDA_OK(ps.alloc(sizeof(double) * elems * (batch + (tail ? 1 : 0)), st));
  double* P = ps.as<double>();
  const int n = static_cast<int>(N), ld = static_cast<int>(m);
  if (nc == 1) {
    const double one = 1.0, zero = 0.0;
    NSK_CUBLAS_OK(cublasDgemmStridedBatched(h, CUBLAS_OP_T, CUBLAS_OP_N, n, n, static_cast<int>(chunk), &one, Q, ld,
                                            chunk, Q, ld, chunk, &zero, P, n, N * N, batch));
    if (tail)
      NSK_CUBLAS_OK(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, n, n, static_cast<int>(tail), &one, Q + chunk * batch,
                                ld, Q + chunk * batch, ld, &zero, P + elems * batch, n));
  } else {
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
    const cuDoubleComplex* Qc = reinterpret_cast<const cuDoubleComplex*>(Q);
    cuDoubleComplex* Pc = reinterpret_cast<cuDoubleComplex*>(P);
    NSK_CUBLAS_OK(cublasZgemmStridedBatched(h, CUBLAS_OP_C, CUBLAS_OP_N, n, n, static_cast<int>(chunk), &one, Qc, ld,
                                            chunk, Qc, ld, chunk, &zero, Pc, n, N * N, batch));
    if (tail)
      NSK_CUBLAS_OK(cublasZgemm(h, CUBLAS_OP_C, CUBLAS_OP_N, n, n, static_cast<int>(tail), &one, Qc + chunk * batch,
                                ld, Qc + chunk * batch, ld, &zero, Pc + N * N * batch, n));
  }
  int64_t blocks = (elems + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  sum_partials_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(P, elems, batch + (tail ? 1 : 0), G);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

// Q <- Q R^{-1} (R upper N x N).
int right_solve(cublasHandle_t h, int nc, double* Q, int64_t m, int64_t N, const double* R) {
  if (nc == 1) {
    const double one = 1.0;
    NSK_CUBLAS_OK(cublasDtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                              static_cast<int>(m), static_cast<int>(N), &one, R, static_cast<int>(N), Q,
                              static_cast<int>(m)));
  } else {
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
    NSK_CUBLAS_OK(cublasZtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                              static_cast<int>(m), static_cast<int>(N), &one,
                              reinterpret_cast<const cuDoubleComplex*>(R), static_cast<int>(N),
                              reinterpret_cast<cuDoubleComplex*>(Q), static_cast<int>(m)));
  }
  return OK;
}

// Out = L * Rr (L upper N x N, Rr full N x N), out of place.
int tri_mul(cublasHandle_t h, int nc, const double* L, const double* Rr, double* Out, int64_t N) {
  const int n = static_cast<int>(N);
  if (nc == 1) {
    const double one = 1.0;
    NSK_CUBLAS_OK(cublasDtrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n,
                              &one, L, n, Rr, n, Out, n));
  } else {
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
    NSK_CUBLAS_OK(cublasZtrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n,
                              &one, reinterpret_cast<const cuDoubleComplex*>(L), n,
                              reinterpret_cast<const cuDoubleComplex*>(Rr), n, reinterpret_cast<cuDoubleComplex*>(Out),
                              n));
  }
  return OK;
}

}  // namespace

namespace {

// One sCQR3 attempt; *hb receives the breakdown flag.  shift_all also shifts
// the two re-orthogonalisation passes (exactly rank-deficient [A|B]: a zero
// direction of C gives a zero column of Q1 and an exactly singular G2).
// cols: device pointers of the N columns of C (m entries x nc each).
// cols: device pointers of the N columns of C (m entries x nc each); src: the
// array each column lives in (a 2-D copy must not span two allocations).
int tall_qr_attempt(int nc, int64_t m, const std::vector<const double*>& cols, const std::vector<int>& src,
                    double* R, bool shift_all, int* hb, cudaStream_t st) {
  const int64_t N = static_cast<int64_t>(cols.size());
  cublasHandle_t h = cublas_for(st);
  if (!h) return fail(ECUDA, "tall QR: cublasCreate failed");
  Scratch qs, gs;
  const size_t qbytes = sizeof(double) * m * N * nc, gbytes = sizeof(double) * N * N * nc;
  NSK_CUDA_OK(qs.alloc(qbytes, st));
  NSK_CUDA_OK(gs.alloc(3 * gbytes + 64, st));
  double* Q = qs.as<double>();
  double* G = gs.as<double>();
  double* R1 = G + N * N * nc;
  double* T = R1 + N * N * nc;
  int* bad = reinterpret_cast<int*>(T + N * N * nc);
  NSK_CUDA_OK(cudaMemsetAsync(bad, 0, sizeof(int), st));
  // Q <- C (column runs with a common stride are one 2-D copy)
  for (int64_t j = 0; j < N;) {
    int64_t e = j + 1;
    int64_t stride = e < N && src[e] == src[j] ? cols[e] - cols[j] : m * nc;
    if (stride < m * nc) stride = m * nc;  // not a forward run: column j alone
    else
      while (e < N && src[e] == src[j] && cols[e] - cols[e - 1] == stride) ++e;
    const cudaError_t ce = cudaMemcpy2DAsync(Q + j * m * nc, sizeof(double) * m * nc, cols[j], sizeof(double) * stride,
                                             sizeof(double) * m * nc, e - j, cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess)
      return fail(ECUDA, std::string("tall QR: copy of columns ") + std::to_string(j) + ".." + std::to_string(e) +
                             " (m " + std::to_string(m) + ", pitch " + std::to_string(stride) + "): " +
                             cudaGetErrorString(ce));
    j = e;
  }
  const double u = 1.1102230246251565e-16;
  const double coef = 11.0 * (static_cast<double>(m) * N + static_cast<double>(N) * (N + 1)) * u;
  auto shift = [&](double* Gm) -> int {
    add_shift_kernel<<<1, 256, 0, st>>>(Gm, N, nc, coef);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    return OK;
  };
  // 1. shifted pass: R1 = chol(C^H C + s I), Q1 = C R1^{-1}
  if (int rc = gram(h, nc, Q, m, N, R1, st)) return rc;
  if (int rc = shift(R1)) return rc;
  if (int rc = cholesky_upper(h, nc, R1, N, bad, st)) return rc;
  if (int rc = right_solve(h, nc, Q, m, N, R1)) return rc;
  // 2. R2 = chol(Q1^H Q1), Q2 = Q1 R2^{-1}
  if (int rc = gram(h, nc, Q, m, N, G, st)) return rc;
  if (shift_all)
    if (int rc = shift(G)) return rc;
  if (int rc = cholesky_upper(h, nc, G, N, bad, st)) return rc;
  if (int rc = right_solve(h, nc, Q, m, N, G)) return rc;
  if (int rc = tri_mul(h, nc, G, R1, T, N)) return rc;  // T = R2 R1
  // 3. R3 = chol(Q2^H Q2); R = R3 R2 R1
  if (int rc = gram(h, nc, Q, m, N, G, st)) return rc;
  if (shift_all)
    if (int rc = shift(G)) return rc;
  if (int rc = cholesky_upper(h, nc, G, N, bad, st)) return rc;
  if (int rc = tri_mul(h, nc, G, T, R, N)) return rc;
  NSK_CUDA_OK(cudaMemcpyAsync(hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return OK;
}

}  // namespace

// nz[j] = 1 when column j (m x nc, stride ld) has a non-zero entry.
__global__ void nonzero_columns_kernel(const double* __restrict__ C, int64_t m, int64_t ld, int nc, int* __restrict__ nz) {
  const double* c = C + blockIdx.x * ld * nc;
  int any = 0;
  for (int64_t e = threadIdx.x; e < m * nc && !any; e += blockDim.x) any = c[e] != 0.0;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) nz[blockIdx.x] = any;
}

int tall_qr_r(int nc, int64_t m, int64_t n, const double* A, int64_t lda, int64_t k, const double* B, int64_t ldb,
              double* R, cudaStream_t st) {
  const int64_t N = n + k;
  if (N < 1 || m < N) return fail(EINVAL_, "tall QR: need m >= n + k >= 1");
  if (m > 0x7fffffff || N > 0x7fffffff) return fail(EINVAL_, "tall QR: dimensions exceed the cuBLAS int range");
  // Exactly zero columns factor as exactly zero columns of R (as Householder
  // gives): they are left out of the Gram passes, which need a definite C.
  Scratch zs;
  NSK_CUDA_OK(zs.alloc(sizeof(int) * N, st));
  nonzero_columns_kernel<<<static_cast<unsigned>(n), 256, 0, st>>>(A, m, lda, nc, zs.as<int>());
  if (k > 0) nonzero_columns_kernel<<<static_cast<unsigned>(k), 256, 0, st>>>(B, m, ldb, nc, zs.as<int>() + n);
  count_launch(k > 0 ? 2 : 1);
  NSK_CUDA_OK(cudaGetLastError());
  std::vector<int> nz(static_cast<size_t>(N));
  NSK_CUDA_OK(cudaMemcpyAsync(nz.data(), zs.p, sizeof(int) * N, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  std::vector<const double*> cols;
  std::vector<int> src;
  std::vector<int64_t> where;
  for (int64_t j = 0; j < N; ++j)
    if (nz[static_cast<size_t>(j)]) {
      cols.push_back(j < n ? A + j * lda * nc : B + (j - n) * ldb * nc);
      src.push_back(j < n ? 0 : 1);
      where.push_back(j);
    }
  const int64_t Nz = static_cast<int64_t>(cols.size());
  double* Rz = R;
  Scratch rs;
  if (Nz < N) {
    NSK_CUDA_OK(cudaMemsetAsync(R, 0, sizeof(double) * N * N * nc, st));
    if (Nz == 0) return OK;
    NSK_CUDA_OK(rs.alloc(sizeof(double) * Nz * Nz * nc, st));
    Rz = rs.as<double>();
  }
  int hb = 0;
  if (int rc = tall_qr_attempt(nc, m, cols, src, Rz, false, &hb, st)) return rc;
  if (hb) {  // exactly rank-deficient C: shift every pass
    hb = 0;
    if (int rc = tall_qr_attempt(nc, m, cols, src, Rz, true, &hb, st)) return rc;
  }
  if (hb) return fail(ENOCONV, "tall QR: Cholesky breakdown (input contains NaN/Inf)");
  if (Nz < N)  // R[0:Nz, where[c]] = Rz[:, c]: R^H R = C^H C with zero columns in place
    for (int64_t c = 0; c < Nz; ++c)
      NSK_CUDA_OK(cudaMemcpyAsync(R + where[static_cast<size_t>(c)] * N * nc, Rz + c * Nz * nc,
                                  sizeof(double) * Nz * nc, cudaMemcpyDeviceToDevice, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return OK;
}

}  // namespace nsk
