// srtt_sketch.cu -- K2: subsampled trigonometric transforms (srdct, srft).
//
// Reference: apply(), srft branch (/root/reference/proj/src/sketch.cpp:206-217,
// transforms.cpp:17-36) and srdct branch (sketch.cpp:218-229,
// transforms.cpp:38-64):
//   srft : SA = sqrt(m/s) R F^* D A,  F^*[a, j] = exp(+2 pi i a j / m) / sqrt(m)
//   srdct: SA = sqrt(m/s) R C D A,    C[a, j] = c_j cos(pi j (2a+1) / (2m)),
//          c_0 = sqrt(1/m), c_j = sqrt(2/m)   (orthonormal DCT-III)
// The reference transforms all m rows with FFTW and keeps s of them; only
// the s sampled outputs are needed, so the B200 path never forms the full
// transform.
//
// This file holds the direct evaluator (exact integer argument reduction,
// one thread per output entry), used for small problems and as the shard
// fallback, and the blocked fast path (srtt_fast.cuh).
#include "nsk_internal.hpp"

namespace nsk {

int srtt_tile_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                    double* SA, int64_t ldsa, cudaStream_t st);
int srtt_fast_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                    int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srft_ws_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                  double* SA, int64_t ldsa, cudaStream_t st);
int srdct_stream_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda, double* SA,
                       int64_t ldsa, cudaStream_t st);

namespace {

// srdct: SA[r, c] = sqrt(m/s) * sum_j c_j cos(pi j (2 idx_r + 1) / 2m) d_j A[j, c].
__global__ void srdct_direct(const double* __restrict__ A, int64_t lda, RowMap rows, int64_t n,
                             const int64_t* __restrict__ idx, int64_t s, int64_t m, PhiloxKey key,
                             double* __restrict__ SA, int64_t ldsa) {
  const double scale = sqrt(static_cast<double>(m) / static_cast<double>(s));
  const double c0 = sqrt(1.0 / static_cast<double>(m)), c1 = sqrt(2.0 / static_cast<double>(m));
  const uint64_t four_m = 4u * static_cast<uint64_t>(m);
  const double inv_2m = 1.0 / (2.0 * static_cast<double>(m));
  const int64_t total = s * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / s, r = e % s;
    const uint64_t odd = 2u * static_cast<uint64_t>(idx[r]) + 1u;
    double v = 0.0;
    for (int64_t j = 0; j < rows.mloc; ++j) {
      const uint64_t g = static_cast<uint64_t>(rows.row0 + rows.rstep * j);
      const uint64_t k = static_cast<uint64_t>((static_cast<unsigned __int128>(g) * odd) % four_m);
      const double w = (g == 0 ? c0 : c1) * cospi(static_cast<double>(k) * inv_2m);
      v = fma(w, apply_sign(A[j + c * lda], stream_word(key, g)), v);
    }
    SA[r + c * ldsa] = scale * v;
  }
}

// srft: SA[r, c] = (1/sqrt s) * sum_j exp(2 pi i (idx_r j mod m) / m) d_j A[j, c].
template <int NCIN>
__global__ void srft_direct(const double* __restrict__ A, int64_t lda, RowMap rows, int64_t n,
                            const int64_t* __restrict__ idx, int64_t s, int64_t m, PhiloxKey key,
                            double* __restrict__ SA, int64_t ldsa) {
  const double scale = 1.0 / sqrt(static_cast<double>(s));
  const double two_over_m = 2.0 / static_cast<double>(m);
  const int64_t total = s * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / s, r = e % s;
    const uint64_t a = static_cast<uint64_t>(idx[r]);
    double vr = 0.0, vi = 0.0;
    for (int64_t j = 0; j < rows.mloc; ++j) {
      const uint64_t g = static_cast<uint64_t>(rows.row0 + rows.rstep * j);
      const uint64_t k = static_cast<uint64_t>((static_cast<unsigned __int128>(g) * a) % static_cast<uint64_t>(m));
      double sn, cs;
      sincospi(static_cast<double>(k) * two_over_m, &sn, &cs);
      const uint32_t w = stream_word(key, g);
      double xr, xi;
      if (NCIN == 1) {
        xr = apply_sign(A[j + c * lda], w);
        xi = 0.0;
      } else {
        xr = apply_sign(A[2 * (j + c * lda)], w);
        xi = apply_sign(A[2 * (j + c * lda) + 1], w);
      }
      vr += cs * xr - sn * xi;
      vi += cs * xi + sn * xr;
    }
    SA[2 * (r + c * ldsa)] = scale * vr;
    SA[2 * (r + c * ldsa) + 1] = scale * vi;
  }
}

}  // namespace

int srtt_direct_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                      int64_t lda, double* SA, int64_t ldsa, cudaStream_t st) {
  const DeviceTables* tb = op.tables();
  if (!tb) return ECUDA;
  const int64_t total = op.s * n;
  if (total == 0) return OK;
  int64_t blocks = (total + 127) / 128;
  if (blocks > 16L * sm_count()) blocks = 16L * sm_count();
  KernelTimer tm(st, op.kind == SRDCT ? "srdct_direct" : "srft_direct");
  count_launch();
  if (op.kind == SRDCT) {
    srdct_direct<<<static_cast<unsigned>(blocks), 128, 0, st>>>(A, lda, rows, n, tb->idx, op.s, op.m, op.key0,
                                                                 SA, ldsa);
  } else if (ncomp == 1) {
    srft_direct<1><<<static_cast<unsigned>(blocks), 128, 0, st>>>(A, lda, rows, n, tb->idx, op.s, op.m, op.key0,
                                                                  SA, ldsa);
  } else {
    srft_direct<2><<<static_cast<unsigned>(blocks), 128, 0, st>>>(A, lda, rows, n, tb->idx, op.s, op.m, op.key0,
                                                                  SA, ldsa);
  }
  tm.stop();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

int srtt_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
               double* SA, int64_t ldsa, cudaStream_t st) {
  // srdct: register-streamed Makhoul tiles (srdct_stream.cu), srft of a real A:
  // warp-specialised tiles (srft_ws.cu), both for m % 16384 == 0; then the
  // tiled single-pass FFT (srtt_tile.cu: complex srft input, m % 4096 == 0
  // srdct), else the strided FFT / cyclic shards (srtt_fast.cu), else the
  // general-length engine (srtt_general.cu), else the direct evaluator.
  if (op.kind == SRDCT && ncomp == 1) {
    const int rsd = srdct_stream_apply(op, rows, n, A, lda, SA, ldsa, st);
    if (rsd != NOTAPPLICABLE) return rsd;
  }
  if (op.kind == SRFT && ncomp == 1) {
    const int rw = srft_ws_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
    if (rw != NOTAPPLICABLE) return rw;
  }
  const int rc = srtt_tile_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
  if (rc != NOTAPPLICABLE) return rc;
  return srtt_fast_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
}

}  // namespace nsk
