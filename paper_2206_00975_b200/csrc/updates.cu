// updates.cu -- incremental sketch maintenance and the sketched TLS solve.
//
// Reference (/root/reference/proj/src/sketch.cpp):
//   sketch_vector(j)  sketch.cpp:130-160   column j of S (closed form, O(s))
//   update_column     sketch.cpp:234-257   sketch of a new column, zeroed rows forced 0
//   update_row        sketch.cpp:268-280   SA += g a_row / sqrt(s), g fresh from stream (seed, 1)
//   downdate_row      sketch.cpp:283-301   SA -= (S e_j) a_row_j, then row j is zeroed
// and tls_solve_sketched (/root/reference/proj/src/tls.cpp:97-113).
//
// All arithmetic runs on the device: the column S e_j is regenerated from the
// counter-based stream (gaussian / appended columns) or from the closed-form
// transform entry with exact integer argument reduction (srft, srdct, srht),
// and the rank-one update is one streaming kernel over SA.
#include <cmath>

#include "nsk_internal.hpp"

namespace nsk {
namespace {

struct ColParams {
  int kind;
  int64_t s, m, j;
  PhiloxKey key0, key1;
  const int64_t* idx;       // srft/srdct/srht sample
  uint32_t cs_entry_bucket; // countsketch bucket of row j
  double cs_sign;
};

__global__ void sketch_column_kernel(ColParams p, double* __restrict__ out, int ncomp) {
  const double inv_sqrt_s = 1.0 / sqrt(static_cast<double>(p.s));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < p.s;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double re = 0.0, im = 0.0;
    if (p.j >= p.m) {  // appended column: Gaussians #((j-m)*s + i) of stream (seed, 1)
      re = inv_sqrt_s * gaussian_at(p.key1, static_cast<uint64_t>(p.j - p.m) * p.s + i);
    } else if (p.kind == GAUSSIAN) {
      re = inv_sqrt_s * gaussian_at(p.key0, static_cast<uint64_t>(p.j) * p.s + i);
    } else if (p.kind == COUNTSKETCH) {
      re = (static_cast<int64_t>(p.cs_entry_bucket) == i) ? p.cs_sign : 0.0;
    } else {
      const double d = (stream_word(p.key0, static_cast<uint64_t>(p.j)) & 1u) ? 1.0 : -1.0;
      const uint64_t a = static_cast<uint64_t>(p.idx[i]), j = static_cast<uint64_t>(p.j),
                     m = static_cast<uint64_t>(p.m);
      if (p.kind == SRFT) {  // sqrt(m/s) * d_j * e^{2 pi i a j / m} / sqrt(m)  (transforms.cpp:66-72)
        const uint64_t r = static_cast<uint64_t>((static_cast<unsigned __int128>(a) * j) % m);
        double sn, cs;
        sincospi(2.0 * static_cast<double>(r) / static_cast<double>(m), &sn, &cs);
        re = inv_sqrt_s * d * cs;
        im = inv_sqrt_s * d * sn;
      } else if (p.kind == SRDCT) {  // sqrt(m/s) d_j c_j cos(pi j (2a+1) / 2m)  (transforms.cpp:74-80)
        const uint64_t r = static_cast<uint64_t>((static_cast<unsigned __int128>(j) * (2 * a + 1)) % (4 * m));
        const double cj = j == 0 ? sqrt(1.0 / static_cast<double>(m)) : sqrt(2.0 / static_cast<double>(m));
        re = sqrt(static_cast<double>(m) / static_cast<double>(p.s)) * d * cj *
             cospi(static_cast<double>(r) / (2.0 * static_cast<double>(m)));
      } else {  // SRHT: (1/sqrt s) d_j (-1)^popc(a & j)
        re = inv_sqrt_s * d * ((__popcll(a & j) & 1) ? -1.0 : 1.0);
      }
    }
    if (ncomp == 1) {
      out[i] = re;
    } else {
      out[2 * i] = re;
      out[2 * i + 1] = im;
    }
  }
}

__global__ void rank1_kernel(double* __restrict__ SA, int64_t ldsa, int ncsa, int64_t s, int64_t n,
                             const double* __restrict__ col, int nccol, const double* __restrict__ row, int ncrow,
                             double alpha) {
  const int64_t total = s * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % s, c = e / s;
    const double cr = col[i * nccol], ci = nccol == 2 ? col[2 * i + 1] : 0.0;
    const double rr = row[c * ncrow], ri = ncrow == 2 ? row[2 * c + 1] : 0.0;
    const double pr = cr * rr - ci * ri, pi = cr * ri + ci * rr;
    if (ncsa == 1) {
      SA[i + c * ldsa] += alpha * pr;
    } else {
      SA[2 * (i + c * ldsa)] += alpha * pr;
      SA[2 * (i + c * ldsa) + 1] += alpha * pi;
    }
  }
}

__global__ void accumulate_kernel(double* __restrict__ SA, int64_t ldsa, int ncsa, const double* __restrict__ T,
                                  int64_t s, int64_t n, int nct) {
  const int64_t total = s * n * nct;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t part = e % nct, rest = e / nct, i = rest % s, c = rest / s;
    SA[(i + c * ldsa) * ncsa + part] += T[e];
  }
}

__global__ void mask_kernel(double* __restrict__ col, int nc, const int64_t* __restrict__ rows, int64_t nz) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = rows[e];
    col[r * nc] = 0.0;
    if (nc == 2) col[r * nc + 1] = 0.0;
  }
}

unsigned grid_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  if (b < 1) b = 1;
  if (b > 8L * sm_count()) b = 8L * sm_count();
  return static_cast<unsigned>(b);
}

}  // namespace

int sketch_column(const Operator& op, int64_t j, double* out, int ncomp_out, cudaStream_t st) {
  const DeviceTables* tb = op.tables(0, 0);  // the sample indices only (no CountSketch row window)
  if (!tb) return ECUDA;
  ColParams p{op.kind, op.s, op.m, j, op.key0, op.key1, tb->idx, 0u, 1.0};
  if (op.kind == COUNTSKETCH && j < op.m) {  // h(j) = below(s) of words m+2j, m+2j+1; sigma(j) = word j
    auto word = [&](uint64_t w) {
      uint64_t ctr = w >> 2;
      uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32), c2 = 0, c3 = 0;
      uint32_t k0 = op.key0.k0, k1 = op.key0.k1;
      for (int r = 0; r < 10; ++r) {
        uint64_t p0 = 0xD2511F53ULL * c0, p1 = 0xCD9E8D57ULL * c2;
        uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0, n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
        c1 = static_cast<uint32_t>(p1);
        c3 = static_cast<uint32_t>(p0);
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      const uint32_t ws[4] = {c0, c1, c2, c3};
      return ws[w & 3];
    };
    const uint64_t w = static_cast<uint64_t>(op.m) + 2u * static_cast<uint64_t>(j);
    const uint64_t u = (static_cast<uint64_t>(word(w + 1)) << 32) | word(w);
    p.cs_entry_bucket = static_cast<uint32_t>((static_cast<unsigned __int128>(u) * static_cast<uint64_t>(op.s)) >> 64);
    p.cs_sign = (word(static_cast<uint64_t>(j)) & 1u) ? 1.0 : -1.0;
  }
  sketch_column_kernel<<<grid_for(op.s), 256, 0, st>>>(p, out, ncomp_out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

int rank1_update(double* SA, int64_t ldsa, int ncomp_sa, int64_t s, int64_t n, const double* col, int ncomp_col,
                 const double* row, int ncomp_row, double alpha, cudaStream_t st) {
  if (s * n == 0) return OK;
  rank1_kernel<<<grid_for(s * n), 256, 0, st>>>(SA, ldsa, ncomp_sa, s, n, col, ncomp_col, row, ncomp_row, alpha);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

int accumulate(double* SA, int64_t ldsa, int ncomp_sa, const double* T, int64_t s, int64_t n, int ncomp_t,
               cudaStream_t st) {
  if (s * n == 0) return OK;
  accumulate_kernel<<<grid_for(s * n * ncomp_t), 256, 0, st>>>(SA, ldsa, ncomp_sa, T, s, n, ncomp_t);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

int mask_zeroed(const Operator& op, double* col, int ncomp, cudaStream_t st) {
  if (op.zeroed.empty()) return OK;
  Scratch rows;
  NSK_CUDA_OK(rows.alloc(sizeof(int64_t) * op.zeroed.size(), st));
  NSK_CUDA_OK(cudaMemcpyAsync(rows.p, op.zeroed.data(), sizeof(int64_t) * op.zeroed.size(), cudaMemcpyHostToDevice, st));
  mask_kernel<<<grid_for(static_cast<int64_t>(op.zeroed.size())), 256, 0, st>>>(
      col, ncomp, rows.as<int64_t>(), static_cast<int64_t>(op.zeroed.size()));
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(st));  // the host vector may change after return
  return OK;
}

// ---- TLS corner solve: X = -V1 V2^{-1} (tls.cpp:26-43) ---------------------
// One CTA: LU with partial pivoting of V2^T (k x k) in shared memory, then one
// thread per row i of X solves V2^T x_i^T = -v1_i^T.  Plain transpose (not
// conjugate) as in the reference, so the complex case matches it too.
namespace {
template <int NC>
__global__ void tls_corner_kernel(const double* __restrict__ Vk, int64_t ldv, int64_t n, int64_t k,
                                  double* __restrict__ X, int64_t ldx, int* singular) {
  extern __shared__ double lu[];  // (k x k) x NC, column-major: lu[r + c k] = V2^T(r, c) = V2(c, r)
  __shared__ int piv[256];
  for (int64_t e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int64_t r = e % k, c = e / k;
    const int64_t src = (n + c) + r * ldv;  // V2(c, r) = Vk(n + c, r)
    for (int q = 0; q < NC; ++q) lu[e * NC + q] = Vk[src * NC + q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t j = 0; j < k; ++j) {  // partial pivoting on column j
      int64_t pr = j;
      double best = -1.0;
      for (int64_t r = j; r < k; ++r) {
        const double re = lu[(r + j * k) * NC], im = NC == 2 ? lu[(r + j * k) * NC + 1] : 0.0;
        const double a = re * re + im * im;
        if (a > best) {
          best = a;
          pr = r;
        }
      }
      piv[j] = static_cast<int>(pr);
      if (best == 0.0) {
        *singular = 1;
        continue;
      }
      if (pr != j)
        for (int64_t c = 0; c < k; ++c)
          for (int q = 0; q < NC; ++q) {
            const double t = lu[(j + c * k) * NC + q];
            lu[(j + c * k) * NC + q] = lu[(pr + c * k) * NC + q];
            lu[(pr + c * k) * NC + q] = t;
          }
      const double dr = lu[(j + j * k) * NC], di = NC == 2 ? lu[(j + j * k) * NC + 1] : 0.0;
      const double den = dr * dr + di * di;
      for (int64_t r = j + 1; r < k; ++r) {
        const double ar = lu[(r + j * k) * NC], ai = NC == 2 ? lu[(r + j * k) * NC + 1] : 0.0;
        const double lr = (ar * dr + ai * di) / den, li = (ai * dr - ar * di) / den;  // a / d
        lu[(r + j * k) * NC] = lr;
        if (NC == 2) lu[(r + j * k) * NC + 1] = li;
        for (int64_t c = j + 1; c < k; ++c) {
          const double ur = lu[(j + c * k) * NC], ui = NC == 2 ? lu[(j + c * k) * NC + 1] : 0.0;
          lu[(r + c * k) * NC] -= lr * ur - li * ui;
          if (NC == 2) lu[(r + c * k) * NC + 1] -= lr * ui + li * ur;
        }
      }
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    // b = -v1_i^T (k entries), permuted; forward (unit L) then backward (U).
    double b[64][NC];
    for (int64_t c = 0; c < k; ++c)
      for (int q = 0; q < NC; ++q) b[c][q] = -Vk[(i + c * ldv) * NC + q];
    // The factor stores L with every later row interchange applied (whole rows are swapped, as
    // LAPACK's getrf does), so P b is formed completely before the forward substitution.
    for (int64_t j = 0; j < k; ++j) {
      const int p = piv[j];
      if (p != j)
        for (int q = 0; q < NC; ++q) {
          const double t = b[j][q];
          b[j][q] = b[p][q];
          b[p][q] = t;
        }
    }
    for (int64_t j = 0; j < k; ++j) {
      for (int64_t r = j + 1; r < k; ++r) {
        const double lr = lu[(r + j * k) * NC], li = NC == 2 ? lu[(r + j * k) * NC + 1] : 0.0;
        b[r][0] -= lr * b[j][0] - (NC == 2 ? li * b[j][NC - 1] : 0.0);
        if (NC == 2) b[r][1] -= lr * b[j][1] + li * b[j][0];
      }
    }
    for (int64_t j = k - 1; j >= 0; --j) {
      double xr = b[j][0], xi = NC == 2 ? b[j][NC - 1] : 0.0;
      for (int64_t c = j + 1; c < k; ++c) {
        const double ur = lu[(j + c * k) * NC], ui = NC == 2 ? lu[(j + c * k) * NC + 1] : 0.0;
        const double br = b[c][0], bi = NC == 2 ? b[c][NC - 1] : 0.0;
        xr -= ur * br - ui * bi;
        xi -= ur * bi + ui * br;
      }
      const double dr = lu[(j + j * k) * NC], di = NC == 2 ? lu[(j + j * k) * NC + 1] : 0.0;
      const double den = dr * dr + di * di;
      b[j][0] = (xr * dr + xi * di) / den;
      if (NC == 2) b[j][1] = (xi * dr - xr * di) / den;
    }
    for (int64_t c = 0; c < k; ++c)
      for (int q = 0; q < NC; ++q) X[(i + c * ldx) * NC + q] = b[c][q];
  }
}
}  // namespace

int tls_corner(int ncomp, const double* Vk, int64_t ldv, int64_t n, int64_t k, double* X, int64_t ldx,
               cudaStream_t st) {
  if (k > 64) return fail(EINVAL_, "tls: this build supports at most 64 right-hand sides");
  Scratch flag;
  NSK_CUDA_OK(flag.alloc(sizeof(int), st));
  NSK_CUDA_OK(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
  const size_t smem = sizeof(double) * k * k * ncomp;
  if (ncomp == 1) {
    NSK_CUDA_OK(cudaFuncSetAttribute(tls_corner_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    tls_corner_kernel<1><<<1, 128, smem, st>>>(Vk, ldv, n, k, X, ldx, flag.as<int>());
  } else {
    NSK_CUDA_OK(cudaFuncSetAttribute(tls_corner_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));  // complex k = 64: 64 KiB
    tls_corner_kernel<2><<<1, 128, smem, st>>>(Vk, ldv, n, k, X, ldx, flag.as<int>());
  }
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  int host = 0;
  NSK_CUDA_OK(cudaMemcpyAsync(&host, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  if (host) return fail(EINVAL_, "tls: V_k2 is singular");
  return OK;
}

}  // namespace nsk
