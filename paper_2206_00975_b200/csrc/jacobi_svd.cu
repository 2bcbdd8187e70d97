// jacobi_svd.cu -- K4: trailing right singular vectors of SA on the device.
//
// Reference: from_sketch_svd (/root/reference/proj/src/nullspace.cpp:10-19)
// runs Eigen BDCSVD (kernels.cpp:14-22) on the s x n sketch and returns
// W = V(:, n-k : n-1) plus all n singular values, non-increasing; failure to
// converge raises SvdConvergenceError (kernels.hpp:18-20).
//
// B200 design: one-sided (Hestenes) Jacobi on a working copy U = SA with V
// accumulated from I, in ONE cooperative persistent kernel.  Each sweep runs
// the n-1 rounds of a round-robin (circle) tournament; the n/2 disjoint
// column pairs of a round are spread over the CTAs, and a grid-wide barrier
// separates rounds.  Columns are staged in shared memory, the three inner
// products are block reductions in fixed order, complex pairs are first
// phase-aligned (u_q *= e^{-i arg c}) and then rotated by the real Jacobi
// rotation.  Convergence: a sweep with no rotation, i.e. every pair has
// |u_p^H u_q| <= tol * ||u_p|| ||u_q||.  One-sided Jacobi computes small
// singular values to high relative accuracy, which the 1e-10 .. 1e-12
// trailing values of the BASELINE configs need.
#include <cooperative_groups.h>

#include "nsk_internal.hpp"

namespace cg = cooperative_groups;

namespace nsk {
namespace {

constexpr int JT = 256;
constexpr int MAX_SWEEPS = 40;

struct JacobiParams {
  double* U;       // s x n (x ncomp), ld = s
  double* V;       // n x n (x ncomp), ld = n
  int64_t s, n, N; // N = n rounded up to even
  double tol;
  int* counter;    // [MAX_SWEEPS + 1] rotations per sweep; [MAX_SWEEPS+1] = sweeps done
  int use_smem;
};

template <int NC>
__device__ __forceinline__ void block_sum4(double& a, double& b, double& c, double& d, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
    if (NC == 2) d += __shfl_xor_sync(0xffffffffu, d, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    red[w * 4 + 0] = a;
    red[w * 4 + 1] = b;
    red[w * 4 + 2] = c;
    red[w * 4 + 3] = d;
  }
  __syncthreads();
  a = b = c = d = 0.0;
  for (int i = 0; i < JT / 32; ++i) {  // fixed order: deterministic
    a += red[i * 4 + 0];
    b += red[i * 4 + 1];
    c += red[i * 4 + 2];
    d += red[i * 4 + 3];
  }
}

__device__ __forceinline__ void pair_of_round(int64_t N, int64_t r, int64_t i, int64_t& p, int64_t& q) {
  const int64_t M = N - 1;
  if (i == 0) {
    p = M;
    q = r;
  } else {
    p = (r + i) % M;
    q = (r - i + M) % M;
  }
  if (p > q) {
    const int64_t t = p;
    p = q;
    q = t;
  }
}

// Rotate columns p, q of X (rows x ld) by (cs, sn) after phase (ph_re, ph_im) on q.
template <int NC>
__device__ __forceinline__ void rotate_cols(double* X, int64_t ld, int64_t rows, int64_t p, int64_t q, double cs,
                                            double sn, double ph_re, double ph_im, const double* cp,
                                            const double* cq) {
  for (int64_t i = threadIdx.x; i < rows; i += JT) {
    if (NC == 1) {
      const double up = cp ? cp[i] : X[i + p * ld];
      const double uq = cq ? cq[i] : X[i + q * ld];
      X[i + p * ld] = cs * up - sn * uq;
      X[i + q * ld] = sn * up + cs * uq;
    } else {
      const double pr = cp ? cp[2 * i] : X[2 * (i + p * ld)];
      const double pi = cp ? cp[2 * i + 1] : X[2 * (i + p * ld) + 1];
      const double qr0 = cq ? cq[2 * i] : X[2 * (i + q * ld)];
      const double qi0 = cq ? cq[2 * i + 1] : X[2 * (i + q * ld) + 1];
      const double qr = qr0 * ph_re - qi0 * ph_im;  // u_q * e^{-i phi}
      const double qi = qr0 * ph_im + qi0 * ph_re;
      X[2 * (i + p * ld)] = cs * pr - sn * qr;
      X[2 * (i + p * ld) + 1] = cs * pi - sn * qi;
      X[2 * (i + q * ld)] = sn * pr + cs * qr;
      X[2 * (i + q * ld) + 1] = sn * pi + cs * qi;
    }
  }
}

template <int NC>
__global__ void __launch_bounds__(JT) jacobi_kernel(JacobiParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double cache[];  // [2][s*NC] when use_smem
  __shared__ double red[(JT / 32) * 4];
  const int64_t s = P.s, n = P.n, N = P.N;
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int64_t r = 0; r < N - 1; ++r) {
      for (int64_t i = blockIdx.x; i < N / 2; i += gridDim.x) {
        int64_t p, q;
        pair_of_round(N, r, i, p, q);
        if (q >= n) continue;  // dummy column for odd n
        double a = 0, b = 0, cr = 0, ci = 0;
        double* cp = P.use_smem ? cache : nullptr;
        double* cq = P.use_smem ? cache + s * NC : nullptr;
        for (int64_t row = threadIdx.x; row < s; row += JT) {
          if (NC == 1) {
            const double up = P.U[row + p * s], uq = P.U[row + q * s];
            if (cp) {
              cp[row] = up;
              cq[row] = uq;
            }
            a += up * up;
            b += uq * uq;
            cr += up * uq;
          } else {
            const double pr = P.U[2 * (row + p * s)], pi = P.U[2 * (row + p * s) + 1];
            const double qr = P.U[2 * (row + q * s)], qi = P.U[2 * (row + q * s) + 1];
            if (cp) {
              cp[2 * row] = pr;
              cp[2 * row + 1] = pi;
              cq[2 * row] = qr;
              cq[2 * row + 1] = qi;
            }
            a += pr * pr + pi * pi;
            b += qr * qr + qi * qi;
            cr += pr * qr + pi * qi;  // conj(u_p) u_q
            ci += pr * qi - pi * qr;
          }
        }
        block_sum4<NC>(a, b, cr, ci, red);
        const double cabs = NC == 1 ? fabs(cr) : hypot(cr, ci);
        if (cabs > P.tol * sqrt(a) * sqrt(b) && cabs > 0.0) {
          // Real pairs keep the sign of u_p^T u_q; complex pairs were phase-aligned
          // so that their inner product is the positive real |c|.
          const double zeta = (b - a) / (2.0 * (NC == 1 ? cr : cabs));
          double t;
          if (fabs(zeta) > 1e150)
            t = 0.5 / zeta;
          else
            t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          double ph_re = 1.0, ph_im = 0.0;
          if (NC == 2) {
            ph_re = cr / cabs;
            ph_im = -ci / cabs;  // e^{-i phi}
          }
          if (threadIdx.x == 0) atomicAdd(P.counter + sweep, 1);
          rotate_cols<NC>(P.U, s, s, p, q, cs, sn, ph_re, ph_im, cp, cq);
          __syncthreads();
          rotate_cols<NC>(P.V, n, n, p, q, cs, sn, ph_re, ph_im, nullptr, nullptr);
        }
        __syncthreads();
      }
      grid.sync();
    }
    const int rot = *reinterpret_cast<volatile int*>(P.counter + sweep);
    if (rot == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.counter[MAX_SWEEPS] = sweep;
}

// sigma_j = ||u_j||; order by non-increasing sigma (ties: lower index first);
// W(:, t) = V(:, order[n-k+t]).
template <int NC>
__global__ void finish_kernel(const double* __restrict__ U, const double* __restrict__ V, int64_t s, int64_t n,
                              int64_t k, double* __restrict__ W, int64_t ldw, double* __restrict__ sigma,
                              double* __restrict__ norms, int* __restrict__ order) {
  // one CTA per column for the norms
  const int64_t j = blockIdx.x;
  __shared__ double red[JT / 32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < s; i += JT) {
    if (NC == 1) {
      const double u = U[i + j * s];
      acc += u * u;
    } else {
      const double ur = U[2 * (i + j * s)], ui = U[2 * (i + j * s) + 1];
      acc += ur * ur + ui * ui;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < JT / 32; ++w) t += red[w];
    norms[j] = sqrt(t);
  }
}

template <int NC>
__global__ void order_kernel(const double* __restrict__ V, int64_t n, int64_t k, double* __restrict__ W,
                             int64_t ldw, double* __restrict__ sigma, const double* __restrict__ norms,
                             int* __restrict__ bad) {
  extern __shared__ int pos_of[];  // rank -> column
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double v = norms[j];
    if (!(v == v) || isinf(v)) atomicExch(bad, 1);
    int64_t rank = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double w = norms[i];
      rank += (w > v) || (w == v && i < j);
    }
    pos_of[rank] = static_cast<int>(j);
    sigma[rank] = v;
  }
  __syncthreads();
  for (int64_t t = 0; t < k; ++t) {
    const int64_t col = pos_of[n - k + t];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      if (NC == 1)
        W[i + t * ldw] = V[i + col * n];
      else {
        W[2 * (i + t * ldw)] = V[2 * (i + col * n)];
        W[2 * (i + t * ldw) + 1] = V[2 * (i + col * n) + 1];
      }
    }
  }
}

__global__ void init_kernel(const double* __restrict__ SA, int64_t ldsa, int64_t s, int64_t n, int nc,
                            double* __restrict__ U, double* __restrict__ V, int* counter) {
  const int64_t tot = s * n * nc, vt = n * n * nc;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot + vt;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (e < tot) {
      const int64_t c = e / (s * nc), rem = e % (s * nc);
      U[e] = SA[c * ldsa * nc + rem];
    } else {
      const int64_t f = e - tot;
      const int64_t c = f / (n * nc), rem = f % (n * nc);
      const int64_t row = rem / nc, part = rem % nc;
      V[f] = (row == c && part == 0) ? 1.0 : 0.0;
    }
  }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i <= MAX_SWEEPS; i += blockDim.x) counter[i] = 0;
}

template <int NC>
int run(int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k, double* W, int64_t ldw, double* sigma,
        cudaStream_t st) {
  Scratch ws;
  const size_t ubytes = sizeof(double) * s * n * NC, vbytes = sizeof(double) * n * n * NC;
  const size_t extra = sizeof(double) * n + sizeof(int) * (MAX_SWEEPS + 2) + 64;
  NSK_CUDA_OK(ws.alloc(ubytes + vbytes + extra, st));
  double* U = ws.as<double>();
  double* V = U + s * n * NC;
  double* norms = V + n * n * NC;
  int* counter = reinterpret_cast<int*>(norms + n);
  int* bad = counter + MAX_SWEEPS + 1;
  {
    int64_t tot = (s * n + n * n) * NC;
    int64_t blocks = (tot + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    init_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(SA, ldsa, s, n, NC, U, V, counter);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    NSK_CUDA_OK(cudaMemsetAsync(bad, 0, sizeof(int), st));
  }
  if (n >= 2) {
    JacobiParams P;
    P.U = U;
    P.V = V;
    P.s = s;
    P.n = n;
    P.N = n + (n & 1);
    // Stopping rule rows * eps: the computed |u_p^T u_q| of two converged
    // columns carries ~sqrt(rows) * eps relative rounding noise, so the
    // tighter sqrt(rows) * eps of dgesvj can stall on 1e-10-graded spectra.
    P.tol = static_cast<double>(s > n ? s : n) * 2.220446049250313e-16;
    P.counter = counter;
    size_t smem = sizeof(double) * 2 * s * NC;
    P.use_smem = smem <= 160 * 1024;
    if (!P.use_smem) smem = 0;
    auto kern = jacobi_kernel<NC>;
    NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    NSK_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, JT, smem));
    if (per_sm < 1) return fail(ECUDA, "jacobi: kernel does not fit on an SM");
    int64_t blocks = P.N / 2;
    const int64_t cap = static_cast<int64_t>(per_sm) * sm_count();
    if (blocks > cap) blocks = cap;
    void* args[] = {&P};
    NSK_CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(static_cast<unsigned>(blocks)),
                                            dim3(JT), args, smem, st));
    count_launch();
  }
  finish_kernel<NC><<<static_cast<unsigned>(n), JT, 0, st>>>(U, V, s, n, k, W, ldw, sigma, norms, nullptr);
  NSK_CUDA_OK(cudaGetLastError());
  order_kernel<NC><<<1, 256, sizeof(int) * n, st>>>(V, n, k, W, ldw, sigma, norms, bad);
  count_launch(2);
  NSK_CUDA_OK(cudaGetLastError());
  // Convergence and NaN checks need host visibility of two ints.
  int host[2] = {0, 0};
  NSK_CUDA_OK(cudaMemcpyAsync(&host[0], counter + MAX_SWEEPS, sizeof(int), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaMemcpyAsync(&host[1], bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  if (n >= 2 && host[0] >= MAX_SWEEPS) return fail(ENOCONV, "svd: one-sided Jacobi did not converge");
  if (host[1]) return fail(ENOCONV, "svd: non-finite singular values (input contains NaN/Inf)");
  return OK;
}

}  // namespace

int jacobi_trailing(int ncomp, int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k, double* W,
                    int64_t ldw, double* sigma, cudaStream_t st) {
  if (s < 1 || n < 1) return fail(EINVAL_, "svd: matrix is empty");
  return ncomp == 1 ? run<1>(s, n, SA, ldsa, k, W, ldw, sigma, st) : run<2>(s, n, SA, ldsa, k, W, ldw, sigma, st);
}

}  // namespace nsk
