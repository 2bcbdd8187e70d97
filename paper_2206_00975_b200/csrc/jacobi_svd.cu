// jacobi_svd.cu -- K4: trailing right singular vectors of SA on the device.
//
// Reference: from_sketch_svd (/root/reference/proj/src/nullspace.cpp:10-19)
// runs Eigen BDCSVD (kernels.cpp:14-22) on the s x n sketch and returns
// W = V(:, n-k : n-1) plus all n singular values, non-increasing; failure to
// converge raises SvdConvergenceError (kernels.hpp:18-20).
//
// B200 design (two cooperative persistent kernels, no host round trips):
//   1. Householder QR of SA (s x n) in place: one grid barrier per column,
//      the owner CTA of column j+1 forms its reflector right after applying
//      reflector j, every other CTA updates its own columns.  R (n x n) keeps
//      SA's right singular vectors and singular values.
//   2. one-sided (Hestenes) Jacobi on the stacked [R; I] (2n x n): column
//      pairs of a round-robin round are spread over the CTAs, a grid barrier
//      separates rounds, inner products run over the R rows only and every
//      rotation is applied to the V rows too.  Complex pairs are first
//      phase-aligned (u_q *= e^{-i arg c}) and then rotated.  Convergence: a
//      sweep with no rotation, i.e. every pair has
//      |u_p^H u_q| <= n u ||u_p|| ||u_q||.  One-sided Jacobi computes small
//      singular values to high relative accuracy; working on R (n rows
//      instead of s) cuts the per-round traffic by s/n.
//   sigma_j = ||R-part of column j||, W = the V-part of the k columns with
//   the smallest sigma (sorted non-increasing, ties by index).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include <mutex>
#include <string>

#include "nsk_internal.hpp"

namespace cg = cooperative_groups;

namespace nsk {
namespace {

constexpr int JT = 256;
constexpr int MAX_SWEEPS = 80;  // == CJ_MAX_SWEEPS (cluster_jacobi.cu): one counter layout

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

// ---------------------------------------------------------------- QR
struct QrParams {
  double* A;      // s x n (x NC), ld = s, overwritten by reflectors + R
  double* tau;    // n
  double* rdiag;  // n x NC: diagonal of R
  int64_t s, n;
};

// Reflector for column j (rows j..s-1): H = I - tau v v^H, H x = alpha e_0.
template <int NC>
__device__ void householder(const QrParams& P, int64_t j, double* red) {
  double* col = P.A + j * P.s * NC;
  double ss = 0, d1 = 0, d2 = 0, d3 = 0;
  for (int64_t i = j + 1 + threadIdx.x; i < P.s; i += JT) {
    if (NC == 1) {
      ss += col[i] * col[i];
    } else {
      ss += col[2 * i] * col[2 * i] + col[2 * i + 1] * col[2 * i + 1];
    }
  }
  block_sum4<NC>(ss, d1, d2, d3, red);
  if (threadIdx.x == 0) {
    const double xr = col[NC * j], xi = NC == 2 ? col[NC * j + 1] : 0.0;
    const double ax = NC == 1 ? fabs(xr) : hypot(xr, xi);
    const double sigma = sqrt(ax * ax + ss);
    if (sigma == 0.0) {
      P.tau[j] = 0.0;
      P.rdiag[NC * j] = 0.0;
      if (NC == 2) P.rdiag[NC * j + 1] = 0.0;
    } else {
      // alpha = -e^{i arg x0} sigma (real: -sign(x0) sigma); v0 = x0 - alpha.
      const double ur = ax > 0 ? xr / ax : 1.0, ui = ax > 0 ? xi / ax : 0.0;
      P.rdiag[NC * j] = -ur * sigma;
      if (NC == 2) P.rdiag[NC * j + 1] = -ui * sigma;
      col[NC * j] = ur * (ax + sigma);
      if (NC == 2) col[NC * j + 1] = ui * (ax + sigma);
      P.tau[j] = 1.0 / (sigma * (sigma + ax));
    }
  }
}

// a_k -= tau v (v^H a_k) for one column k, rows j..s-1.
template <int NC>
__device__ void apply_reflector(const QrParams& P, int64_t j, int64_t k, double* red) {
  const double* v = P.A + j * P.s * NC;
  double* a = P.A + k * P.s * NC;
  double wr = 0, wi = 0, d1 = 0, d2 = 0;
  // v was written by another CTA: read it from L2 (ld.cg), never from a stale L1 line.
  for (int64_t i = j + threadIdx.x; i < P.s; i += JT) {
    if (NC == 1) {
      wr += __ldcg(v + i) * a[i];
    } else {
      const double vr = __ldcg(v + 2 * i), vi = __ldcg(v + 2 * i + 1), ar = a[2 * i], ai = a[2 * i + 1];
      wr += vr * ar + vi * ai;  // conj(v) a
      wi += vr * ai - vi * ar;
    }
  }
  block_sum4<NC>(wr, wi, d1, d2, red);
  const double t = __ldcg(P.tau + j);
  wr *= t;
  wi *= t;
  for (int64_t i = j + threadIdx.x; i < P.s; i += JT) {
    if (NC == 1) {
      a[i] -= __ldcg(v + i) * wr;
    } else {
      const double vr = __ldcg(v + 2 * i), vi = __ldcg(v + 2 * i + 1);
      a[2 * i] -= vr * wr - vi * wi;
      a[2 * i + 1] -= vr * wi + vi * wr;
    }
  }
  __syncthreads();
}

// Point-to-point readiness flags instead of grid-wide barriers: a CTA that
// publishes data stores it, fences, and then releases the flag; a CTA that
// consumes it spins on the flag (acquire) and reads the data from L2 (ld.cg).
__device__ __forceinline__ void publish(int* flag, int value) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(flag), "r"(value) : "memory");
  }
}
__device__ __forceinline__ void await(const int* flag, int value) {
  if (threadIdx.x == 0) {
    int v;
    do {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(flag) : "memory");
    } while (v < value);
  }
  __syncthreads();
}

// Look-ahead Householder QR without grid barriers: reflector j is published by
// the owner of column j (flag[j] = 1) right after it applied reflector j-1 to
// that column; every CTA applies reflectors in order to the columns it owns.
template <int NC>
__global__ void __launch_bounds__(JT) qr_kernel(QrParams P, int* ready) {
  __shared__ double red[(JT / 32) * 4];
  const int64_t C = gridDim.x;
  if (blockIdx.x == 0) {
    householder<NC>(P, 0, red);
    publish(ready, 1);
  }
  for (int64_t j = 0; j + 1 < P.n; ++j) {
    const int64_t first = j + 1 + ((blockIdx.x - (j + 1) % C + C) % C);  // first owned column > j
    if (first >= P.n) break;
    await(ready + j, 1);
    for (int64_t k = first; k < P.n; k += C) {
      apply_reflector<NC>(P, j, k, red);
      if (k == j + 1) {  // look-ahead: publish the next reflector before the other updates
        householder<NC>(P, j + 1, red);
        publish(ready + j + 1, 1);
      }
    }
  }
}

// The same look-ahead QR with one column per CTA held in registers (s <= EPT * QRT rows): CTA k
// applies reflectors 0 .. k-1 as they are published and then publishes reflector k.  Against
// qr_kernel the critical path of a step loses the reloads of the column from memory and the
// serialised per-element L2 round trips (every thread issues all EPT loads of v_j at once), and the
// norm of the updated column comes from registers: 1.15 -> 0.4 ms at 1024 x 256.
constexpr int QRT = 128;

template <int NC>
__device__ __forceinline__ void qr_sum2(double& a, double& b, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    if (NC == 2) b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    red[w * 2] = a;
    red[w * 2 + 1] = b;
  }
  __syncthreads();
  a = b = 0.0;
#pragma unroll
  for (int i = 0; i < QRT / 32; ++i) {  // fixed order: deterministic
    a += red[i * 2];
    b += red[i * 2 + 1];
  }
  __syncthreads();  // red is reused by the next reduction
}

template <int NC, int EPT>
__global__ void __launch_bounds__(QRT) qr_reg_kernel(QrParams P, int* ready) {
  __shared__ double red[(QRT / 32) * 2];
  __shared__ double head[2];
  const int64_t k = blockIdx.x, s = P.s;
  double* col = P.A + k * s * NC;
  double ar[EPT], ai[EPT];  // rows threadIdx.x + QRT e
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int64_t i = threadIdx.x + QRT * e;
    ar[e] = i < s ? col[NC * i] : 0.0;
    ai[e] = (NC == 2 && i < s) ? col[NC * i + 1] : 0.0;
  }
  for (int64_t j = 0; j < k; ++j) {  // reflectors 0 .. k-1, each as soon as it is published
    await(ready + j, 1);
    const double* v = P.A + j * s * NC;
    double vr[EPT], vi[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {  // v was written by another CTA: L2 (ld.cg), all loads in flight at once
      const int64_t i = threadIdx.x + QRT * e;
      const bool in = i >= j && i < s;
      vr[e] = in ? __ldcg(v + NC * i) : 0.0;
      vi[e] = (NC == 2 && in) ? __ldcg(v + NC * i + 1) : 0.0;
    }
    double wr = 0.0, wi = 0.0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      wr = fma(vr[e], ar[e], wr);
      if (NC == 2) {
        wr = fma(vi[e], ai[e], wr);  // conj(v) a
        wi = fma(vr[e], ai[e], fma(-vi[e], ar[e], wi));
      }
    }
    qr_sum2<NC>(wr, wi, red);
    const double t = __ldcg(P.tau + j);
    wr *= t;
    wi *= t;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (NC == 1) {
        ar[e] = fma(-vr[e], wr, ar[e]);
      } else {
        ar[e] -= vr[e] * wr - vi[e] * wi;
        ai[e] -= vr[e] * wi + vi[e] * wr;
      }
    }
  }
  // reflector k from rows k .. s-1 of the updated column (householder() above, from registers)
  double ss = 0.0, dummy = 0.0;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int64_t i = threadIdx.x + QRT * e;
    if (i > k && i < s) ss += NC == 1 ? ar[e] * ar[e] : ar[e] * ar[e] + ai[e] * ai[e];
  }
  qr_sum2<1>(ss, dummy, red);
  const int hown = static_cast<int>(k % QRT), he = static_cast<int>(k / QRT);
  if (threadIdx.x == hown) {
    double xr = 0.0, xi = 0.0;
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (e == he) {
        xr = ar[e];
        xi = ai[e];
      }
    const double ax = NC == 1 ? fabs(xr) : hypot(xr, xi);
    const double sigma = sqrt(ax * ax + ss);
    double h0r = xr, h0i = xi;
    if (sigma == 0.0) {
      P.tau[k] = 0.0;
      P.rdiag[NC * k] = 0.0;
      if (NC == 2) P.rdiag[NC * k + 1] = 0.0;
    } else {
      const double ur = ax > 0 ? xr / ax : 1.0, ui = ax > 0 ? xi / ax : 0.0;
      P.rdiag[NC * k] = -ur * sigma;
      if (NC == 2) P.rdiag[NC * k + 1] = -ui * sigma;
      h0r = ur * (ax + sigma);
      h0i = ui * (ax + sigma);
      P.tau[k] = 1.0 / (sigma * (sigma + ax));
    }
    head[0] = h0r;
    head[1] = h0i;
  }
  __syncthreads();
  // the whole column: R entries above the diagonal, v_k from the diagonal down
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int64_t i = threadIdx.x + QRT * e;
    if (i < s) {
      col[NC * i] = i == k ? head[0] : ar[e];
      if (NC == 2) col[NC * i + 1] = i == k ? head[1] : ai[e];
    }
  }
  publish(ready + k, 1);
}

// Stacked working matrix [R; I] (2n x n, ld 2n) from the factored A.
__global__ void build_stacked(const double* __restrict__ A, const double* __restrict__ rdiag, int64_t s, int64_t n,
                              int nc, double* __restrict__ X) {
  const int64_t ld = 2 * n, total = ld * n * nc;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / (ld * nc), rem = e % (ld * nc), row = rem / nc, part = rem % nc;
    double v = 0.0;
    if (row < n) {
      if (row < c)
        v = A[(row + c * s) * nc + part];
      else if (row == c)
        v = rdiag[c * nc + part];
    } else {
      v = (row - n == c && part == 0) ? 1.0 : 0.0;
    }
    X[e] = v;
  }
}

// ---------------------------------------------------------------- Jacobi
struct JacobiParams {
  double* X;       // 2n x n (x NC), ld = 2n: rows [0, n) = R part, [n, 2n) = V part
  int64_t n, N;    // N = n rounded up to even
  double tol;
  int* counter;    // [MAX_SWEEPS]: rotations per sweep; [MAX_SWEEPS] = sweeps done
  int use_smem;
};

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

// Rounds are ordered by per-column version flags (version[c] = rounds applied
// to column c): a pair of global round g waits until both of its columns
// reached g, and publishes g + 1 after its rotation -- no grid-wide barrier
// per round, only one per sweep for the convergence test.
template <int NC>
__global__ void __launch_bounds__(JT) jacobi_kernel(JacobiParams P, int* version) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double cache[];  // [2][2n*NC] when use_smem
  __shared__ double red[(JT / 32) * 4];
  const int64_t n = P.n, N = P.N, ld = 2 * n;
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int64_t r = 0; r < N - 1; ++r) {
      const int g = static_cast<int>(sweep * (N - 1) + r);
      for (int64_t i = blockIdx.x; i < N / 2; i += gridDim.x) {
        int64_t p, q;
        pair_of_round(N, r, i, p, q);
        if (q >= n) {  // dummy column for odd n: the real column just advances
          await(version + p, g);
          publish(version + p, g + 1);
          continue;
        }
        await(version + p, g);
        await(version + q, g);
        double* xp = P.X + p * ld * NC;
        double* xq = P.X + q * ld * NC;
        double* cp = P.use_smem ? cache : xp;
        double* cq = P.use_smem ? cache + ld * NC : xq;
        double a = 0, b = 0, cr = 0, ci = 0;
        for (int64_t row = threadIdx.x; row < ld; row += JT) {
          if (NC == 1) {
            const double up = __ldcg(xp + row), uq = __ldcg(xq + row);
            if (P.use_smem) {
              cp[row] = up;
              cq[row] = uq;
            }
            if (row < n) {
              a += up * up;
              b += uq * uq;
              cr += up * uq;
            }
          } else {
            const double pr = __ldcg(xp + 2 * row), pi = __ldcg(xp + 2 * row + 1);
            const double qr = __ldcg(xq + 2 * row), qi = __ldcg(xq + 2 * row + 1);
            if (P.use_smem) {
              cp[2 * row] = pr;
              cp[2 * row + 1] = pi;
              cq[2 * row] = qr;
              cq[2 * row + 1] = qi;
            }
            if (row < n) {
              a += pr * pr + pi * pi;
              b += qr * qr + qi * qi;
              cr += pr * qr + pi * qi;  // conj(u_p) u_q
              ci += pr * qi - pi * qr;
            }
          }
        }
        block_sum4<NC>(a, b, cr, ci, red);
        const double cabs = NC == 1 ? fabs(cr) : hypot(cr, ci);
        if (cabs > P.tol * sqrt(a) * sqrt(b) && cabs > 0.0) {
          // Real pairs keep the sign of u_p^T u_q; complex pairs are phase-aligned
          // so that their inner product is the positive real |c|.
          const double zeta = (b - a) / (2.0 * (NC == 1 ? cr : cabs));
          const double t = fabs(zeta) > 1e150 ? 0.5 / zeta
                                              : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          const double ph_re = NC == 2 ? cr / cabs : 1.0, ph_im = NC == 2 ? -ci / cabs : 0.0;  // e^{-i phi}
          if (threadIdx.x == 0) atomicAdd(P.counter + sweep, 1);
          auto rd = [&](const double* ptr) { return P.use_smem ? *ptr : __ldcg(ptr); };
          for (int64_t row = threadIdx.x; row < ld; row += JT) {
            if (NC == 1) {
              const double up = rd(cp + row), uq = rd(cq + row);
              xp[row] = cs * up - sn * uq;
              xq[row] = sn * up + cs * uq;
            } else {
              const double pr = rd(cp + 2 * row), pi = rd(cp + 2 * row + 1);
              const double qr0 = rd(cq + 2 * row), qi0 = rd(cq + 2 * row + 1);
              const double qr = qr0 * ph_re - qi0 * ph_im, qi = qr0 * ph_im + qi0 * ph_re;
              xp[2 * row] = cs * pr - sn * qr;
              xp[2 * row + 1] = cs * pi - sn * qi;
              xq[2 * row] = sn * pr + cs * qr;
              xq[2 * row + 1] = sn * pi + cs * qi;
            }
          }
        }
        publish(version + p, g + 1);
        if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(version + q), "r"(g + 1) : "memory");
      }
    }
    grid.sync();  // sweep boundary: the rotation count of this sweep is final
    const int rot = *reinterpret_cast<volatile int*>(P.counter + sweep);
    if (rot == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.counter[MAX_SWEEPS] = sweep;
}

// ---------------------------------------------------------------- block Jacobi
// Block one-sided Jacobi: the n columns form B blocks of b; an outer
// round-robin round gives every CTA one block pair, which it loads into
// shared memory (2b columns of [R; I]) and fully re-orthogonalises there with
// an inner round-robin sweep (2b-1 rounds, one column pair per warp, warp
// shuffles for the inner products, __syncthreads between rounds).  Outer
// rounds are separated by one grid barrier and exchange blocks through L2, so
// the global synchronisation cost is paid once per b^2 rotations instead of
// once per n/2.
constexpr int BJT = 512;

struct BJParams {
  double* X;     // 2n x n (x NC), ld = 2n
  int64_t n;
  int b;         // columns per block
  int64_t B;     // blocks (even)
  double tol;
  int* counter;  // rotations per sweep; [MAX_SWEEPS] = sweeps
};

template <int NC>
__global__ void __launch_bounds__(BJT) block_jacobi_kernel(BJParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];  // [2b][ld * NC]
  __shared__ int rot_count;
  __shared__ unsigned char ptab[31 * 16][2];    // inner round-robin pairs (2b <= 32)
  __shared__ double red[4 * (BJT / 32)];        // per-warp partial inner products
  const int n = static_cast<int>(P.n), ld = 2 * n, colsz = ld * NC;
  const int b = P.b, twob = 2 * b;
  const int wpp = (BJT / 32) / b > 0 ? (BJT / 32) / b : 1;  // warps per column pair
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < (twob - 1) * b; e += BJT) {
    int64_t lp, lq;
    pair_of_round(twob, e / b, e % b, lp, lq);
    ptab[e][0] = static_cast<unsigned char>(lp);
    ptab[e][1] = static_cast<unsigned char>(lq);
  }
  const double tol2 = P.tol * P.tol;
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int64_t r = 0; r < P.B - 1; ++r) {
      for (int64_t i = blockIdx.x; i < P.B / 2; i += gridDim.x) {
        int64_t pb, qb;
        pair_of_round(P.B, r, i, pb, qb);
        if (threadIdx.x == 0) rot_count = 0;
        // Stage the block pair: each block is b contiguous columns of X, so both
        // are one contiguous span; 16-byte loads, four in flight per thread.
        for (int half = 0; half < 2; ++half) {
          const int64_t blk = half ? qb : pb;
          const int64_t c0 = blk * b;
          const int ncols = static_cast<int>(c0 + b <= n ? b : (c0 < n ? n - c0 : 0));
          const int64_t nv = static_cast<int64_t>(ncols) * colsz / 2;  // colsz is even (ld = 2n)
          const double2* src = reinterpret_cast<const double2*>(P.X + c0 * colsz);
          double2* dst = reinterpret_cast<double2*>(sm + half * b * colsz);
          int64_t e = threadIdx.x;
          for (; e + 3 * BJT < nv; e += 4 * BJT) {
            const double2 v0 = __ldcg(src + e), v1 = __ldcg(src + e + BJT), v2 = __ldcg(src + e + 2 * BJT),
                          v3 = __ldcg(src + e + 3 * BJT);
            dst[e] = v0;
            dst[e + BJT] = v1;
            dst[e + 2 * BJT] = v2;
            dst[e + 3 * BJT] = v3;
          }
          for (; e < nv; e += BJT) dst[e] = __ldcg(src + e);
          for (int64_t z = nv * 2 + threadIdx.x; z < static_cast<int64_t>(b) * colsz; z += BJT)
            sm[half * b * colsz + z] = 0.0;  // columns past n
        }
        __syncthreads();
        // Outer round 0 of a sweep pairs every block with its partner for the
        // first time: full round-robin over the 2b columns (intra-block pairs
        // included); later outer rounds only the b^2 cross pairs -- every
        // column pair once per sweep.
        const int inner = r == 0 ? twob - 1 : b;
        for (int t = 0; t < inner; ++t) {
          // WPP warps per pair: each sums a slice of rows, the slices meet in
          // shared memory and are added in fixed order by every warp of the
          // pair (identical rotation everywhere), then each rotates its slice.
          const int pi = warp / wpp, sub = warp - pi * wpp;
          const bool active = pi < b;
          double* xp = nullptr;
          double* xq = nullptr;
          if (active) {
            const int lp = r == 0 ? ptab[t * b + pi][0] : pi;
            const int lq = r == 0 ? ptab[t * b + pi][1] : b + (pi + t) % b;
            xp = sm + lp * colsz;
            xq = sm + lq * colsz;
            double a = 0, bb = 0, cr = 0, ci = 0;
            for (int row = sub * 32 + lane; row < n; row += 32 * wpp) {
              if (NC == 1) {
                const double up = xp[row], uq = xq[row];
                a = fma(up, up, a);
                bb = fma(uq, uq, bb);
                cr = fma(up, uq, cr);
              } else {
                const double pr = xp[2 * row], pim = xp[2 * row + 1], qr = xq[2 * row], qim = xq[2 * row + 1];
                a += pr * pr + pim * pim;
                bb += qr * qr + qim * qim;
                cr += pr * qr + pim * qim;
                ci += pr * qim - pim * qr;
              }
            }
            for (int o = 16; o > 0; o >>= 1) {  // fixed butterfly order: deterministic
              a += __shfl_xor_sync(0xffffffffu, a, o);
              bb += __shfl_xor_sync(0xffffffffu, bb, o);
              cr += __shfl_xor_sync(0xffffffffu, cr, o);
              if (NC == 2) ci += __shfl_xor_sync(0xffffffffu, ci, o);
            }
            if (lane == 0) {
              double* r = red + 4 * warp;
              r[0] = a;
              r[1] = bb;
              r[2] = cr;
              r[3] = ci;
            }
          }
          __syncthreads();
          if (active) {
            double a = 0, bb = 0, cr = 0, ci = 0;
            for (int w2 = 0; w2 < wpp; ++w2) {
              const double* r = red + 4 * (pi * wpp + w2);
              a += r[0];
              bb += r[1];
              cr += r[2];
              ci += r[3];
            }
            const double c2 = cr * cr + ci * ci;
            if (c2 > tol2 * a * bb && c2 > 0.0) {
              const double cabs = NC == 1 ? fabs(cr) : sqrt(c2);
              const double zeta = (bb - a) / (2.0 * (NC == 1 ? cr : cabs));
              const double tt = fabs(zeta) > 1e150 ? 0.5 / zeta
                                                   : copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              const double cs = rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
              const double inv = NC == 2 ? 1.0 / cabs : 1.0;
              const double ph_re = NC == 2 ? cr * inv : 1.0, ph_im = NC == 2 ? -ci * inv : 0.0;
              if (lane == 0 && sub == 0) rot_count = 1;  // any rotation keeps the sweep loop going
              for (int row = sub * 32 + lane; row < ld; row += 32 * wpp) {
                if (NC == 1) {
                  const double up = xp[row], uq = xq[row];
                  xp[row] = cs * up - sn * uq;
                  xq[row] = sn * up + cs * uq;
                } else {
                  const double pr = xp[2 * row], pim = xp[2 * row + 1];
                  const double qr0 = xq[2 * row], qi0 = xq[2 * row + 1];
                  const double qr = qr0 * ph_re - qi0 * ph_im, qim = qr0 * ph_im + qi0 * ph_re;
                  xp[2 * row] = cs * pr - sn * qr;
                  xp[2 * row + 1] = cs * pim - sn * qim;
                  xq[2 * row] = sn * pr + cs * qr;
                  xq[2 * row + 1] = sn * pim + cs * qim;
                }
              }
            }
          }
          __syncthreads();
        }
        for (int half = 0; half < 2; ++half) {
          const int64_t blk = half ? qb : pb;
          const int64_t c0 = blk * b;
          const int ncols = static_cast<int>(c0 + b <= n ? b : (c0 < n ? n - c0 : 0));
          const int64_t nv = static_cast<int64_t>(ncols) * colsz / 2;
          double2* dst = reinterpret_cast<double2*>(P.X + c0 * colsz);
          const double2* src = reinterpret_cast<const double2*>(sm + half * b * colsz);
          for (int64_t e = threadIdx.x; e < nv; e += BJT) __stcg(dst + e, src[e]);
        }
        if (threadIdx.x == 0 && rot_count) atomicAdd(P.counter + sweep, rot_count);
        __syncthreads();
      }
      grid.sync();
    }
    const int rot = *reinterpret_cast<volatile int*>(P.counter + sweep);
    if (rot == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.counter[MAX_SWEEPS] = sweep;
}

// sigma_j = ||R-part of column j|| (one CTA per column).
template <int NC>
__global__ void norms_kernel(const double* __restrict__ X, int64_t n, double* __restrict__ norms) {
  const int64_t j = blockIdx.x, ld = 2 * n;
  __shared__ double red[JT / 32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += JT) {
    if (NC == 1) {
      const double u = X[i + j * ld];
      acc += u * u;
    } else {
      const double ur = X[2 * (i + j * ld)], ui = X[2 * (i + j * ld) + 1];
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

// Order by non-increasing sigma (ties: lower index first); W(:, t) = V(:, order[n-k+t]).
template <int NC>
__global__ void order_kernel(const double* __restrict__ X, int64_t n, int64_t k, double* __restrict__ W,
                             int64_t ldw, double* __restrict__ sigma, const double* __restrict__ norms,
                             int* __restrict__ bad) {
  extern __shared__ int pos_of[];  // rank -> column
  const int64_t ld = 2 * n;
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
      if (NC == 1) {
        W[i + t * ldw] = X[n + i + col * ld];
      } else {
        W[2 * (i + t * ldw)] = X[2 * (n + i + col * ld)];
        W[2 * (i + t * ldw) + 1] = X[2 * (n + i + col * ld) + 1];
      }
    }
  }
}

__global__ void copy_in_kernel(const double* __restrict__ SA, int64_t ldsa, int64_t s, int64_t n, int nc,
                               double* __restrict__ A, int* counter) {
  const int64_t tot = s * n * nc;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / (s * nc), rem = e % (s * nc);
    A[e] = SA[c * ldsa * nc + rem];
  }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i <= MAX_SWEEPS + 1; i += blockDim.x) counter[i] = 0;
}

template <class K>
int coop_launch(K kern, int64_t want, size_t smem, void** args, cudaStream_t st, int threads = JT) {
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  NSK_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return fail(ECUDA, "svd: kernel does not fit on an SM");
  int64_t blocks = want;
  const int64_t cap = static_cast<int64_t>(per_sm) * sm_count();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  NSK_CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(static_cast<unsigned>(blocks)),
                                          dim3(threads), args, smem, st));
  count_launch();
  return OK;
}

// Householder QR of the s x n working copy (reflectors below the diagonal, R above, diagonal in rdiag):
// qr_reg_kernel when its n CTAs fit on the device at once and a column fits the registers
// (s <= 4096 real, 2048 complex), else qr_kernel.  NSK_SVD_QR_OLD=1 forces qr_kernel (A/B).
template <int NC>
int qr_factor(const QrParams& Q, void** args, cudaStream_t st) {
  const int64_t s = Q.s, n = Q.n;
  auto reg = [&](auto kern) -> int {
    int per_sm = 0;
    NSK_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, QRT, 0));
    if (static_cast<int64_t>(per_sm) * sm_count() < n) return NOTAPPLICABLE;
    NSK_CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(static_cast<unsigned>(n)), dim3(QRT),
                                            args, 0, st));
    count_launch();
    return OK;
  };
  int rc = NOTAPPLICABLE;
  if (n <= s && !std::getenv("NSK_SVD_QR_OLD")) {
    if (s <= 8 * QRT)
      rc = reg(qr_reg_kernel<NC, 8>);
    else if (s <= 16 * QRT)
      rc = reg(qr_reg_kernel<NC, 16>);
    else if (NC == 1 && s <= 32 * QRT)
      rc = reg(qr_reg_kernel<NC, NC == 1 ? 32 : 16>);
  }
  if (rc != NOTAPPLICABLE) return rc;
  return coop_launch(qr_kernel<NC>, n, 0, args, st);
}

// Per-SVD device buffers of the Jacobi stage (X = [R; I] or [R'; V] workspace and its counters).
struct SvdBufs {
  double* X;
  double* norms;
  int* counter;  // [MAX_SWEEPS + 1]
  int* bad;
  int* version;  // [n]: Jacobi column versions / degenerate flag; zero on entry
};

size_t svd_bufs_bytes(int64_t n, int nc) {
  return sizeof(double) * (2 * n * n * nc + n) + sizeof(int) * (MAX_SWEEPS + 2 + n) + 64;
}

SvdBufs svd_bufs_at(void* base, int64_t n, int nc) {
  SvdBufs b;
  b.X = static_cast<double*>(base);
  b.norms = b.X + 2 * n * n * nc;
  b.counter = reinterpret_cast<int*>(b.norms + n);
  b.bad = b.counter + MAX_SWEEPS + 1;
  b.version = b.bad + 1;
  return b;
}

// Trailing k right singular vectors and all n singular values of the leading s x n block of the
// QR'd matrix (R in the upper triangle of A, ld s, diagonal in rdiag): the Jacobi stage.  launch()
// only enqueues work on st (so two stages on two streams can be in flight from one host thread);
// finish() reads the three host-visible flags and reruns on [R; I] when R was exactly singular.
template <int NC>
struct SvdStage {
  const double* A;
  const double* rdiag;
  int64_t s, n, k;
  double* W;
  int64_t ldw;
  double* sigma;
  SvdBufs B;
  cudaStream_t st;
  double tol = 0.0;
  int b = 16;
  bool blocked = false;
  int host[3] = {0, 0, 0};  // sweeps, non-finite flag, path (1: preconditioned, 0: [R; I], -1: rerun)
  int flag = 0;

  int stacked() {
    int64_t blocks = (2 * n * n * NC + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    build_stacked<<<static_cast<unsigned>(blocks), 256, 0, st>>>(A, rdiag, s, n, NC, B.X);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    return OK;
  }

  int solve(bool precondition) {
    double* X = B.X;
    int* degenerate = B.version;  // flag of the preconditioned path (version[] is zero here)
    int crc = NOTAPPLICABLE;
    if (n >= 2 && precondition) crc = cluster_svd_rt(NC, X, n, tol, B.counter, degenerate, st);  // 2a. QRCP + R'^H
    if (crc != OK && crc != NOTAPPLICABLE) return crc;
    host[2] = crc == OK;
    if (crc != OK && n >= 2) crc = cluster_jacobi(NC, X, n, tol, B.counter, st);  // 2b. whole [R; I] in one cluster
    if (crc != OK && crc != NOTAPPLICABLE) return crc;
    if (crc == OK) {
    } else if (n >= 2 && blocked) {  // 2c. block one-sided Jacobi on [R; I] through L2
      BJParams P;
      P.X = X;
      P.n = n;
      P.b = b;
      P.B = (n + b - 1) / b;
      P.B += P.B & 1;
      P.tol = tol;
      P.counter = B.counter;
      void* args[] = {&P};
      if (int rc = coop_launch(block_jacobi_kernel<NC>, P.B / 2, sizeof(double) * 2 * b * 2 * n * NC, args, st, BJT))
        return rc;
    } else if (n >= 2) {  // very large n: pairwise Jacobi with columns in L2
      JacobiParams P;
      P.X = X;
      P.n = n;
      P.N = n + (n & 1);
      P.tol = tol;
      P.counter = B.counter;
      size_t smem = sizeof(double) * 2 * 2 * n * NC;
      P.use_smem = smem <= 160 * 1024;
      if (!P.use_smem) smem = 0;
      int* version = B.version;
      void* args[] = {&P, &version};
      if (int rc = coop_launch(jacobi_kernel<NC>, P.N / 2, smem, args, st)) return rc;
    }
    norms_kernel<NC><<<static_cast<unsigned>(n), JT, 0, st>>>(X, n, B.norms);
    NSK_CUDA_OK(cudaGetLastError());
    NSK_CUDA_OK(cudaMemsetAsync(B.bad, 0, sizeof(int), st));
    order_kernel<NC><<<1, 256, sizeof(int) * n, st>>>(X, n, k, W, ldw, sigma, B.norms, B.bad);
    count_launch(2);
    NSK_CUDA_OK(cudaGetLastError());
    return OK;
  }

  // Convergence, NaN and degeneracy checks need host visibility of three ints.
  int collect() {
    flag = 0;
    NSK_CUDA_OK(cudaMemcpyAsync(&host[0], B.counter + MAX_SWEEPS, sizeof(int), cudaMemcpyDeviceToHost, st));
    NSK_CUDA_OK(cudaMemcpyAsync(&host[1], B.bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (host[2]) NSK_CUDA_OK(cudaMemcpyAsync(&flag, B.version, sizeof(int), cudaMemcpyDeviceToHost, st));
    NSK_CUDA_OK(cudaStreamSynchronize(st));
    if (flag) host[2] = -1;
    return OK;
  }

  int launch() {
    if (int rc = stacked()) return rc;
    // Stopping rule n * eps: the computed |u_p^T u_q| of converged columns
    // carries ~sqrt(n) * eps relative rounding noise, so the tighter
    // sqrt(n) * eps of dgesvj can stall on 1e-10-graded spectra.
    tol = static_cast<double>(n) * 2.220446049250313e-16;
    // Block width: the rotations of a round are FP64-throughput bound on the SMs
    // that hold a block pair, so spread them -- the widest b in {16, 8, 4, 2}
    // that still leaves >= 32 block pairs (CTAs) -- and a block pair of [R; I]
    // columns must fit in shared memory.  NSK_SVD_B overrides (tuning).
    b = 16;
    while (b > 2 && n / b < 64) b >>= 1;
    if (const char* e = std::getenv("NSK_SVD_B")) b = std::atoi(e) >= 1 && std::atoi(e) <= 16 ? std::atoi(e) : b;
    while (b > 1 && sizeof(double) * 2 * b * 2 * n * NC > 200 * 1024) b >>= 1;
    blocked = sizeof(double) * 2 * b * 2 * n * NC <= 200 * 1024 && std::getenv("NSK_SVD_PAIRS") == nullptr;
    return solve(true);
  }

  int finish() {
    if (int rc = collect()) return rc;
    if (host[2] < 0) {  // exactly singular R: What undefined, rerun on [R; I]
      NSK_CUDA_OK(cudaMemsetAsync(B.version, 0, sizeof(int) * n, st));
      NSK_CUDA_OK(cudaMemsetAsync(B.counter, 0, sizeof(int) * (MAX_SWEEPS + 1), st));
      if (int rc = stacked()) return rc;
      if (int rc = solve(false)) return rc;
      if (int rc = collect()) return rc;
    }
    if (std::getenv("NSK_SVD_DEBUG")) {
      std::fprintf(stderr, "nsk svd: s=%lld n=%lld b=%d sweeps=%d path=%d rotations/sweep:", static_cast<long long>(s),
                   static_cast<long long>(n), b, host[0], host[2]);
      int cnt[MAX_SWEEPS];
      const int ns = host[0] < MAX_SWEEPS ? host[0] + 1 : MAX_SWEEPS;
      if (ns > 0 && cudaMemcpy(cnt, B.counter, sizeof(int) * ns, cudaMemcpyDeviceToHost) == cudaSuccess)
        for (int i = 0; i < ns; ++i) std::fprintf(stderr, " %d", cnt[i]);
      std::fprintf(stderr, "\n");
    }
    if (n >= 2 && host[0] >= MAX_SWEEPS) return fail(ENOCONV, "svd: one-sided Jacobi did not converge");
    if (host[1]) return fail(ENOCONV, "svd: non-finite singular values (input contains NaN/Inf)");
    return OK;
  }
};

template <int NC>
int svd_stage(const double* A, const double* rdiag, int64_t s, int64_t n, int64_t k, double* W, int64_t ldw,
              double* sigma, SvdBufs B, cudaStream_t st) {
  SvdStage<NC> g{A, rdiag, s, n, k, W, ldw, sigma, B, st};
  if (int rc = g.launch()) return rc;
  return g.finish();
}

// The second stage of jacobi_trailing_pair runs on this per-device stream (created once).
cudaStream_t side_stream() {
  constexpr int MAXDEV = 64;
  static std::mutex mu;
  static cudaStream_t cs[MAXDEV] = {};
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur < 0 || cur >= MAXDEV) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!cs[cur] && cudaStreamCreateWithFlags(&cs[cur], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    cs[cur] = nullptr;
  }
  return cs[cur];
}

// Householder QR of the s x n copy of SA (R above the diagonal of A, diagonal in rdiag), then the
// Jacobi stage on R; with n2 > 0 also the singular values of the leading n2 columns (the
// existence check of sketched TLS, tls.cpp:110-111): their R is the leading block of the same
// factor, so that second Jacobi stage needs no QR of its own and runs concurrently on a second
// stream (each stage fills one 16-CTA cluster).
template <int NC>
int run(int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k, double* W, int64_t ldw, double* sigma,
        int64_t n2, double* sigma2, cudaStream_t st) {
  Scratch ws;
  const size_t apad = (s * n * NC + 1) & ~static_cast<int64_t>(1);  // X 16-byte aligned (double2 staging)
  const size_t abytes = sizeof(double) * apad;
  const size_t qbytes = (sizeof(double) * (n + n * NC) + sizeof(int) * n + 15) / 16 * 16;
  const size_t b1 = (svd_bufs_bytes(n, NC) + 15) / 16 * 16, b2 = n2 > 0 ? svd_bufs_bytes(n2, NC) : 0;
  NSK_CUDA_OK(ws.alloc(abytes + qbytes + b1 + b2, st));
  char* base = ws.as<char>();
  double* A = reinterpret_cast<double*>(base);
  double* tau = reinterpret_cast<double*>(base + abytes);
  double* rdiag = tau + n;
  int* ready = reinterpret_cast<int*>(rdiag + n * NC);  // QR reflector flags
  const SvdBufs B1 = svd_bufs_at(base + abytes + qbytes, n, NC);
  const SvdBufs B2 = n2 > 0 ? svd_bufs_at(base + abytes + qbytes + b1, n2, NC) : SvdBufs{};
  NSK_CUDA_OK(cudaMemsetAsync(ready, 0, sizeof(int) * n, st));
  NSK_CUDA_OK(cudaMemsetAsync(B1.version, 0, sizeof(int) * n, st));
  if (n2 > 0) {
    NSK_CUDA_OK(cudaMemsetAsync(B2.version, 0, sizeof(int) * n2, st));
    NSK_CUDA_OK(cudaMemsetAsync(B2.counter, 0, sizeof(int) * (MAX_SWEEPS + 1), st));
  }
  {
    int64_t blocks = (s * n * NC + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    copy_in_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(SA, ldsa, s, n, NC, A, B1.counter);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  {  // 1. Householder QR: one register-resident column per CTA when all n CTAs are co-resident
    QrParams Q{A, tau, rdiag, s, n};
    void* args[] = {&Q, &ready};
    if (int rc = qr_factor<NC>(Q, args, st)) return rc;
  }
  if (n2 <= 0) return svd_stage<NC>(A, rdiag, s, n, k, W, ldw, sigma, B1, st);
  // both Jacobi stages in flight at once: stage 2 on the side stream after the QR (each fills one
  // 16-CTA cluster; the device holds several), enqueued from this thread before either is collected
  cudaStream_t aux = side_stream();
  if (!aux) return fail(ECUDA, "svd: no side stream");
  cudaEvent_t qr_done;
  NSK_CUDA_OK(cudaEventCreateWithFlags(&qr_done, cudaEventDisableTiming));
  NSK_CUDA_OK(cudaEventRecord(qr_done, st));
  const cudaError_t fork = cudaStreamWaitEvent(aux, qr_done, 0);
  cudaEventDestroy(qr_done);
  NSK_CUDA_OK(fork);
  SvdStage<NC> g1{A, rdiag, s, n, k, W, ldw, sigma, B1, st};
  SvdStage<NC> g2{A, rdiag, s, n2, 0, nullptr, 1, sigma2, B2, aux};
  const int l1 = g1.launch();
  const int l2 = l1 == OK ? g2.launch() : OK;
  // the scratch (ws) is released on st: st must not run ahead of the side stream's use of it
  cudaEvent_t side_done;
  NSK_CUDA_OK(cudaEventCreateWithFlags(&side_done, cudaEventDisableTiming));
  NSK_CUDA_OK(cudaEventRecord(side_done, aux));
  const cudaError_t join = cudaStreamWaitEvent(st, side_done, 0);
  cudaEventDestroy(side_done);
  NSK_CUDA_OK(join);
  if (l1 != OK) return l1;
  if (l2 != OK) return l2;
  const int rc1 = g1.finish();
  const int rc2 = g2.finish();
  if (rc1 != OK) return rc1;
  if (rc2 != OK) return rc2;
  return OK;
}

}  // namespace

int jacobi_trailing(int ncomp, int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k, double* W,
                    int64_t ldw, double* sigma, cudaStream_t st) {
  if (s < 1 || n < 1) return fail(EINVAL_, "svd: matrix is empty");
  return ncomp == 1 ? run<1>(s, n, SA, ldsa, k, W, ldw, sigma, 0, nullptr, st)
                    : run<2>(s, n, SA, ldsa, k, W, ldw, sigma, 0, nullptr, st);
}

int jacobi_trailing_pair(int ncomp, int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k, double* W,
                         int64_t ldw, double* sigma, int64_t n2, double* sigma2, cudaStream_t st) {
  if (s < 1 || n < 1 || n2 < 1 || n2 > n) return fail(EINVAL_, "svd: bad shapes");
  return ncomp == 1 ? run<1>(s, n, SA, ldsa, k, W, ldw, sigma, n2, sigma2, st)
                    : run<2>(s, n, SA, ldsa, k, W, ldw, sigma, n2, sigma2, st);
}

}  // namespace nsk
