// jacobi_pair.cuh -- one warp orthogonalises one column pair of [R; I]
// (one-sided Jacobi step, shared by the cluster and global-memory kernels).
//
// Columns hold the R part in rows [0, n) and the V part in rows [n, ld); the
// inner products run over the R part only, the rotation over all ld rows.
// Real: the classical Rutishauser angle; complex: q is first phase-aligned
// (u_q *= e^{-i arg c}) and then rotated.  Rows are processed in batches of
// four per lane with all loads issued before any store, so shared-memory
// latency overlaps instead of serialising the chain (the two columns never
// alias).  Accumulation order is the row order: results do not depend on the
// batching.  Returns 0 when the pair was not rotated, 1 for a rotation with
// |cos(p, q)| <= sqrt(eps) / 2 ("small"), 2 for a larger one (JACOBI_BIG2).

#pragma once

#include <cuda_runtime.h>

namespace nsk {

// Rotate rows [0, ld) of the column pair (xp, xq): p' = c p - s q', q' = s p + c q'
// with q' = e^{-i phi} q (phi = 0 for real data).
template <int NC>
__device__ __forceinline__ void rotate_cols(double* __restrict__ xp, double* __restrict__ xq, int ld, int lane,
                                            double cs, double sn, double ph_re, double ph_im) {
  int row = lane;
  if (NC == 1) {
    for (; row + 96 < ld; row += 128) {
      double up[4], uq[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        up[k] = xp[row + 32 * k];
        uq[k] = xq[row + 32 * k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        xp[row + 32 * k] = cs * up[k] - sn * uq[k];
        xq[row + 32 * k] = sn * up[k] + cs * uq[k];
      }
    }
    for (; row < ld; row += 32) {
      const double up = xp[row], uq = xq[row];
      xp[row] = cs * up - sn * uq;
      xq[row] = sn * up + cs * uq;
    }
  } else {
    double2* p2 = reinterpret_cast<double2*>(xp);
    double2* q2 = reinterpret_cast<double2*>(xq);
    for (; row + 32 < ld; row += 64) {
      double2 pp[2], qq[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        pp[k] = p2[row + 32 * k];
        qq[k] = q2[row + 32 * k];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double qr = qq[k].x * ph_re - qq[k].y * ph_im, qim = qq[k].x * ph_im + qq[k].y * ph_re;
        p2[row + 32 * k] = make_double2(cs * pp[k].x - sn * qr, cs * pp[k].y - sn * qim);
        q2[row + 32 * k] = make_double2(sn * pp[k].x + cs * qr, sn * pp[k].y + cs * qim);
      }
    }
    for (; row < ld; row += 32) {
      const double2 pp = p2[row], qq = q2[row];
      const double qr = qq.x * ph_re - qq.y * ph_im, qim = qq.x * ph_im + qq.y * ph_re;
      p2[row] = make_double2(cs * pp.x - sn * qr, cs * pp.y - sn * qim);
      q2[row] = make_double2(sn * pp.x + cs * qr, sn * pp.y + cs * qim);
    }
  }
}

// cos^2 above which a rotation is "big": eps / 4, i.e. |cos| > 7.45e-9.  A sweep whose rotations
// are all small leaves every pair at |cos| <~ tol (quadratic convergence: each small rotation moves
// the other pairs' cosines by O(cos^2) = O(eps)), so the sweep after it would rotate nothing.
constexpr double JACOBI_BIG2 = 0.25 * 2.220446049250313e-16;

template <int NC>
__device__ __forceinline__ int jacobi_pair(double* __restrict__ xp, double* __restrict__ xq, int n, int ld,
                                            int lane, double tol2) {
  double a = 0, bb = 0, cr = 0, ci = 0;
  int row = lane;
  if (NC == 1) {
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
  } else {
    for (; row + 32 < n; row += 64) {
      double v[2][4];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double2 pp = reinterpret_cast<const double2*>(xp)[row + 32 * k];
        const double2 qq = reinterpret_cast<const double2*>(xq)[row + 32 * k];
        v[k][0] = pp.x;
        v[k][1] = pp.y;
        v[k][2] = qq.x;
        v[k][3] = qq.y;
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double pr = v[k][0], pim = v[k][1], qr = v[k][2], qim = v[k][3];
        a += pr * pr + pim * pim;
        bb += qr * qr + qim * qim;
        cr += pr * qr + pim * qim;
        ci += pr * qim - pim * qr;
      }
    }
    for (; row < n; row += 32) {
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
  const double c2 = cr * cr + ci * ci;
  if (!(c2 > tol2 * a * bb && c2 > 0.0)) return 0;
  const int kind = c2 > JACOBI_BIG2 * a * bb ? 2 : 1;
  const double cabs = NC == 1 ? fabs(cr) : sqrt(c2);
  const double zeta = (bb - a) / (2.0 * (NC == 1 ? cr : cabs));
  const double tt =
      fabs(zeta) > 1e150 ? 0.5 / zeta : copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
  const double cs = rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
  double ph_re = 1.0, ph_im = 0.0;
  if (NC == 2) {
    const double inv = 1.0 / cabs;
    ph_re = cr * inv;
    ph_im = -ci * inv;
  }
  rotate_cols<NC>(xp, xq, ld, lane, cs, sn, ph_re, ph_im);
  return kind;
}

}  // namespace nsk

namespace nsk {

// ---- register-resident pair step (cluster kernels) ---------------------------
// Fast double-precision reciprocal / reciprocal square root: the hardware
// approximation (~2^-22) refined by two Newton steps (quadratic convergence,
// ~1 ulp).  Used only for the rotation angle, whose rounding does not affect
// orthogonality: cs = rsqrt(1 + t^2), sn = cs t is a rotation for any t.
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double h = 0.5 * x * y;
    y = fma(y, fma(-h, y, 0.5), y);
  }
  return y;
}

// One-sided Jacobi step on the pair (xp, xq) with the leading n rows held in
// registers between the inner products and the rotation (shared memory is
// read once and written once; rows [n, ld) -- the V part of [R; I] -- are
// rotated in place).  RPL >= ceil(n / 32).  Same rotation as jacobi_pair
// (t = tan of the Rutishauser angle), written as
//   t = sign(d) 2c / (|d| + sqrt(d^2 + 4 c^2)),  d = ||q||^2 - ||p||^2,
// on power-of-two-scaled d, 2c (no overflow), with fast rcp / rsqrt.
// Rows r = lane + 32 k < n of a column into / out of registers.
template <int NC, int RPL>
__device__ __forceinline__ void load_col(const double* __restrict__ x, int n, int lane, double (&re)[RPL],
                                         double (&im)[RPL]) {
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int r = lane + 32 * k;
    re[k] = im[k] = 0.0;
    if (r < n) {
      if (NC == 1) {
        re[k] = x[r];
      } else {
        const double2 u = reinterpret_cast<const double2*>(x)[r];
        re[k] = u.x;
        im[k] = u.y;
      }
    }
  }
}
template <int NC, int RPL>
__device__ __forceinline__ void store_col(double* __restrict__ x, int n, int lane, const double (&re)[RPL],
                                          const double (&im)[RPL]) {
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int r = lane + 32 * k;
    if (r < n) {
      if (NC == 1)
        x[r] = re[k];
      else
        reinterpret_cast<double2*>(x)[r] = make_double2(re[k], im[k]);
    }
  }
}

// Core of the register step: p held in registers (pr, pim; updated in place),
// q read from and written back to shared memory; rows [n, ld) of both (the V
// part of [R; I]) rotated in place.
template <int NC, int RPL>
__device__ __forceinline__ int jacobi_step_preg(double (&pr)[RPL], double (&pim)[RPL], double* __restrict__ xp,
                                                 double* __restrict__ xq, int n, int ld, int lane, double tol2) {
  double qr[RPL], qim[RPL];
  load_col<NC, RPL>(xq, n, lane, qr, qim);
  double a = 0, bb = 0, cr = 0, ci = 0;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    a = fma(pr[k], pr[k], a);
    bb = fma(qr[k], qr[k], bb);
    cr = fma(pr[k], qr[k], cr);
    if (NC == 2) {
      a = fma(pim[k], pim[k], a);
      bb = fma(qim[k], qim[k], bb);
      cr = fma(pim[k], qim[k], cr);
      ci = fma(pr[k], qim[k], ci);
      ci = fma(-pim[k], qr[k], ci);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {  // fixed butterfly order: deterministic
    a += __shfl_xor_sync(0xffffffffu, a, o);
    bb += __shfl_xor_sync(0xffffffffu, bb, o);
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
    if (NC == 2) ci += __shfl_xor_sync(0xffffffffu, ci, o);
  }
  const double c2 = cr * cr + ci * ci;
  if (!(c2 > tol2 * a * bb && c2 > 0.0)) return 0;
  const int kind = c2 > JACOBI_BIG2 * a * bb ? 2 : 1;
  double ph_re = 1.0, ph_im = 0.0, c = cr;
  if (NC == 2) {
    const double inv = rsqrt_fast(c2);
    c = c2 * inv;  // |c|
    ph_re = cr * inv;
    ph_im = -ci * inv;
  }
  const double d = bb - a, e = 2.0 * c;
  const double mx = fmax(fabs(d), fabs(e));
  // 2^(1023 - exponent(mx)): exact scaling of d, e into [1, 4)
  int ex = (__double2hiint(mx) >> 20) & 0x7ff;
  ex = ex < 1 ? 1 : (ex > 2045 ? 2045 : ex);
  const double sc = __hiloint2double((2046 - ex) << 20, 0);
  const double ds = d * sc, es = e * sc;
  const double h2 = fma(ds, ds, es * es);
  const double hs = h2 * rsqrt_fast(h2);
  const double tt = copysign(1.0, d) * es * rcp_fast(fabs(ds) + hs);
  const double cs = rsqrt_fast(fma(tt, tt, 1.0)), sn = cs * tt;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    if (NC == 1) {
      const double up = pr[k], uq = qr[k];
      pr[k] = cs * up - sn * uq;
      qr[k] = sn * up + cs * uq;
    } else {
      const double q1 = qr[k] * ph_re - qim[k] * ph_im, q2 = qr[k] * ph_im + qim[k] * ph_re;
      const double p1 = pr[k], p2 = pim[k];
      pr[k] = cs * p1 - sn * q1;
      pim[k] = cs * p2 - sn * q2;
      qr[k] = sn * p1 + cs * q1;
      qim[k] = sn * p2 + cs * q2;
    }
  }
  store_col<NC, RPL>(xq, n, lane, qr, qim);
  if (ld > n) rotate_cols<NC>(xp + n * NC, xq + n * NC, ld - n, lane, cs, sn, ph_re, ph_im);
  return kind;
}

// One-sided Jacobi step on the pair (xp, xq) with the leading n rows held in
// registers between the inner products and the rotation (shared memory is
// read once and written once; rows [n, ld) -- the V part of [R; I] -- are
// rotated in place).  RPL >= ceil(n / 32).  Same rotation as jacobi_pair
// (t = tan of the Rutishauser angle), written as
//   t = sign(d) 2c / (|d| + sqrt(d^2 + 4 c^2)),  d = ||q||^2 - ||p||^2,
// on power-of-two-scaled d, 2c (no overflow), with fast rcp / rsqrt.
template <int NC, int RPL>
__device__ __forceinline__ int jacobi_pair_reg(double* __restrict__ xp, double* __restrict__ xq, int n, int ld,
                                               int lane, double tol2) {
  double pr[RPL], pim[RPL];
  load_col<NC, RPL>(xp, n, lane, pr, pim);
  const int rot = jacobi_step_preg<NC, RPL>(pr, pim, xp, xq, n, ld, lane, tol2);
  if (rot) store_col<NC, RPL>(xp, n, lane, pr, pim);
  return rot;
}

}  // namespace nsk
