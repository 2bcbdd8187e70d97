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
// batching.  Returns whether the pair was rotated.
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

template <int NC>
__device__ __forceinline__ bool jacobi_pair(double* __restrict__ xp, double* __restrict__ xq, int n, int ld,
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
  if (!(c2 > tol2 * a * bb && c2 > 0.0)) return false;
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
  return true;
}

}  // namespace nsk
