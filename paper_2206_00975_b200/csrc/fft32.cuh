// fft32.cuh -- register-resident 32-point DFT building blocks (kernel
// e^{+2 pi i nk/N}, the unitary inverse DFT's sign, transforms.cpp:17-36),
// shared by the SRFT/SRDCT kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace nsk {
namespace fft {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// v * e^{+2 pi i k/32}, k < 16 (compile-time k after unrolling).
__device__ __forceinline__ double2 twmul32(double2 v, int k) {
  // cos(pi k / 16), k = 0..8; sin(pi k/16) = cos(pi (8 - k)/16)
  constexpr double C[9] = {1.0,
                           0.98078528040323044912618223613,
                           0.92387953251128675612818318939,
                           0.83146961230254523707878837761,
                           0.70710678118654752440084436210,
                           0.55557023301960222474283081394,
                           0.38268343236508977172845998403,
                           0.19509032201612826784828486847,
                           0.0};
  if (k == 0) return v;
  if (k == 8) return make_double2(-v.y, v.x);  // * i
  const double c = k < 8 ? C[k] : -C[16 - k];
  const double s = k < 8 ? C[8 - k] : C[k - 8];
  return make_double2(fma(v.x, c, -v.y * s), fma(v.x, s, v.y * c));
}

// a * b mod N for a, b < N <= 2^44 without 128-bit division: the quotient
// from FP64 (error below 1 for these sizes), the remainder exact in wrapping
// 64-bit arithmetic, then at most two corrections.
__device__ __forceinline__ uint64_t mulmod_fast(uint64_t a, uint64_t b, uint64_t N, double invN) {
  const double q = floor(static_cast<double>(a) * static_cast<double>(b) * invN);
  int64_t r = static_cast<int64_t>(a * b - static_cast<uint64_t>(q) * N);
  const int64_t n = static_cast<int64_t>(N);
  if (r < 0) r += n;
  if (r < 0) r += n;
  if (r >= n) r -= n;
  if (r >= n) r -= n;
  return static_cast<uint64_t>(r);
}

// e^{2 pi i r / N} for an exact integer r in [0, N); two_over_N = 2.0 / N.
__device__ __forceinline__ double2 unit_phase(uint64_t r, double two_over_N) {
  double sn, cs;
  sincospi(static_cast<double>(r) * two_over_N, &sn, &cs);
  return make_double2(cs, sn);
}

__device__ __forceinline__ constexpr int brev5(int i) {
  return ((i & 1) << 4) | ((i & 2) << 2) | (i & 4) | ((i & 8) >> 2) | ((i & 16) >> 4);
}

// In-register 32-point DFT, kernel e^{+2 pi i nk/32}, natural order in and out.
__device__ __forceinline__ void dft32(double2 (&x)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = brev5(i);
    if (r > i) {
      const double2 t = x[i];
      x[i] = x[r];
      x[r] = t;
    }
  }
#pragma unroll
  for (int stage = 1; stage <= 5; ++stage) {
    const int half = 1 << (stage - 1);
#pragma unroll
    for (int e = 0; e < 16; ++e) {  // 16 butterflies per stage
      const int j = e & (half - 1), i = (e >> (stage - 1)) << stage;
      const double2 u = x[i + j];
      const double2 t = twmul32(x[i + j + half], j << (5 - stage));
      x[i + j] = cadd(u, t);
      x[i + j + half] = csub(u, t);
    }
  }
}

// Butterfly (u, v) -> (u + W v, u - W v), W = e^{2 pi i k/32} for a compile-time
// k < 16, in 6 FP64 instructions for a non-trivial W: W = f (1 + i t) or
// W = f (t + i) with |t| <= 1 (f = cos and t = tan where |cos| >= |sin|, else
// f = sin and t = cot), so W v / f costs two FMAs and the scale by f folds into
// the sum and difference (the plain form is 4 for W v plus 4 additions).
__device__ __forceinline__ void bfly32(double2& u, double2& v, int k) {
  constexpr double C[9] = {1.0,
                           0.98078528040323044912618223613,
                           0.92387953251128675612818318939,
                           0.83146961230254523707878837761,
                           0.70710678118654752440084436210,
                           0.55557023301960222474283081394,
                           0.38268343236508977172845998403,
                           0.19509032201612826784828486847,
                           0.0};
  constexpr double T[5] = {0.0, 0.198912367379658006911597622645, 0.41421356237309504880168872421,
                           0.668178637919298919997757686523, 1.0};  // tan(pi j / 16)
  const double2 a = u;
  if (k == 0) {
    u = cadd(a, v);
    v = csub(a, v);
    return;
  }
  if (k == 8) {  // W = i
    u = make_double2(a.x - v.y, a.y + v.x);
    v = make_double2(a.x + v.y, a.y - v.x);
    return;
  }
  double f, p, q;
  if (k < 4) {  // W = cos (1 + i tan)
    f = C[k];
    p = fma(-T[k], v.y, v.x);
    q = fma(T[k], v.x, v.y);
  } else if (k <= 8) {  // W = sin (cot + i), cot = tan(pi (8 - k) / 16)
    f = C[8 - k];
    p = fma(T[8 - k], v.x, -v.y);
    q = fma(T[8 - k], v.y, v.x);
  } else if (k <= 12) {  // W = sin (cot + i), sin = cos(pi (k - 8) / 16), cot = -tan(pi (k - 8) / 16)
    f = C[k - 8];
    p = fma(-T[k - 8], v.x, -v.y);
    q = fma(-T[k - 8], v.y, v.x);
  } else {  // W = cos (1 + i tan), cos = -cos(pi (16 - k) / 16), tan = -tan(pi (16 - k) / 16)
    f = -C[16 - k];
    p = fma(T[16 - k], v.y, v.x);
    q = fma(-T[16 - k], v.x, v.y);
  }
  u = make_double2(fma(f, p, a.x), fma(f, q, a.y));
  v = make_double2(fma(-f, p, a.x), fma(-f, q, a.y));
}

// dft32 with the fused butterflies (same result to rounding, ~15% fewer FP64 instructions).
__device__ __forceinline__ void dft32f(double2 (&x)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = brev5(i);
    if (r > i) {
      const double2 t = x[i];
      x[i] = x[r];
      x[r] = t;
    }
  }
#pragma unroll
  for (int stage = 1; stage <= 5; ++stage) {
    const int half = 1 << (stage - 1);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int j = e & (half - 1), i = (e >> (stage - 1)) << stage;
      bfly32(x[i + j], x[i + j + half], j << (5 - stage));
    }
  }
}

}  // namespace fft
}  // namespace nsk
