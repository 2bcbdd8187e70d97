// nsk_common.cuh -- device-side building blocks shared by every sketch kernel.
//
// Counter-based draws restated for the GPU.  Each function is the
// random-access form of the reference's sequential stream
// (/root/reference/proj/include/nullsketch/rng.hpp):
//   key derivation       rng.hpp:19-23, 66-71   (host side, nsk_key())
//   Philox4x32-10        rng.hpp:73-96          (philox4x32_10)
//   u32 word i           block i>>2, word i&3   (stream_word)
//   Gaussian #L          rng.hpp:42-54          (gaussian_pair / gaussian_at)
//   sign of row i        rng.hpp:57             (word i, bit 0 set -> +1)
//   next_below(n)        rng.hpp:60-63          (mulhi64)
// Integer draws are bit-exact with the reference; Gaussians differ from glibc
// only by the last-ulp behaviour of CUDA's log / sincospi.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nsk {

struct PhiloxKey {
  uint32_t k0, k1;
};

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ inline PhiloxKey make_key(uint64_t seed, uint64_t stream) {
  uint64_t k = splitmix64(seed) ^ splitmix64(stream ^ 0xb5ad4eceda1ce2a9ULL);
  return PhiloxKey{static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32)};
}

__device__ __forceinline__ uint4 philox4x32_10(PhiloxKey key, uint64_t ctr) {
  uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32);
  uint32_t c2 = 0u, c3 = 0u;
  uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ uint32_t word_of(uint4 b, int w) {
  return w == 0 ? b.x : (w == 1 ? b.y : (w == 2 ? b.z : b.w));
}

__device__ __forceinline__ uint32_t stream_word(PhiloxKey key, uint64_t i) {
  return word_of(philox4x32_10(key, i >> 2), static_cast<int>(i & 3u));
}

// Box-Muller pair from one Philox block (rng.hpp:42-54): returns
// (r cos t, r sin t) = (Gaussian #2b, Gaussian #2b+1).
__device__ __forceinline__ double2 box_muller(uint4 b) {
  const uint64_t a = (static_cast<uint64_t>(b.y) << 32) | b.x;
  const uint64_t c = (static_cast<uint64_t>(b.w) << 32) | b.z;
  const double u1 = 1.0 - static_cast<double>(a >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(c >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);  // sin/cos(2*pi*u2); reference forms t = 2*M_PI*u2 first
  return make_double2(r * cs, r * sn);
}

__device__ __forceinline__ double2 gaussian_pair(PhiloxKey key, uint64_t block) {
  return box_muller(philox4x32_10(key, block));
}

__device__ __forceinline__ double gaussian_at(PhiloxKey key, uint64_t L) {
  const double2 g = gaussian_pair(key, L >> 1);
  return (L & 1u) ? g.y : g.x;
}

__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// Fold of a double's sign with a Rademacher draw: bit 0 of word -> +1.
__device__ __forceinline__ double apply_sign(double x, uint32_t word) {
  return (word & 1u) ? x : -x;
}

}  // namespace nsk

#define NSK_CUDA_OK(expr)                                       \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return ::nsk::cuda_fail(_e, #expr);  \
  } while (0)
