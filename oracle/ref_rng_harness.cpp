// ref_rng_harness.cpp -- drives the reference's own, unmodified RNG header
// (/root/reference/proj/include/nullsketch/rng.hpp) through the exact call
// sequences the reference library issues, so that the oracle restatement in
// nsk_oracle.c and the CUDA draws can be pinned bit-for-bit against it.
//
// TEST INFRASTRUCTURE ONLY: built by oracle/Makefile into oracle/_ref/ (never
// committed), used by tests/golden/make_golden.py and the -m "not gpu" tests
// when the reference tree is present.  No reference source is copied: the
// header is included from where it lies.
#include <cstdint>
#include <vector>

#include "nullsketch/rng.hpp"

using nullsketch::PhiloxStream;

extern "C" {

// next_u32 x count from a fresh stream (rng.hpp:25-28).
void nskref_words(std::uint64_t seed, std::uint64_t stream, std::uint64_t count,
                  std::uint32_t* out) {
  PhiloxStream r(seed, stream);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next_u32();
}

// next_gaussian x count from a fresh stream (rng.hpp:42-54).
void nskref_gaussians(std::uint64_t seed, std::uint64_t stream, std::uint64_t count,
                      double* out) {
  PhiloxStream r(seed, stream);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next_gaussian();
}

// next_double x count (rng.hpp:36-39); used by the AAA sampler protocol.
void nskref_doubles(std::uint64_t seed, std::uint64_t stream, std::uint64_t count,
                    double* out) {
  PhiloxStream r(seed, stream);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next_double();
}

// SketchOperator::draw for gaussian (sketch.cpp:117-121): G column-major s x m.
void nskref_gaussian_G(std::uint64_t seed, std::int64_t s, std::int64_t m, double* out) {
  PhiloxStream base(seed, 0);
  for (std::int64_t j = 0; j < m; ++j)
    for (std::int64_t i = 0; i < s; ++i) out[j * s + i] = base.next_gaussian();
}

// SketchOperator::draw for srft/srdct (sketch.cpp:122-126): m signs, then the
// sorted Fisher-Yates sample.
void nskref_srtt_draw(std::uint64_t seed, std::int64_t m, std::int64_t s, double* signs,
                      std::int64_t* idx) {
  PhiloxStream base(seed, 0);
  for (std::int64_t i = 0; i < m; ++i) signs[i] = base.next_sign();
  std::vector<std::int64_t> v = nullsketch::sample_without_replacement(m, s, base);
  for (std::int64_t i = 0; i < s; ++i) idx[i] = v[static_cast<std::size_t>(i)];
}

// CountSketch draw protocol defined by this framework on top of the reference
// stream: m x next_sign(), then m x next_below(s).
void nskref_countsketch_draw(std::uint64_t seed, std::int64_t m, std::int64_t s,
                             std::int32_t* bucket, double* sign) {
  PhiloxStream base(seed, 0);
  for (std::int64_t i = 0; i < m; ++i) sign[i] = base.next_sign();
  for (std::int64_t i = 0; i < m; ++i)
    bucket[i] = static_cast<std::int32_t>(base.next_below(static_cast<std::uint64_t>(s)));
}

// Row-update Gaussians (sketch.cpp:273-275, 325-328): appended column c, entry
// i = next_gaussian #(c*s + i) of stream (seed, 1).
void nskref_update_gaussians(std::uint64_t seed, std::int64_t s, std::int64_t p, double* out) {
  PhiloxStream upd(seed, 1);
  for (std::int64_t c = 0; c < p; ++c)
    for (std::int64_t i = 0; i < s; ++i) out[c * s + i] = upd.next_gaussian();
}

}  // extern "C"
