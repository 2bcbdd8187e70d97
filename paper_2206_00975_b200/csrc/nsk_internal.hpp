// nsk_internal.hpp -- host-side state and kernel launchers behind the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <deque>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "nsk_common.cuh"

namespace nsk {

enum Kind { GAUSSIAN = 0, SRFT = 1, SRDCT = 2, SRHT = 3, COUNTSKETCH = 4 };
enum Status { OK = 0, EINVAL_ = 1, ERANGE_ = 2, ENOCONV = 3, ECUDA = 4, ENOMEM_ = 5 };

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
const char* kind_name(int kind);

// Per-device copy of the small draw tables an operator needs on the GPU.
struct DeviceTables {
  int device = -1;
  int64_t* idx = nullptr;           // s sorted sample indices (srft/srdct/srht)
  uint32_t* srht_slot = nullptr;    // SRHT output slots sorted by r_lo: r_lo | (r_hi << lo_bits)
  int32_t* srht_row = nullptr;      // output row of each slot
  uint32_t* sign_mask = nullptr;    // SRHT: m-bit Rademacher mask, lane-transposed per 1024 rows
  uint32_t* cs_table = nullptr;     // CountSketch: per-row bucket | sign | tile chain (4 B/row)
  uint32_t* sign_bits = nullptr;    // srft/srdct: bit j of word j/32 = Rademacher bit of row j
};

// Device-side table builders (run once per operator and device).
int build_sign_mask(PhiloxKey key, int64_t m, uint32_t** out);
int build_cs_table(PhiloxKey key, int64_t m, int64_t s, uint32_t** out);
int build_sign_bits(PhiloxKey key, int64_t m, uint32_t** out);

// The operator is its descriptor (sketch.cpp:303-313): nothing else is stored.
struct Operator {
  int kind = GAUSSIAN;
  int64_t s = 0, m = 0;
  uint64_t seed = 0, id = 0;
  PhiloxKey key0{0, 0};  // stream (seed, 0): base draws
  PhiloxKey key1{0, 0};  // stream (seed, 1): row updates
  std::vector<int64_t> idx;  // sorted sample (srft/srdct/srht)
  // SRHT slot table (host): outputs ordered by their low index bits.
  int srht_lo_bits = 0;
  std::vector<uint32_t> srht_slot;
  std::vector<int32_t> srht_row;

  mutable std::mutex mu;
  mutable std::deque<DeviceTables> dev;  // one entry per device used (stable addresses)
  const DeviceTables* tables() const;      // uploads on first use on the current device
  ~Operator();
};

int draw_operator(int kind, int64_t s, int64_t m, uint64_t seed, Operator** out);

// Sampled Fisher-Yates with an O(s) map (bit-identical to rng.hpp:108-121).
std::vector<int64_t> sample_without_replacement(PhiloxKey key, int64_t m, int64_t s);

// ---- kernel launchers (return Status) ------------------------------------
// A shard view: local row j of A is global row row0 + rstep * j, j < mloc.
struct RowMap {
  int64_t row0 = 0, rstep = 1, mloc = 0;
};

int gaussian_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                   int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srht_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda,
               double* SA, int64_t ldsa, cudaStream_t st);
int countsketch_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A,
                      int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srtt_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
               int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);

// One-sided Jacobi SVD of SA (s x n, ncomp = 1 real / 2 complex interleaved).
// Writes the trailing k right singular vectors and all n singular values
// (device, non-increasing).  Returns ENOCONV if the sweep limit is hit.
int jacobi_trailing(int ncomp, int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k,
                    double* W, int64_t ldw, double* sigma, cudaStream_t st);

int residual_fro(int ncomp, int64_t m, int64_t n, const double* A, int64_t lda, int64_t k,
                 const double* W, int64_t ldw, double* out_host, cudaStream_t st);

// Stream-ordered scratch allocation (cudaMallocAsync from the device pool).
struct Scratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t s) {
    st = s;
    return cudaMallocAsync(&p, bytes ? bytes : 8, s);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int sm_count();

// ---- instrumentation -------------------------------------------------------
void count_launch(int n = 1);
// Records events around the dominant kernel of an apply when timing is enabled.
struct KernelTimer {
  cudaStream_t st;
  void* pair = nullptr;
  explicit KernelTimer(cudaStream_t s, bool enabled = true);
  void stop();
};

}  // namespace nsk
