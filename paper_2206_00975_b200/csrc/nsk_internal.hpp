// nsk_internal.hpp -- host-side state and kernel launchers behind the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <deque>
#include <functional>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "nsk_common.cuh"

namespace nsk {

enum Kind { GAUSSIAN = 0, SRFT = 1, SRDCT = 2, SRHT = 3, COUNTSKETCH = 4 };
enum Status { OK = 0, EINVAL_ = 1, ERANGE_ = 2, ENOCONV = 3, ECUDA = 4, ENOMEM_ = 5 };
constexpr int NOTAPPLICABLE = -100;  // internal: a specialised path declines, the caller falls back

int fail(int code, const std::string& msg);
const char* last_error();  // this thread's message of the last failure
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
  int64_t* srtt_freq = nullptr;     // srft/srdct: sample indices sorted by idx mod 1024 (tile FFT bin)
  int32_t* srtt_row = nullptr;      // output row of each sorted slot
  uint64_t* srdct_sgn = nullptr;    // srdct (srdct_stream.cu): per tile, row class and column, main | mirror negate bits
  uint64_t* srft_sgn = nullptr;     // srft (srft_ws.cu): per 16-column tile, row class and column pair, 64 negate bits
  int64_t* dct_freq = nullptr;      // srdct (srdct_stream.cu): v index n(a) of each sample, sorted by n mod 1024
  int32_t* dct_row = nullptr;       // output row of each sorted srdct slot
  // CountSketch owner schedule (cs_schedule.cpp) over CS_T-row tiles.
  uint64_t* cs_ent = nullptr;       // [tile][warp][CS_GMAX][32] packed entries
  uint8_t* cs_cnt = nullptr;        // [tile][warp] iterations
  int64_t cs_ntiles = 0;            // full tiles covered (window tiles 0 .. cs_ntiles-1)
  // CountSketch row window: cs_table / the schedule cover global rows [cs_base, cs_base + cs_rows)
  // (cs_base a multiple of CS_T), so a rank of the multi-GPU path holds tables for its shard only.
  int64_t cs_base = 0, cs_rows = 0;
};

// CountSketch owner kernel geometry (countsketch.cu / cs_schedule.cpp).
constexpr int CS_T = 4096;        // rows per tile (12-bit row field of an entry)
constexpr int CS_T_MAX = 4096;
constexpr int CS_THREADS = 1024;  // bin owners per CTA
constexpr int CS_WARPS = CS_THREADS / 32;
constexpr int CS_GMAX = 6;        // groups of 4 iterations per warp and tile
int build_cs_schedule(const uint32_t* table, int64_t ntiles, int T, int64_t s, std::vector<uint64_t>& ent,
                      std::vector<uint8_t>& cnt);
int build_cs_schedule_into(const uint32_t* table, int64_t ntiles, int T, int64_t s, uint64_t* ent, uint8_t* cnt);
// Process-wide pinned host scratch (grown on demand, kept): the CountSketch table readback and schedule
// upload go through it at DMA speed.  Callers hold the returned lock while they use the buffer.
std::unique_lock<std::mutex> pinned_scratch(size_t bytes, void** out);
void release_pinned_host();
// Whether the owner kernel applies (bins fit 4 registers per thread, s large
// enough that ~4 rows per lane per tile spread over distinct owners, at least
// one full tile; NSK_CS_MODE=stream|tma forces the older kernels).
bool cs_owner_eligible(int64_t s, int64_t m);

// Device-side table builders (run once per operator and device).
int build_sign_mask(PhiloxKey key, int64_t m, uint32_t** out);
int build_cs_table(PhiloxKey key, int64_t m, int64_t s, int64_t base, int64_t rows, uint32_t** out);
int build_sign_bits(PhiloxKey key, int64_t m, uint32_t** out);
int build_srdct_sgn(const uint32_t* sign_bits, int64_t m, uint64_t** out);  // null when m % 16384 != 0
int build_srft_sgn(const uint32_t* sign_bits, int64_t m, uint64_t** out);  // null when m % 16384 != 0

// A shard view: local row j of A is global row row0 + rstep * j, j < mloc.
struct RowMap {
  int64_t row0 = 0, rstep = 1, mloc = 0;
};

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

  // Incremental state (sketch.hpp:70-80): row updates append Gaussian columns
  // drawn from stream (seed, 1) (appended column c = Gaussians #(c*s + i));
  // row downdates record the removed rows (sorted).  Single writer.
  int64_t appended = 0;
  std::vector<int64_t> zeroed;
  int64_t m_eff() const { return m + appended; }
  bool is_zeroed(int64_t j) const;

  mutable std::mutex mu;
  mutable std::deque<DeviceTables> dev;  // one entry per device used (stable addresses)
  // Uploads on first use on the current device.  CountSketch tables cover a row window: the first
  // call that needs rows [row_lo, row_hi) not covered yet builds one for them (tile-aligned);
  // row_hi < 0 means m, row_hi <= row_lo means no CountSketch rows are needed.
  const DeviceTables* tables(int64_t row_lo = 0, int64_t row_hi = -1) const;
  // Device bitmask of the zeroed rows (m_eff bits) on the current device in
  // *out, nullptr when no row is zeroed.  Re-uploaded after every downdate.
  // Returns ECUDA (with the message set) when the upload fails -- never a
  // silent "no zeroed rows".
  int zero_mask(const uint32_t** out) const;
  mutable std::vector<std::pair<int, uint32_t*>> zmask_dev;  // (device, mask)
  // srft cyclic-shard tables for the warp-specialised tile kernel (srft_ws.cu), per (device, g, P):
  // the shard's sign bits and negate masks, its frequencies a mod (m / P) sorted by bin, the output
  // row of each slot and the shard twiddle w_m^{a g} of each output row.
  struct ShardTables {
    int device = -1;
    int64_t g = 0, P = 1;
    uint32_t* bits = nullptr;
    uint64_t* sgn = nullptr;
    int64_t* freq = nullptr;
    int32_t* row = nullptr;
    double2* post = nullptr;
  };
  mutable std::deque<ShardTables> shard_tabs;
  mutable uint64_t zmask_version = 0, state_version = 0;
  ~Operator();
};

// Gaussian sketch with an explicit stream and zero mask: SA (+)= (1/sqrt s) G A
// with G(i, j) = Gaussian #((row0 + j) * s + i) of `key`; rows whose bit
// (zoff + row0 + j) is set in zmask contribute nothing.
int gaussian_apply_key(PhiloxKey key, int64_t s, const uint32_t* zmask, int64_t zoff, int ncomp,
                       const RowMap& rows, int64_t n, const double* A, int64_t lda, double* SA,
                       int64_t ldsa, cudaStream_t st);

// The same for [A | B] (B: kb columns, ldb) in one pass, SA columns n .. n+kb-1 = S B.
int gaussian_apply_key2(PhiloxKey key, int64_t s, const uint32_t* zmask, int64_t zoff, int ncomp,
                        const RowMap& rows, int64_t n, const double* A, int64_t lda, int64_t kb, const double* B,
                        int64_t ldb, double* SA, int64_t ldsa, cudaStream_t st);

int draw_operator(int kind, int64_t s, int64_t m, uint64_t seed, Operator** out);

// Sampled Fisher-Yates with an O(s) map (bit-identical to rng.hpp:108-121).
std::vector<int64_t> sample_without_replacement(PhiloxKey key, int64_t m, int64_t s);

// ---- kernel launchers (return Status) ------------------------------------

int gaussian_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                   int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srht_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda,
               double* SA, int64_t ldsa, cudaStream_t st);
int countsketch_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A,
                      int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srtt_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
               int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);

// srft / srdct as samples of one DFT of a local sequence (srtt_general.cu): the
// engine's eligibility (full matrix or cyclic shard g of P with P | m), the
// per-slot tables of shard g (frequency in [0, N), conjugation flag, shard
// twiddle) and the fixed-order reduction of per-CTA partials into SA.
struct Scratch;
bool srtt_general_eligible(const Operator& op, const RowMap& rows);
int shard_slot_tables(const Operator& op, int64_t g, int64_t N, Scratch& tab, int64_t** dfreq, double2** dpost,
                      uint8_t** dconj, cudaStream_t st);
int srtt_post_reduce(int kind, const double2* part, int64_t rstride, int64_t cstride, int64_t ranges, int64_t n,
                     int ns, int base, const double2* post, const uint8_t* conj, double scale, double* SA,
                     int64_t ldsa, cudaStream_t st);

// One-sided Jacobi on [R; I] (2n x n, ld 2n) inside one thread-block cluster
// (cluster_jacobi.cu); NOTAPPLICABLE when it does not fit one cluster.
int cluster_jacobi(int ncomp, double* X, int64_t n, double tol, int* counter, cudaStream_t st);
// QRCP of R + one-sided Jacobi on R'^H in one cluster (cluster_jacobi.cu); writes
// the same [W; V] layout.  NOTAPPLICABLE when it does not fit; *degenerate
// (device) is raised when R is exactly singular and the caller must rerun.
int cluster_svd_rt(int ncomp, double* X, int64_t n, double tol, int* counter, int* degenerate, cudaStream_t st);
// One-sided Jacobi SVD of SA (s x n, ncomp = 1 real / 2 complex interleaved).
// Writes the trailing k right singular vectors and all n singular values
// (device, non-increasing).  Returns ENOCONV if the sweep limit is hit.
int jacobi_trailing(int ncomp, int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k,
                    double* W, int64_t ldw, double* sigma, cudaStream_t st);
// The same plus all n2 singular values of the leading s x n2 block (one shared QR; the two Jacobi
// stages run concurrently).
int jacobi_trailing_pair(int ncomp, int64_t s, int64_t n, const double* SA, int64_t ldsa, int64_t k, double* W,
                         int64_t ldw, double* sigma, int64_t n2, double* sigma2, cudaStream_t st);

// R factor (N x N upper, ld N, N = n + k) of the thin QR of [A | B] (m x N),
// shifted CholeskyQR3 (tall_qr.cu).  B may be null when k = 0.
int tall_qr_r(int nc, int64_t m, int64_t n, const double* A, int64_t lda, int64_t k, const double* B, int64_t ldb,
              double* R, cudaStream_t st);

int residual_fro(int ncomp, int64_t m, int64_t n, const double* A, int64_t lda, int64_t k,
                 const double* W, int64_t ldw, double* out_host, cudaStream_t st);

// ---- incremental maintenance (sketch.cpp:234-301) --------------------------
// out (s entries, ncomp_out) = S e_j: column j of the current operator.
int sketch_column(const Operator& op, int64_t j, double* out, int ncomp_out, cudaStream_t st);
// SA(:, c) -= col * row(c) (rank one; complex when either side is).
int rank1_update(double* SA, int64_t ldsa, int ncomp_sa, int64_t s, int64_t n, const double* col, int ncomp_col,
                 const double* row, int ncomp_row, double alpha, cudaStream_t st);
// SA += T (T s x n dense, ncomp_t <= ncomp_sa).
int accumulate(double* SA, int64_t ldsa, int ncomp_sa, const double* T, int64_t s, int64_t n, int ncomp_t,
               cudaStream_t st);
// Zero the entries of a device column (m_eff rows) at the operator's zeroed rows.
int mask_zeroed(const Operator& op, double* col, int ncomp, cudaStream_t st);

// ---- sketched total least squares (tls.cpp:97-113) -------------------------
// X = -V1 V2^{-1} from the trailing (n+k) x k basis Vk (device, one CTA).
int tls_corner(int ncomp, const double* Vk, int64_t ldv, int64_t n, int64_t k, double* X, int64_t ldx,
               cudaStream_t st);

// The library's own stream-ordered memory pool on the current device (created
// on first use).  Freed scratch stays mapped in it -- repeated calls with
// gigabyte-sized scratch (host staging, the exact solver's Q) would otherwise
// re-map HBM every call -- without touching the device's default pool that
// PyTorch and other libraries use; nsk_release_scratch() trims it.
cudaMemPool_t scratch_pool();

// Stream-ordered scratch allocation from scratch_pool().
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
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(&p, bytes ? bytes : 8, pool, s);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int sm_count();

// ---- host -> device (h2d.cpp) ---------------------------------------------
// Copies host A (m x n column-major, lda, elem bytes per entry) to device dA
// in row chunks of `chunk` rows on a per-thread copy stream, chunk-major: chunk
// c is a rows_c x n column-major block (ld rows_c) at element offset c chunk n
// (one chunk = plain column-major, ld m).  Each landed chunk is handed to on_chunk(r0, rows, landed): the
// callback owns the event (its work must wait on it, then destroy it) and may
// defer that work; without a callback st simply waits for every chunk.
// Pageable sources stream through a pinned staging ring filled by host
// threads; pinned sources are DMAed directly.
using ChunkFn = std::function<int(int64_t, int64_t, cudaEvent_t)>;
// dcols (>= n): columns of each destination chunk block (room for a second column block after A).
int h2d_rows(const void* A, int64_t m, int64_t n, int64_t lda, size_t elem, void* dA, int64_t chunk,
             cudaStream_t st, const ChunkFn& on_chunk, int64_t dcols = 0);
bool host_is_pinned(const void* p);
cudaStream_t copy_stream();
cudaStream_t thread_stream();

// ---- instrumentation -------------------------------------------------------
void count_launch(int n = 1);
// Records events around the dominant kernel of an apply when timing is enabled.
// `name` is the kernel's name as ncu prints it (nsk_timing_kernel reports the
// name of the most recently timed kernel).
struct KernelTimer {
  cudaStream_t st;
  void* pair = nullptr;
  KernelTimer(cudaStream_t s, const char* name, bool enabled = true);
  void stop();
};

}  // namespace nsk
