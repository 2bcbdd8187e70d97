/*
 * nullsketch_b200.h -- C ABI of the B200-native sketch-and-solve hot path.
 *
 * Drop-in boundary for the reference's C++ API (paths relative to
 * /root/reference/proj):
 *
 *   reference symbol                                       replaced by
 *   ---------------------------------------------------   ---------------------------
 *   SketchOperator::draw(kind, s, m, seed)  sketch.hpp:42   nsk_op_draw
 *   SketchOperator::descriptor()            sketch.hpp:48   nsk_op_descriptor
 *   SketchOperator::from_descriptor(json)   sketch.hpp:47   nsk_op_from_descriptor
 *   SketchOperator::{kind,s,m,seed,id}()    sketch.hpp:50-59 nsk_op_info
 *   (the sorted sample R, sketch.hpp:77)                    nsk_op_sample_indices
 *   apply(S, A)                             sketch.hpp:89   nsk_apply / nsk_apply_host
 *   solve_k(A, k, S)                        nullspace.hpp:24 nsk_solve_k / nsk_solve_k_host
 *   solve_tol(A, eps, S)                    nullspace.hpp:30 nsk_solve_tol / nsk_solve_tol_host
 *   residual_certificate(A, W)              nullspace.hpp:33 nsk_residual_fro
 *   svd(SA) -> trailing V block             kernels.hpp:24 + nullspace.cpp:10-19
 *                                                           nsk_svd_trailing
 *   (no reference: row-sharded multi-GPU partial S_g A_g)   nsk_apply_shard
 *
 * Conventions (matrix.hpp:13-18, 32-105 of the reference):
 *   - dense column-major storage, leading dimension in elements;
 *   - NSK_REAL = IEEE double, NSK_COMPLEX = interleaved (re, im) doubles
 *     (std::complex<double> / Eigen::MatrixXcd layout);
 *   - srft output is always complex; gaussian keeps the input kind; srdct,
 *     srht and countsketch reject complex input (sketch.cpp:219-221);
 *   - the caller owns every buffer; the library owns only the opaque
 *     operator (its descriptor state: kind, s, m, seed, and the sorted
 *     sample).  Gaussian S, signs and hash buckets are regenerated on the
 *     device from the counter-based stream and never stored.
 *   - "device" entry points take device pointers and a cudaStream_t (passed
 *     as void*); they are stream-ordered and do not synchronise unless a
 *     host result is returned (nsk_solve_tol's k, nsk_residual_fro's value).
 *     "_host" entry points take host pointers (the reference's value
 *     semantics) and return when the results are in host memory.
 *
 * Errors: C++ exceptions of the reference become status codes
 *   std::invalid_argument -> NSK_EINVAL, std::out_of_range -> NSK_ERANGE,
 *   SvdConvergenceError (kernels.hpp:18-20) -> NSK_ENOCONV,
 *   CUDA failures -> NSK_ECUDA, allocation failure -> NSK_ENOMEM;
 *   nsk_last_error() returns the thread-local message of the last failure.
 *   No entry point returns NaN silently (kernels.hpp:22-23).
 *
 * Threading: an operator is immutable after draw; concurrent calls on the
 * same operator from several threads/streams are safe.
 * Results are bit-identical across re-runs on the same GPU model and launch
 * configuration: every reduction has a fixed order (no float atomics).
 */
#ifndef NULLSKETCH_B200_H
#define NULLSKETCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nsk_operator nsk_operator;

enum nsk_kind {
  NSK_GAUSSIAN = 0,    /* dense N(0,1) G scaled by 1/sqrt(s)            sketch.hpp:24 */
  NSK_SRFT = 1,        /* sqrt(m/s) R F^* D, complex                     sketch.hpp:25-26 */
  NSK_SRDCT = 2,       /* sqrt(m/s) R C_III^T D, real                     sketch.hpp:27 */
  NSK_SRHT = 3,        /* sqrt(m/s) R H D, m a power of two (no reference) */
  NSK_COUNTSKETCH = 4  /* SA[h(i),:] += sigma(i) A[i,:]   (no reference) */
};

enum nsk_scalar { NSK_REAL = 0, NSK_COMPLEX = 1 };

enum nsk_status {
  NSK_OK = 0,
  NSK_EINVAL = 1,
  NSK_ERANGE = 2,
  NSK_ENOCONV = 3,
  NSK_ECUDA = 4,
  NSK_ENOMEM = 5,
  NSK_ETLS_EXISTENCE = 6, /* TlsExistenceError (tls.hpp:37-48) */
  NSK_ETLS_CONDITION = 7  /* TlsConditionError (tls.hpp:50-57) */
};

/* Thread-local message describing the last non-OK status. */
const char* nsk_last_error(void);

/* Library version string and the CUDA architecture it was compiled for. */
const char* nsk_version(void);

/* ---- operator lifecycle (sketch.hpp:42-59) ------------------------------ */

/* SketchOperator::draw.  s >= 1, m >= 1; s <= m for srft/srdct/srht; srht
 * additionally needs m to be a power of two.  Draws the sample indices
 * (Fisher-Yates over stream (seed, 0) after the m sign words) on the host. */
int nsk_op_draw(int kind, int64_t s, int64_t m, uint64_t seed, nsk_operator** out);

void nsk_op_destroy(nsk_operator* op);

int nsk_op_info(const nsk_operator* op, int* kind, int64_t* s, int64_t* m, uint64_t* seed,
                uint64_t* id);

/* Sorted sample R (s indices) for srft/srdct/srht; NSK_EINVAL otherwise. */
int nsk_op_sample_indices(const nsk_operator* op, int64_t* idx_host);

/* JSON descriptor {"format":1,"kind":..,"s":..,"m":..,"seed":..,"appended":0,
 * "zeroed_rows":[]} (sketch.cpp:303-313).  Writes at most cap bytes including
 * the terminating NUL; *len receives the length without NUL. */
int nsk_op_descriptor(const nsk_operator* op, char* buf, size_t cap, size_t* len);

/* SketchOperator::from_descriptor (sketch.cpp:315-337): replays the draw, then
 * the appended Gaussian columns (stream (seed, 1)) and the zeroed rows, so the
 * operator applies exactly as the one that wrote the descriptor. */
int nsk_op_from_descriptor(const char* json, nsk_operator** out);

/* ---- apply (sketch.hpp:89) ---------------------------------------------- */

/* SA (s x n) = S A (m x n) on the device.  ldsa >= s.  For srft with
 * NSK_REAL input, SA is complex (interleaved) as in the reference. */
int nsk_apply(const nsk_operator* op, int scalar, int64_t m, int64_t n, const void* A,
              int64_t lda, void* SA, int64_t ldsa, void* stream);

/* Row shard of apply for multi-GPU: the caller holds local rows
 * j = 0..mloc-1 of A, which are global rows row0 + rstep*j.  Writes the
 * partial SA_g = S[:, rows] A_g; the sum of the partials over a partition of
 * the rows is apply(S, A).  gaussian/countsketch/srht need rstep == 1
 * (contiguous shards; countsketch: row0 a multiple of 512, and each shard
 * builds its tables for its own rows only); srft/srdct take cyclic shards
 * (row0 = g < rstep = P, P | m: the local length-m/P transform, decimation in
 * time) and, less efficiently, any other row map. */
int nsk_apply_shard(const nsk_operator* op, int scalar, int64_t row0, int64_t rstep,
                    int64_t mloc, int64_t n, const void* A, int64_t lda, void* SA,
                    int64_t ldsa, void* stream);

/* ---- solve (nullspace.hpp:24-33) ---------------------------------------- */

/* Trailing k right singular vectors of a sketch SA (s x n, s >= n > k >= 0)
 * by on-device one-sided Jacobi: W (n x k, column k-1 belongs to the
 * smallest singular value) and all n singular values, non-increasing, into
 * sigma (device, n doubles).  W has the scalar kind of SA. */
int nsk_svd_trailing(int scalar, int64_t s, int64_t n, const void* SA, int64_t ldsa, int64_t k,
                     void* W, int64_t ldw, double* sigma, void* stream);

/* solve_k: apply, then nsk_svd_trailing.  Device pointers. */
int nsk_solve_k(const nsk_operator* op, int scalar, int64_t m, int64_t n, const void* A,
                int64_t lda, int64_t k, void* W, int64_t ldw, double* sigma, void* stream);

/* solve_tol: k = number of sketched singular values below eps; selecting
 * all n is NSK_EINVAL.  W must hold n x (n-1) entries; *k_out (host) is
 * written after the stream has been synchronised. */
int nsk_solve_tol(const nsk_operator* op, int scalar, int64_t m, int64_t n, const void* A,
                  int64_t lda, double eps, int64_t* k_out, void* W, int64_t ldw, double* sigma,
                  void* stream);

/* ||A W||_F in one pass over A (device pointers; *out on the host). */
int nsk_residual_fro(int scalar, int64_t m, int64_t n, const void* A, int64_t lda, int64_t k,
                     const void* W, int64_t ldw, double* out, void* stream);

/* ---- host-buffer entry points (the reference's value semantics) --------- */

int nsk_apply_host(const nsk_operator* op, int scalar, int64_t m, int64_t n, const void* A,
                   int64_t lda, void* SA, int64_t ldsa);

int nsk_solve_k_host(const nsk_operator* op, int scalar, int64_t m, int64_t n, const void* A,
                     int64_t lda, int64_t k, void* W, int64_t ldw, double* sigma);

int nsk_solve_tol_host(const nsk_operator* op, int scalar, int64_t m, int64_t n, const void* A,
                       int64_t lda, double eps, int64_t* k_out, void* W, int64_t ldw,
                       double* sigma);

int nsk_residual_fro_host(int scalar, int64_t m, int64_t n, const void* A, int64_t lda, int64_t k,
                          const void* W, int64_t ldw, double* out);

/* ---- incremental maintenance (sketch.hpp:90-109, sketch.cpp:234-301) ---- */

/* Operator state: m_effective = m + appended rows, the sorted zeroed rows
 * (up to cap of them into zeroed_rows when non-null). */
int nsk_op_state(const nsk_operator* op, int64_t* m_eff, int64_t* appended, int64_t* nzeroed,
                 int64_t* zeroed_rows, int64_t cap);

/* update_row: append row a_row (1 x n, device) to the underlying matrix.  Draws
 * the next Gaussian column g of stream (seed, 1) and adds g a_row / sqrt(s) to
 * SA (s x n, device) in place; m_effective grows by one.  srdct rejects a
 * complex row; a complex row needs a complex SA (promote it first). */
int nsk_update_row(nsk_operator* op, int scalar_sa, int64_t n, int scalar_row, const void* a_row, void* SA,
                   int64_t ldsa, void* stream);

/* downdate_row: remove row j whose current content is a_row (1 x n, device):
 * SA -= (S e_j) a_row, then row j is recorded as zeroed.  NSK_ERANGE for j
 * outside [0, m_effective), NSK_EINVAL if j was already removed; warns on
 * stderr when fewer than 2s live rows remain (sketch.cpp:296-299). */
int nsk_downdate_row(nsk_operator* op, int64_t j, int scalar_sa, int64_t n, int scalar_row, const void* a_row,
                     void* SA, int64_t ldsa, void* stream);

/* update_column: out (s x 1, device) = S a_col with a_col's entries at zeroed
 * rows forced to zero (sketch.cpp:244-252); the caller splices it into SA
 * (downdate_column is a pure splice and needs no call). */
int nsk_update_column(const nsk_operator* op, int scalar, int64_t m, const void* a_col, void* out,
                      void* stream);

/* Host-buffer variants of the three calls above (SA, rows and columns in host
 * memory, column-major; SA is updated in place, out receives the s entries). */
int nsk_update_row_host(nsk_operator* op, int scalar_sa, int64_t n, int scalar_row, const void* a_row, void* SA,
                        int64_t ldsa);
int nsk_downdate_row_host(nsk_operator* op, int64_t j, int scalar_sa, int64_t n, int scalar_row,
                          const void* a_row, void* SA, int64_t ldsa);
int nsk_update_column_host(const nsk_operator* op, int scalar, int64_t m, const void* a_col, void* out);

/* ---- sketched total least squares (tls.hpp:59-65, tls.cpp:97-113) ------- */

/* X (n x k) = -V_k1 V_k2^{-1} from the trailing k right singular vectors Vk
 * ((n+k) x k) of S [A | B]; sigma receives the n+k sketched singular values;
 * info[4] = {tls_residual, cond(V_k2), sigma_n(S A), sigma_{n+1}(S [A|B])}.
 * NSK_ETLS_EXISTENCE when sigma_n(S A) <= sigma_{n+1} and !allow_marginal,
 * NSK_ETLS_CONDITION when cond(V_k2) > cond_limit.  Device pointers. */
int nsk_tls_solve_sketched(const nsk_operator* op, int scalar, int64_t m, int64_t n, int64_t k,
                           const void* A, int64_t lda, const void* B, int64_t ldb, double cond_limit,
                           int allow_marginal, void* X, int64_t ldx, void* Vk, int64_t ldv, double* sigma,
                           double* info, void* stream);
int nsk_tls_solve_sketched_host(const nsk_operator* op, int scalar, int64_t m, int64_t n, int64_t k,
                                const void* A, int64_t lda, const void* B, int64_t ldb, double cond_limit,
                                int allow_marginal, void* X, int64_t ldx, void* Vk, int64_t ldv,
                                double* sigma, double* info);

/* ---- exact total least squares (tls.hpp:59-61, tls.cpp:83-95) ----------- */

/* Same outputs as nsk_tls_solve_sketched, from the thin QR of [A | B] (no
 * sketch): R = shifted CholeskyQR3 factor on the device (cuBLAS level-3
 * Gram products and triangular solves), then the SVDs of the (n+k)^2
 * triangle; sigma = singular values of [A|B], info[2] = sigma_n(A).
 * Replaces tls_solve_exact (tls.cpp:83).  NSK_ENOCONV on a Cholesky
 * breakdown (NaN/Inf input). */
int nsk_tls_solve_exact(int scalar, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                        int64_t ldb, double cond_limit, int allow_marginal, void* X, int64_t ldx, void* Vk,
                        int64_t ldv, double* sigma, double* info, void* stream);
int nsk_tls_solve_exact_host(int scalar, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                             const void* B, int64_t ldb, double cond_limit, int allow_marginal, void* X,
                             int64_t ldx, void* Vk, int64_t ldv, double* sigma, double* info);

/* ---- multi-GPU: row shards + NCCL (one process per GPU) ------------------
 * SA = sum_g S[:, rows_g] A_g.  Rank g holds local rows j of
 * A_local = global rows row0 + rstep * j (contiguous shards: rstep = 1; srft /
 * srdct cyclic shards: row0 = g, rstep = P, P | m).  The operator regenerates S
 * for the global rows; one ncclAllReduce (sum, FP64) of the s x n partials on
 * `nccl_comm` (an ncclComm_t) leaves the same SA on every rank.  Callers of the
 * reference API this replaces: solve_k (nullspace.hpp:24, nullspace.cpp:23-32)
 * and apply (sketch.hpp:89) with A row-sharded across GPUs.  NCCL is loaded at
 * run time (libnccl.so.2, or NSK_NCCL_LIB); NSK_ECUDA if it is absent. */
#define NSK_NCCL_UNIQUE_ID_BYTES 128
/* ncclGetUniqueId / ncclCommInitRank / ncclCommDestroy for callers without a communicator. */
int nsk_nccl_unique_id(char* id_out /* NSK_NCCL_UNIQUE_ID_BYTES */);
int nsk_nccl_comm_init(int nranks, const char* id, int rank, void** comm_out);
int nsk_nccl_comm_destroy(void* comm);
/* SA (device, s x n, ldsa) = the full sketch, on every rank. */
int nsk_apply_allreduce(const nsk_operator* op, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                        const void* A_local, int64_t lda, void* SA, int64_t ldsa, void* nccl_comm, void* stream);
/* solve_k on row shards: the all-reduced SA, then the on-device SVD on every rank (bitwise-identical SA
 * gives identical W and sigma everywhere).  W (device, n x k, ldw), sigma (device, n). */
int nsk_solve_k_sharded(const nsk_operator* op, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                        const void* A_local, int64_t lda, int64_t k, void* W, int64_t ldw, double* sigma,
                        void* nccl_comm, void* stream);
/* The same from host buffers (A_local m_loc x n with lda, W n x k with ldw, sigma n). */
int nsk_solve_k_sharded_host(const nsk_operator* op, int scalar, int64_t row0, int64_t rstep, int64_t mloc,
                             int64_t n, const void* A_local, int64_t lda, int64_t k, void* W, int64_t ldw,
                             double* sigma, void* nccl_comm);

/* ---- memory --------------------------------------------------------------
 * Scratch (device copies of host inputs, partial sketches, SVD workspaces)
 * comes from a library-private stream-ordered pool per device, so it never
 * holds on to the default pool other libraries (PyTorch) allocate from.  Freed
 * blocks stay mapped for the next call; this returns them to the device
 * (synchronises the current device first) and frees the pinned host buffers of
 * the host-buffer entry points (the pageable-input staging ring and the
 * CountSketch schedule scratch), which the next such call allocates again. */
int nsk_release_scratch(void);

/* ---- instrumentation (bench.py; no effect on results) ------------------- */

/* Number of CUDA kernels this library has launched in this process. */
int64_t nsk_kernel_launches(void);

/* When enabled, every apply records CUDA events around its dominant kernel
 * (gaussian_sketch / srht / countsketch / srtt main kernel) on the caller's
 * stream; nsk_timing_collect synchronises those events, returns the summed
 * duration and count since the last collect, and clears them. */
void nsk_timing_enable(int on);
int nsk_timing_collect(double* total_ms, int64_t* count);
/* Name (as ncu prints it) of the kernel most recently timed on this thread. */
const char* nsk_timing_kernel(void);

#ifdef __cplusplus
}
#endif

#endif /* NULLSKETCH_B200_H */
