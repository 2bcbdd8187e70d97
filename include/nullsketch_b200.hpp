// nullsketch_b200.hpp -- C++ host API over the C ABI, mirroring the reference.
//
// Same names, argument meaning and error behaviour as the reference's
// /root/reference/proj/include/nullsketch/{sketch,nullspace}.hpp, so a caller
// of the reference can switch by changing the include and the namespace:
//
//   reference (Eigen-backed, host)              this header (B200 device)
//   ------------------------------------------  ------------------------------------------
//   SketchOperator::draw(kind, s, m, seed)      SketchOperator::draw(kind, s, m, seed)
//   SketchOperator::descriptor()/from_...()     same
//   apply(S, A) -> SketchedMatrix               apply(S, A) -> SketchedMatrix
//   solve_k(A, k, S) -> NullspaceResult         solve_k(A, k, S) -> NullspaceResult
//   solve_tol(A, eps, S)                        solve_tol(A, eps, S)
//   residual_certificate(A, W)                  residual_certificate(A, W)
//   update_row / downdate_row (sketch.hpp:90-109) same (S mutated, SA returned)
//   update_column / downdate_column             same
//   tls_solve_sketched(p, S, options) (tls.hpp) same, TlsExistenceError / TlsConditionError
//   tls_solve_exact(p, options), tls_error_metrics(exact, sk) (tls.hpp:60,73)
//   std::invalid_argument / std::out_of_range   same (from NSK_EINVAL / NSK_ERANGE)
//   SvdConvergenceError                         SvdConvergenceError (NSK_ENOCONV)
//
// Matrix is a dense column-major host matrix (real or interleaved complex),
// the reference's value-semantics carrier (matrix.hpp:32-105).  The device
// entry points (nsk_apply, nsk_solve_k on device pointers and a stream) are
// available to callers that keep A resident in HBM.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nullsketch_b200.h"

namespace nullsketch_b200 {

using Index = int64_t;
using Complex = std::complex<double>;

enum class SketchKind { gaussian = NSK_GAUSSIAN, srft = NSK_SRFT, srdct = NSK_SRDCT, srht = NSK_SRHT,
                        countsketch = NSK_COUNTSKETCH };
enum class ScalarKind { real = NSK_REAL, complex = NSK_COMPLEX };

struct SvdConvergenceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == NSK_OK) return;
  const char* msg = nsk_last_error();
  std::string m = msg ? msg : "";
  switch (rc) {
    case NSK_EINVAL: throw std::invalid_argument(m);
    case NSK_ERANGE: throw std::out_of_range(m);
    case NSK_ENOCONV: throw SvdConvergenceError(m);
    case NSK_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error("nullsketch CUDA failure: " + m);
  }
}

inline std::string to_string(SketchKind k) {
  switch (k) {
    case SketchKind::gaussian: return "gaussian";
    case SketchKind::srft: return "srft";
    case SketchKind::srdct: return "srdct";
    case SketchKind::srht: return "srht";
    case SketchKind::countsketch: return "countsketch";
  }
  throw std::logic_error("unknown sketch kind");
}

inline SketchKind sketch_kind_from_string(const std::string& name) {
  for (SketchKind k : {SketchKind::gaussian, SketchKind::srft, SketchKind::srdct, SketchKind::srht,
                       SketchKind::countsketch})
    if (to_string(k) == name) return k;
  throw std::invalid_argument("unknown sketch kind: " + name);
}

// sketch.cpp:99-101 (2n transforms, 4n gaussian); n^2 for countsketch.
inline Index default_sketch_size(SketchKind kind, Index n) {
  if (kind == SketchKind::gaussian) return 4 * n;
  if (kind == SketchKind::countsketch) return n * n;
  return 2 * n;
}

// Dense column-major host matrix; complex entries interleaved (re, im).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols, ScalarKind kind = ScalarKind::real)
      : rows_(rows), cols_(cols), kind_(kind), data_(static_cast<size_t>(rows * cols * ncomp()), 0.0) {}
  static Matrix zeros(Index rows, Index cols, ScalarKind kind) { return Matrix(rows, cols, kind); }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  ScalarKind kind() const { return kind_; }
  bool is_real() const { return kind_ == ScalarKind::real; }
  int ncomp() const { return kind_ == ScalarKind::real ? 1 : 2; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }

  double& operator()(Index i, Index j) {  // real entry
    return data_[static_cast<size_t>(i + j * rows_)];
  }
  double operator()(Index i, Index j) const { return data_[static_cast<size_t>(i + j * rows_)]; }
  Complex at(Index i, Index j) const {
    if (is_real()) return Complex(data_[static_cast<size_t>(i + j * rows_)], 0.0);
    const size_t p = static_cast<size_t>(2 * (i + j * rows_));
    return Complex(data_[p], data_[p + 1]);
  }
  void set(Index i, Index j, Complex v) {
    if (is_real()) {
      data_[static_cast<size_t>(i + j * rows_)] = v.real();
    } else {
      const size_t p = static_cast<size_t>(2 * (i + j * rows_));
      data_[p] = v.real();
      data_[p + 1] = v.imag();
    }
  }

 private:
  Index rows_ = 0, cols_ = 0;
  ScalarKind kind_ = ScalarKind::real;
  std::vector<double> data_;
};

class SketchOperator {
 public:
  static SketchOperator draw(SketchKind kind, Index s, Index m, uint64_t seed) {
    nsk_operator* h = nullptr;
    check(nsk_op_draw(static_cast<int>(kind), s, m, seed, &h));
    return SketchOperator(h);
  }
  static SketchOperator from_descriptor(const std::string& json_text) {
    nsk_operator* h = nullptr;
    check(nsk_op_from_descriptor(json_text.c_str(), &h));
    return SketchOperator(h);
  }
  std::string descriptor() const {
    char buf[512];
    size_t len = 0;
    check(nsk_op_descriptor(h_, buf, sizeof buf, &len));
    return std::string(buf, len);
  }

  SketchOperator(SketchOperator&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  SketchOperator& operator=(SketchOperator&& o) noexcept {
    if (this != &o) {
      nsk_op_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  SketchOperator(const SketchOperator&) = delete;
  SketchOperator& operator=(const SketchOperator&) = delete;
  ~SketchOperator() { nsk_op_destroy(h_); }

  SketchKind kind() const { return static_cast<SketchKind>(info().kind); }
  Index s() const { return info().s; }
  Index m() const { return info().m; }
  Index m_effective() const {  // m plus rows appended by update_row (sketch.hpp:52)
    int64_t me = 0;
    check(nsk_op_state(h_, &me, nullptr, nullptr, nullptr, 0));
    return me;
  }
  nsk_operator* mutable_handle() { return h_; }
  uint64_t seed() const { return info().seed; }
  uint64_t id() const { return info().id; }
  std::vector<int64_t> sample_indices() const {
    std::vector<int64_t> idx(static_cast<size_t>(s()));
    check(nsk_op_sample_indices(h_, idx.data()));
    return idx;
  }
  const nsk_operator* handle() const { return h_; }

 private:
  explicit SketchOperator(nsk_operator* h) : h_(h) {}
  struct Info {
    int kind;
    int64_t s, m;
    uint64_t seed, id;
  };
  Info info() const {
    Info i{};
    check(nsk_op_info(h_, &i.kind, &i.s, &i.m, &i.seed, &i.id));
    return i;
  }
  nsk_operator* h_ = nullptr;
};

struct SketchedMatrix {
  Matrix data;
  uint64_t operator_id = 0;
};

struct NullspaceResult {
  Matrix W;                                   // n x k, orthonormal columns
  std::vector<double> sketched_singular_values;  // all n, non-increasing
  bool has_residual = false;
  double residual_fro = 0.0;
  Index k = 0;
};

inline ScalarKind out_kind(const SketchOperator& S, const Matrix& A) {
  return (S.kind() == SketchKind::srft || !A.is_real()) ? ScalarKind::complex : ScalarKind::real;
}

// sketch.hpp:89
inline SketchedMatrix apply(const SketchOperator& S, const Matrix& A) {
  Matrix out(S.s(), A.cols(), out_kind(S, A));
  check(nsk_apply_host(S.handle(), static_cast<int>(A.kind()), A.rows(), A.cols(), A.data(),
                       A.rows() > 0 ? A.rows() : 1, out.data(), S.s()));
  return {std::move(out), S.id()};
}

// nullspace.hpp:24
inline NullspaceResult solve_k(const Matrix& A, Index k, const SketchOperator& S) {
  NullspaceResult r;
  if (k < 0 || k >= A.cols())
    throw std::invalid_argument("nullspace: k must satisfy 0 <= k < n, got k = " + std::to_string(k) +
                                ", n = " + std::to_string(A.cols()));
  r.W = Matrix(A.cols(), k, out_kind(S, A));
  r.sketched_singular_values.resize(static_cast<size_t>(A.cols()));
  check(nsk_solve_k_host(S.handle(), static_cast<int>(A.kind()), A.rows(), A.cols(), A.data(),
                         A.rows() > 0 ? A.rows() : 1, k, r.W.data(), A.cols(),
                         r.sketched_singular_values.data()));
  r.k = k;
  return r;
}

// ---- multi-GPU (one process per GPU; not in the reference, which is single-process) ----------
// This rank's rows of A: local row j is global row row0 + rstep * j (contiguous blocks for gaussian /
// srht / countsketch, cyclic row0 = g, rstep = P for srft / srdct).
struct RowShard {
  Index row0 = 0, rstep = 1;
};

// An NCCL communicator made by the library (ncclGetUniqueId on rank 0, the 128-byte id distributed by
// the caller, ncclCommInitRank); callers that already own an ncclComm_t pass it to solve_k_sharded.
class NcclComm {
 public:
  static std::string unique_id() {
    std::string id(NSK_NCCL_UNIQUE_ID_BYTES, '\0');
    check(nsk_nccl_unique_id(&id[0]));
    return id;
  }
  NcclComm(int nranks, const std::string& id, int rank) { check(nsk_nccl_comm_init(nranks, id.data(), rank, &c_)); }
  ~NcclComm() { nsk_nccl_comm_destroy(c_); }
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  void* get() const { return c_; }

 private:
  void* c_ = nullptr;
};

// solve_k (nullspace.hpp:24) with A row-sharded across the ranks of `nccl_comm` (an ncclComm_t):
// every rank passes its rows and receives the same W and sigma.
inline NullspaceResult solve_k_sharded(const Matrix& A_local, const RowShard& shard, Index k, const SketchOperator& S,
                                       void* nccl_comm) {
  NullspaceResult r;
  const Index n = A_local.cols();
  if (k < 0 || k >= n)
    throw std::invalid_argument("nullspace: k must satisfy 0 <= k < n, got k = " + std::to_string(k) +
                                ", n = " + std::to_string(n));
  r.W = Matrix(n, k, out_kind(S, A_local));
  r.sketched_singular_values.resize(static_cast<size_t>(n));
  check(nsk_solve_k_sharded_host(S.handle(), static_cast<int>(A_local.kind()), shard.row0, shard.rstep,
                                 A_local.rows(), n, A_local.data(), A_local.rows() > 0 ? A_local.rows() : 1, k,
                                 r.W.data(), n, r.sketched_singular_values.data(), nccl_comm));
  r.k = k;
  return r;
}

// nullspace.hpp:30
inline NullspaceResult solve_tol(const Matrix& A, double eps, const SketchOperator& S) {
  NullspaceResult r;
  const Index n = A.cols();
  Matrix Wfull(n, n > 1 ? n - 1 : 1, out_kind(S, A));
  r.sketched_singular_values.resize(static_cast<size_t>(n));
  int64_t k = 0;
  check(nsk_solve_tol_host(S.handle(), static_cast<int>(A.kind()), A.rows(), n, A.data(),
                           A.rows() > 0 ? A.rows() : 1, eps, &k, Wfull.data(), n,
                           r.sketched_singular_values.data()));
  r.W = Matrix(n, k, Wfull.kind());
  for (Index j = 0; j < k; ++j)
    for (Index i = 0; i < n; ++i) r.W.set(i, j, Wfull.at(i, j));
  r.k = k;
  return r;
}

// nullspace.hpp:33 -- ||A W||_F, one pass over A on the device.
inline double residual_certificate(const Matrix& A, const Matrix& W) {
  if (A.cols() != W.rows())
    throw std::invalid_argument("residual_certificate: basis lives in dimension " + std::to_string(W.rows()) +
                                ", matrix has " + std::to_string(A.cols()) + " columns");
  if (A.kind() != W.kind()) {  // promote the real side, as matmul does (matrix.cpp:13-20)
    auto promote = [](const Matrix& x) {
      Matrix c(x.rows(), x.cols(), ScalarKind::complex);
      for (Index j = 0; j < x.cols(); ++j)
        for (Index i = 0; i < x.rows(); ++i) c.set(i, j, x.at(i, j));
      return c;
    };
    return A.is_real() ? residual_certificate(promote(A), W) : residual_certificate(A, promote(W));
  }
  double out = 0.0;
  check(nsk_residual_fro_host(static_cast<int>(A.kind()), A.rows(), A.cols(), A.data(),
                              A.rows() > 0 ? A.rows() : 1, W.cols(), W.data(), W.rows() > 0 ? W.rows() : 1, &out));
  return out;
}

// ---- incremental maintenance (sketch.hpp:90-109) ---------------------------

namespace detail {
inline Matrix promote(const Matrix& x) {
  if (!x.is_real()) return x;
  Matrix c(x.rows(), x.cols(), ScalarKind::complex);
  for (Index j = 0; j < x.cols(); ++j)
    for (Index i = 0; i < x.rows(); ++i) c.set(i, j, x.at(i, j));
  return c;
}
inline void same_operator(const SketchedMatrix& sa, const SketchOperator& S) {  // sketch.cpp:75-79
  if (sa.operator_id != S.id())
    throw std::invalid_argument("sketched matrix was produced by a different sketch operator");
}
}  // namespace detail

// Append row a_row (1 x n): SA + g a_row / sqrt(s) with g the next Gaussian
// column of stream (seed, 1); mutates S (m_effective grows by one).
inline SketchedMatrix update_row(const SketchedMatrix& sa, SketchOperator& S, const Matrix& a_row) {
  detail::same_operator(sa, S);
  if (a_row.rows() != 1 || a_row.cols() != sa.data.cols())
    throw std::invalid_argument("update_row: expected a 1 x " + std::to_string(sa.data.cols()) + " row");
  SketchedMatrix out{a_row.is_real() ? sa.data : detail::promote(sa.data), sa.operator_id};
  check(nsk_update_row_host(S.mutable_handle(), static_cast<int>(out.data.kind()), out.data.cols(),
                            static_cast<int>(a_row.kind()), a_row.data(), out.data.data(), out.data.rows()));
  return out;
}

// Remove row j whose current content is a_row_j (1 x n): SA - (S e_j) a_row_j.
inline SketchedMatrix downdate_row(const SketchedMatrix& sa, SketchOperator& S, Index j, const Matrix& a_row_j) {
  detail::same_operator(sa, S);
  if (a_row_j.rows() != 1 || a_row_j.cols() != sa.data.cols())
    throw std::invalid_argument("downdate_row: expected a 1 x " + std::to_string(sa.data.cols()) + " row");
  SketchedMatrix out{a_row_j.is_real() ? sa.data : detail::promote(sa.data), sa.operator_id};
  check(nsk_downdate_row_host(S.mutable_handle(), j, static_cast<int>(out.data.kind()), out.data.cols(),
                              static_cast<int>(a_row_j.kind()), a_row_j.data(), out.data.data(), out.data.rows()));
  return out;
}

// Insert the sketch of a_col (m_effective x 1; entries at zeroed rows are
// forced to zero) as column `position` of SA.
inline SketchedMatrix update_column(const SketchedMatrix& sa, const SketchOperator& S, const Matrix& a_col,
                                    Index position) {
  detail::same_operator(sa, S);
  if (position < 0 || position > sa.data.cols()) throw std::out_of_range("update_column: position out of range");
  if (a_col.cols() != 1) throw std::invalid_argument("update_column: expected a single column");
  Matrix col(S.s(), 1, out_kind(S, a_col));
  check(nsk_update_column_host(S.handle(), static_cast<int>(a_col.kind()), a_col.rows(), a_col.data(), col.data()));
  const bool cplx = !sa.data.is_real() || !col.is_real();
  Matrix out(sa.data.rows(), sa.data.cols() + 1, cplx ? ScalarKind::complex : ScalarKind::real);
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i)
      out.set(i, j, j < position ? sa.data.at(i, j) : (j == position ? col.at(i, 0) : sa.data.at(i, j - 1)));
  return {std::move(out), sa.operator_id};
}

// Remove column `position`: an exact splice.
inline SketchedMatrix downdate_column(const SketchedMatrix& sa, Index position) {
  if (position < 0 || position >= sa.data.cols()) throw std::out_of_range("downdate_column: position out of range");
  Matrix out(sa.data.rows(), sa.data.cols() - 1, sa.data.kind());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out.set(i, j, sa.data.at(i, j < position ? j : j + 1));
  return {std::move(out), sa.operator_id};
}

// ---- sketched total least squares (tls.hpp) ---------------------------------

struct TlsProblem {
  Matrix A;  // m x n
  Matrix B;  // m x k, m >= n + k, n >= k
};

struct TlsOptions {
  bool allow_marginal = false;
  bool certificate = false;  // exact ||[A|B] Vk||_F (one pass on the device)
  double cond_limit = 1e12;
};

struct TlsSolution {
  Matrix X;                                     // n x k, X = -V_k1 V_k2^{-1}
  Matrix Vk;                                    // (n+k) x k trailing subspace of S [A|B]
  double tls_residual = 0.0;                    // sqrt(sum of the k trailing sketched sigma^2)
  double cond_Vk2 = 0.0;
  std::vector<double> augmented_singular_values;
  bool has_residual_certificate = false;
  double residual_certificate = 0.0;
};

class TlsExistenceError : public std::runtime_error {
 public:
  TlsExistenceError(double sigma_n_a, double sigma_trailing)
      : std::runtime_error("tls: solution does not exist (sigma_n(A) = " + std::to_string(sigma_n_a) +
                           " <= sigma_{n+1}([A|B]) = " + std::to_string(sigma_trailing) + ")"),
        sigma_n_a_(sigma_n_a),
        sigma_trailing_(sigma_trailing) {}
  double sigma_n_A() const { return sigma_n_a_; }
  double sigma_trailing() const { return sigma_trailing_; }

 private:
  double sigma_n_a_, sigma_trailing_;
};

class TlsConditionError : public std::runtime_error {
 public:
  explicit TlsConditionError(double cond)
      : std::runtime_error("tls: V_k2 is too ill-conditioned (cond = " + std::to_string(cond) + ")"), cond_(cond) {}
  double cond() const { return cond_; }

 private:
  double cond_;
};

namespace detail {
// ||[A|B] Vk||_F, one pass on the device (tls.cpp:55-58).
inline void certify(TlsSolution& r, const Matrix& A, const Matrix& B) {
  const Index m = A.rows(), n = A.cols(), k = B.cols();
  Matrix AB(m, n + k, A.kind());
  for (Index j = 0; j < n + k; ++j)
    for (Index i = 0; i < m; ++i) AB.set(i, j, j < n ? A.at(i, j) : B.at(i, j - n));
  r.residual_certificate = residual_certificate(AB, r.Vk);
  r.has_residual_certificate = true;
}
}  // namespace detail

// tls.hpp: tls_solve_sketched -- the trailing subspace comes from S [A|B].
inline TlsSolution tls_solve_sketched(const TlsProblem& p, const SketchOperator& S, const TlsOptions& options = {}) {
  const Index m = p.A.rows(), n = p.A.cols(), k = p.B.cols();
  if (p.B.rows() != m) throw std::invalid_argument("tls: A and B must have the same number of rows");
  const bool cplx = !p.A.is_real() || !p.B.is_real();
  const Matrix A = cplx ? detail::promote(p.A) : p.A, B = cplx ? detail::promote(p.B) : p.B;
  const ScalarKind ok = (cplx || S.kind() == SketchKind::srft) ? ScalarKind::complex : ScalarKind::real;
  TlsSolution r;
  r.X = Matrix(n, k, ok);
  r.Vk = Matrix(n + k, k, ok);
  r.augmented_singular_values.resize(static_cast<size_t>(n + k));
  double info[4] = {0, 0, 0, 0};
  const int rc = nsk_tls_solve_sketched_host(S.handle(), static_cast<int>(A.kind()), m, n, k, A.data(),
                                             m > 0 ? m : 1, B.data(), m > 0 ? m : 1, options.cond_limit,
                                             options.allow_marginal ? 1 : 0, r.X.data(), n, r.Vk.data(), n + k,
                                             r.augmented_singular_values.data(), info);
  if (rc == NSK_ETLS_EXISTENCE) throw TlsExistenceError(info[2], info[3]);
  if (rc == NSK_ETLS_CONDITION) throw TlsConditionError(info[1]);
  check(rc);
  r.tls_residual = info[0];
  r.cond_Vk2 = info[1];
  if (options.certificate) detail::certify(r, A, B);
  return r;
}

// tls.hpp: tls_solve_exact -- thin QR of [A|B] on the device (shifted
// CholeskyQR3), then the SVDs of the (n+k)^2 triangle (tls.cpp:83-95).
inline TlsSolution tls_solve_exact(const TlsProblem& p, const TlsOptions& options = {}) {
  const Index m = p.A.rows(), n = p.A.cols(), k = p.B.cols();
  if (p.B.rows() != m) throw std::invalid_argument("tls: A and B row counts differ");
  const bool cplx = !p.A.is_real() || !p.B.is_real();
  const Matrix A = cplx ? detail::promote(p.A) : p.A, B = cplx ? detail::promote(p.B) : p.B;
  const ScalarKind ok = cplx ? ScalarKind::complex : ScalarKind::real;
  TlsSolution r;
  r.X = Matrix(n, k, ok);
  r.Vk = Matrix(n + k, k, ok);
  r.augmented_singular_values.resize(static_cast<size_t>(n + k));
  double info[4] = {0, 0, 0, 0};
  const int rc = nsk_tls_solve_exact_host(static_cast<int>(A.kind()), m, n, k, A.data(), m > 0 ? m : 1, B.data(),
                                          m > 0 ? m : 1, options.cond_limit, options.allow_marginal ? 1 : 0,
                                          r.X.data(), n, r.Vk.data(), n + k, r.augmented_singular_values.data(), info);
  if (rc == NSK_ETLS_EXISTENCE) throw TlsExistenceError(info[2], info[3]);
  if (rc == NSK_ETLS_CONDITION) throw TlsConditionError(info[1]);
  check(rc);
  r.tls_residual = info[0];
  r.cond_Vk2 = info[1];
  if (options.certificate) detail::certify(r, A, B);
  return r;
}

// ---- tls_error_metrics (tls.cpp:115-131), small host-side linear algebra -----

struct TlsErrorMetrics {
  double rel_err = 0.0;  // ||X - Xs||_2 / ||X||_2
  double sin_X = 0.0;    // spectral sin between the column spans of X and Xs
  double sin_Vk = 0.0;   // spectral sin between the trailing subspaces
};

namespace detail {
using cd = std::complex<double>;
using Dense = std::vector<std::vector<cd>>;  // column list

inline Dense columns(const Matrix& a) {
  Dense c(static_cast<size_t>(a.cols()), std::vector<cd>(static_cast<size_t>(a.rows())));
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) c[static_cast<size_t>(j)][static_cast<size_t>(i)] = a.at(i, j);
  return c;
}

inline cd dot(const std::vector<cd>& x, const std::vector<cd>& y) {  // x^H y
  cd s = 0.0;
  for (size_t i = 0; i < x.size(); ++i) s += std::conj(x[i]) * y[i];
  return s;
}

// Largest singular value of a small column list (one-sided Jacobi, host).
inline double spectral_norm(Dense c) {
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (size_t p = 0; p + 1 < c.size(); ++p)
      for (size_t q = p + 1; q < c.size(); ++q) {
        const double a = std::real(dot(c[p], c[p])), b = std::real(dot(c[q], c[q]));
        const cd g = dot(c[p], c[q]);
        if (std::abs(g) <= 1e-15 * std::sqrt(a * b) || std::abs(g) == 0.0) continue;
        rotated = true;
        const double zeta = (b - a) / (2.0 * std::abs(g));
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        const cd ph = std::conj(g) / std::abs(g);
        for (size_t i = 0; i < c[p].size(); ++i) {
          const cd up = c[p][i], uq = c[q][i] * ph;
          c[p][i] = cs * up - sn * uq;
          c[q][i] = sn * up + cs * uq;
        }
      }
    if (!rotated) break;
  }
  double best = 0.0;
  for (auto& x : c) best = std::max(best, std::sqrt(std::real(dot(x, x))));
  return best;
}

inline Dense orthonormal(Dense c) {  // modified Gram-Schmidt, twice
  for (int pass = 0; pass < 2; ++pass)
    for (size_t j = 0; j < c.size(); ++j) {
      for (size_t i = 0; i < j; ++i) {
        const cd r = dot(c[i], c[j]);
        for (size_t e = 0; e < c[j].size(); ++e) c[j][e] -= r * c[i][e];
      }
      const double nr = std::sqrt(std::real(dot(c[j], c[j])));
      if (nr > 0)
        for (auto& v : c[j]) v /= nr;
    }
  return c;
}

// Largest sine between two orthonormal column spans: ||(I - U U^H) V||_2 (kernels.cpp:153-167).
inline double sin_theta(const Dense& u, const Dense& v) {
  const Dense& big = u.size() >= v.size() ? u : v;
  Dense small = u.size() >= v.size() ? v : u;
  if (big.empty() || small.empty()) return 0.0;
  for (auto& x : small)
    for (const auto& b : big) {
      const cd r = dot(b, x);
      for (size_t e = 0; e < x.size(); ++e) x[e] -= r * b[e];
    }
  return std::min(1.0, spectral_norm(small));
}
}  // namespace detail

inline TlsErrorMetrics tls_error_metrics(const TlsSolution& exact, const TlsSolution& sk) {
  if (exact.X.rows() != sk.X.rows() || exact.X.cols() != sk.X.cols())
    throw std::invalid_argument("tls_error_metrics: X shapes differ");
  const detail::Dense x = detail::columns(exact.X), xs = detail::columns(sk.X);
  const double xn = detail::spectral_norm(x);
  if (xn == 0.0) throw std::invalid_argument("tls_error_metrics: exact X is zero; rel_err undefined");
  detail::Dense d = x;
  for (size_t j = 0; j < d.size(); ++j)
    for (size_t i = 0; i < d[j].size(); ++i) d[j][i] -= xs[j][i];
  TlsErrorMetrics m;
  m.rel_err = detail::spectral_norm(d) / xn;
  m.sin_X = detail::sin_theta(detail::orthonormal(x), detail::orthonormal(xs));
  m.sin_Vk = detail::sin_theta(detail::columns(exact.Vk), detail::columns(sk.Vk));
  return m;
}

}  // namespace nullsketch_b200
