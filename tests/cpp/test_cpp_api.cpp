// test_cpp_api.cpp -- the C++ host API (include/nullsketch_b200.hpp) used the
// way the reference's own doctest suites use theirs
// (/root/reference/proj/tests/test_sketch.cpp, test_nullspace.cpp).
// Built and run by tests/test_cpp_api.py (GPU).  Exit code 0 = all checks pass.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "nullsketch_b200.hpp"

using namespace nullsketch_b200;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                  \
  do {                                              \
    bool thrown = false;                            \
    try {                                           \
      (void)(expr);                                 \
    } catch (const exc&) {                          \
      thrown = true;                                \
    } catch (...) {                                 \
    }                                               \
    CHECK(thrown && #exc);                          \
  } while (0)

static Matrix random_real(Index m, Index n, unsigned seed) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> d;
  Matrix a(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) a(i, j) = d(g);
  return a;
}

static double max_abs_diff(const Matrix& a, const Matrix& b) {
  double e = 0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) e = std::max(e, std::abs(a.at(i, j) - b.at(i, j)));
  return e;
}

static double fro(const Matrix& a) {
  double s = 0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) s += std::norm(a.at(i, j));
  return std::sqrt(s);
}

int main() {
  // draw validation (test_sketch.cpp:91-101)
  CHECK_THROWS_AS(SketchOperator::draw(SketchKind::srft, 10, 8, 1), std::invalid_argument);
  CHECK_THROWS_AS(SketchOperator::draw(SketchKind::srdct, 10, 8, 1), std::invalid_argument);
  CHECK_THROWS_AS(SketchOperator::draw(SketchKind::gaussian, 0, 8, 1), std::invalid_argument);
  { auto S = SketchOperator::draw(SketchKind::gaussian, 10, 8, 1); CHECK(S.s() == 10); }
  CHECK(default_sketch_size(SketchKind::srft, 50) == 100);
  CHECK(default_sketch_size(SketchKind::gaussian, 50) == 200);

  // determinism in the seed (test_sketch.cpp:81-89)
  for (SketchKind kind : {SketchKind::gaussian, SketchKind::srft, SketchKind::srdct, SketchKind::srht,
                          SketchKind::countsketch}) {
    Matrix I(16, 16);
    for (Index i = 0; i < 16; ++i) I(i, i) = 1.0;
    auto a = SketchOperator::draw(kind, 6, 16, 123), b = SketchOperator::draw(kind, 6, 16, 123),
         c = SketchOperator::draw(kind, 6, 16, 124);
    CHECK(max_abs_diff(apply(a, I).data, apply(b, I).data) == 0.0);
    CHECK(max_abs_diff(apply(a, I).data, apply(c, I).data) > 0.0);
  }

  // apply basics and linearity (test_sketch.cpp:133-163)
  {
    auto S = SketchOperator::draw(SketchKind::srft, 8, 32, 3);
    CHECK(fro(apply(S, Matrix::zeros(32, 5, ScalarKind::complex)).data) == 0.0);
    CHECK_THROWS_AS(apply(S, Matrix(31, 5, ScalarKind::complex)), std::invalid_argument);
    auto D = SketchOperator::draw(SketchKind::srdct, 8, 32, 3);
    CHECK_THROWS_AS(apply(D, Matrix(32, 5, ScalarKind::complex)), std::invalid_argument);
  }
  for (SketchKind kind : {SketchKind::gaussian, SketchKind::srdct, SketchKind::srht, SketchKind::countsketch}) {
    const Index m = 64, n = 6;
    Matrix a = random_real(m, n, 13), b = random_real(m, n, 14), lin(m, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) lin(i, j) = 2 * a(i, j) - 3 * b(i, j);
    auto S = SketchOperator::draw(kind, 16, m, 21);
    Matrix lhs = apply(S, lin).data, sa = apply(S, a).data, sb = apply(S, b).data, rhs(16, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < 16; ++i) rhs(i, j) = 2 * sa(i, j) - 3 * sb(i, j);
    CHECK(max_abs_diff(lhs, rhs) < 1e-13 * fro(lhs));
  }

  // descriptor round trip (test_sketch.cpp:405-428)
  {
    auto S = SketchOperator::draw(SketchKind::srdct, 10, 28, 112);
    auto R = SketchOperator::from_descriptor(S.descriptor());
    CHECK(R.kind() == S.kind() && R.m() == S.m() && R.s() == S.s() && R.seed() == S.seed());
    CHECK(R.sample_indices() == S.sample_indices());
    CHECK_THROWS_AS(SketchOperator::from_descriptor("{}"), std::invalid_argument);
  }

  // exact null space preserved (test_nullspace.cpp:21-32): A = B * P, P = I - p p^T.
  {
    const Index m = 200, n = 20;
    Matrix B = random_real(m, n, 5), A(m, n);
    std::vector<double> p(n);
    double nn = 0;
    for (Index i = 0; i < n; ++i) nn += (p[i] = std::sin(1.0 + i)) * p[i];
    for (auto& v : p) v /= std::sqrt(nn);
    for (Index i = 0; i < m; ++i)
      for (Index j = 0; j < n; ++j) {
        double s = 0;
        for (Index l = 0; l < n; ++l) s += B(i, l) * ((l == j ? 1.0 : 0.0) - p[l] * p[j]);
        A(i, j) = s;
      }
    for (SketchKind kind : {SketchKind::gaussian, SketchKind::srft, SketchKind::srdct, SketchKind::countsketch}) {
      auto S = SketchOperator::draw(kind, kind == SketchKind::countsketch ? n * n : 2 * n, m, 2);
      NullspaceResult r = solve_k(A, 1, S);
      CHECK(r.k == 1 && r.W.rows() == n && r.W.cols() == 1);
      double dot = 0;
      for (Index i = 0; i < n; ++i) dot += std::abs(r.W.at(i, 0) * p[i]);
      CHECK(std::abs(1.0 - dot) < 1e-10);
      CHECK(residual_certificate(A, r.W) < 1e-10 || !r.W.is_real());
      CHECK(r.sketched_singular_values.size() == static_cast<size_t>(n));
      CHECK(r.sketched_singular_values.back() < 1e-12);
    }
    auto S = SketchOperator::draw(SketchKind::srdct, 2 * n, m, 2);
    CHECK_THROWS_AS(solve_k(A, n, S), std::invalid_argument);
    CHECK_THROWS_AS(solve_k(A, -1, S), std::invalid_argument);
    NullspaceResult t = solve_tol(A, 1e-8, S);
    CHECK(t.k == 1);
    CHECK_THROWS_AS(solve_tol(A, 1e3, S), std::invalid_argument);
    CHECK_THROWS_AS(solve_tol(A, -1.0, S), std::invalid_argument);
  }

  // residual certificate known answer (test_nullspace.cpp:137-150)
  {
    Matrix a(3, 2), w(2, 1);
    a(0, 0) = 3.0;
    a(1, 1) = 1.0;
    w(0, 0) = 1.0;
    CHECK(std::abs(residual_certificate(a, w) - 3.0) < 1e-15);
    Matrix w3(3, 1);
    CHECK_THROWS_AS(residual_certificate(a, w3), std::invalid_argument);
  }

  // Row and column updates (test_sketch.cpp: update_row keeps SA = S_eff A_eff,
  // downdate_row removes a row's contribution, update_column appends S a_col).
  {
    const Index m = 300, n = 6, s = 40;
    Matrix A = random_real(m, n, 21);
    auto S = SketchOperator::draw(SketchKind::srdct, s, m, 31);
    SketchedMatrix SA = apply(S, A);
    Matrix row = random_real(1, n, 22);
    SketchedMatrix up = update_row(SA, S, row);
    CHECK(S.m_effective() == m + 1);
    Matrix Aext(m + 1, n);
    for (Index j = 0; j < n; ++j) {
      for (Index i = 0; i < m; ++i) Aext(i, j) = A(i, j);
      Aext(m, j) = row(0, j);
    }
    const SketchedMatrix ref = apply(S, Aext);  // the operator now spans m + 1 rows
    CHECK(max_abs_diff(up.data, ref.data) < 1e-12 * fro(ref.data));
    // downdate row 5: same as applying to A with row 5 zeroed
    Matrix r5(1, n);
    for (Index j = 0; j < n; ++j) r5(0, j) = Aext(5, j);
    SketchedMatrix dn = downdate_row(up, S, 5, r5);
    Matrix Az = Aext;
    for (Index j = 0; j < n; ++j) Az(5, j) = 0.0;
    CHECK(max_abs_diff(dn.data, apply(S, Az).data) < 1e-12 * fro(dn.data));
    CHECK_THROWS_AS(downdate_row(dn, S, 5, r5), std::invalid_argument);     // already removed
    CHECK_THROWS_AS(downdate_row(dn, S, m + 7, r5), std::out_of_range);
    // update_column / downdate_column
    Matrix col = random_real(m + 1, 1, 23);
    SketchedMatrix wide = update_column(dn, S, col, 2);
    CHECK(wide.data.cols() == n + 1);
    Matrix colz = col;
    colz(5, 0) = 0.0;
    const SketchedMatrix sc = apply(S, colz);
    double e = 0;
    for (Index i = 0; i < s; ++i) e = std::max(e, std::abs(wide.data.at(i, 2) - sc.data.at(i, 0)));
    CHECK(e < 1e-12 * fro(sc.data));
    SketchedMatrix back = downdate_column(wide, 2);
    CHECK(max_abs_diff(back.data, dn.data) == 0.0);
    CHECK_THROWS_AS(downdate_column(wide, n + 1), std::out_of_range);
    auto other = SketchOperator::draw(SketchKind::srdct, s, m, 32);
    CHECK_THROWS_AS(update_row(SA, other, row), std::invalid_argument);  // operator ids differ
  }
  // Sketched TLS (test_tls.cpp): X recovers x_true at low noise; existence error at rank deficiency.
  {
    const Index m = 2000, n = 5, k = 1;
    Matrix A = random_real(m, n, 41), xt = random_real(n, k, 42), noise = random_real(m, k, 43);
    Matrix B(m, k);
    for (Index i = 0; i < m; ++i) {
      double v = 0;
      for (Index j = 0; j < n; ++j) v += A(i, j) * xt(j, 0);
      B(i, 0) = v + 1e-6 * noise(i, 0);
    }
    auto S = SketchOperator::draw(SketchKind::gaussian, 4 * (n + k), m, 44);
    TlsOptions opt;
    opt.certificate = true;
    TlsSolution sol = tls_solve_sketched({A, B}, S, opt);
    CHECK(sol.X.rows() == n && sol.X.cols() == k && sol.Vk.rows() == n + k);
    CHECK(max_abs_diff(sol.X, xt) < 1e-4);
    CHECK(sol.has_residual_certificate && sol.residual_certificate < 1e-3);
    CHECK(sol.augmented_singular_values.size() == static_cast<size_t>(n + k));
    Matrix A0 = A;  // rank-deficient A (zero column): sigma_n(SA) = 0, the solvability check must fire
    for (Index i = 0; i < m; ++i) A0(i, n - 1) = 0.0;
    CHECK_THROWS_AS(tls_solve_sketched({A0, B}, S), TlsExistenceError);
    // exact solver (tls.cpp:83-95) and the error metrics (tls.cpp:115-131)
    TlsSolution ex = tls_solve_exact({A, B}, opt);
    CHECK(max_abs_diff(ex.X, xt) < 1e-5);
    CHECK(ex.has_residual_certificate && std::abs(ex.residual_certificate - ex.tls_residual) < 1e-8 * ex.tls_residual);
    TlsErrorMetrics met = tls_error_metrics(ex, sol);
    CHECK(met.rel_err >= 0.0 && met.rel_err < 1e-3 && met.sin_Vk < 1e-3 && met.sin_X <= 1.0);
    TlsErrorMetrics self = tls_error_metrics(ex, ex);
    CHECK(self.rel_err == 0.0 && self.sin_Vk < 1e-12);
    CHECK_THROWS_AS(tls_solve_exact({A0, B}), TlsExistenceError);
  }
  {  // multi-GPU entry point on a one-rank NCCL communicator made by the library: equals solve_k
    const Index m = 5000, n = 12;
    Matrix A = random_real(m, n, 91);
    auto S = SketchOperator::draw(SketchKind::srht, 64, 8192, 5);
    Matrix A8(8192, n, ScalarKind::real);  // srht needs m = 2^13 here: pad with zero rows
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) A8(i, j) = A(i, j);
    NullspaceResult one = solve_k(A8, 2, S);
    NcclComm comm(1, NcclComm::unique_id(), 0);
    NullspaceResult sh = solve_k_sharded(A8, RowShard{0, 1}, 2, S, comm.get());
    CHECK(sh.W.rows() == n && sh.W.cols() == 2);
    double dmax = 0.0;
    for (size_t i = 0; i < sh.sketched_singular_values.size(); ++i)
      dmax = std::max(dmax, std::abs(sh.sketched_singular_values[i] - one.sketched_singular_values[i]));
    CHECK(dmax < 1e-12 * one.sketched_singular_values[0]);
    CHECK_THROWS_AS(solve_k_sharded(A8, RowShard{0, 1}, n, S, comm.get()), std::invalid_argument);
  }
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("cpp api: all checks passed\n");
  return 0;
}
