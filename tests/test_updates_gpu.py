"""Incremental sketch maintenance and sketched TLS on the device, against the
reference's own identities (tests/test_sketch.cpp:202-428, test_tls.cpp:135-174)
and against the oracle restatement (oracle/sketch_oracle.py)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsk():
    import torch
    from paper_2206_00975_b200 import build
    build.build()
    import paper_2206_00975_b200 as nsk
    torch.cuda.init()
    return nsk


def dev(x):
    import torch
    return torch.from_numpy(np.asfortranarray(x)).cuda()


def host(t):
    return t.cpu().numpy()


def fro(x):
    return float(np.linalg.norm(x))


KINDS3 = ["gaussian", "srft", "srdct"]


def _mat(oracle, kind, m, n, seed):
    return oracle.random_real(m, n, seed) if kind != "srft" else oracle.random_complex(m, n, seed)


@pytest.mark.parametrize("kind", KINDS3 + ["srht", "countsketch"])
def test_column_update_and_downdate(nsk, oracle, kind):
    # test_sketch.cpp:202-255
    m, n = 64 if kind == "srht" else 40, 5
    a = _mat(oracle, kind, m, n, 31)
    c = _mat(oracle, kind, m, 1, 32)
    S = nsk.SketchOperator.draw(kind, 12, m, 33)
    sa = nsk.apply(S, dev(a))
    up = nsk.update_column(sa, S, dev(np.zeros((m, 1), dtype=a.dtype)), n)
    assert up.data.shape[1] == n + 1 and float(abs(up.data[:, n]).max()) == 0.0
    for pos in (0, 2, n):  # append then downdate restores the sketch bit for bit
        back = nsk.downdate_column(nsk.update_column(sa, S, dev(c), pos), pos)
        assert np.array_equal(host(back.data), host(sa.data))
    up = nsk.update_column(sa, S, dev(c), 2)
    widened = np.concatenate([a[:, :2], c, a[:, 2:]], axis=1)
    assert np.max(np.abs(host(up.data) - host(nsk.apply(S, dev(widened)).data))) < 1e-13 * fro(a)
    down = nsk.downdate_column(sa, 1)
    narrowed = np.concatenate([a[:, :1], a[:, 2:]], axis=1)
    assert np.max(np.abs(host(down.data) - host(nsk.apply(S, dev(narrowed)).data))) < 1e-13 * fro(a)
    with pytest.raises(IndexError):
        nsk.update_column(sa, S, dev(c), n + 1)
    with pytest.raises(IndexError):
        nsk.downdate_column(sa, n)
    other = nsk.SketchOperator.draw(kind, 12, m, 99)
    with pytest.raises(ValueError):
        nsk.update_column(sa, other, dev(c), 0)


@pytest.mark.parametrize("kind", KINDS3 + ["srht", "countsketch"])
def test_row_update_matches_widened_operator(nsk, oracle, kind):
    # test_sketch.cpp:270-284: update_row(apply(S, a), row) == apply(S', [a; row])
    m, n, s = (32 if kind == "srht" else 24), 4, 10
    a = _mat(oracle, kind, m, n, 43)
    row = _mat(oracle, kind, 1, n, 44)
    S = nsk.SketchOperator.draw(kind, s, m, 45)
    up = nsk.update_row(nsk.apply(S, dev(a)), S, dev(row))
    taller = np.vstack([a, row])
    assert S.appended_count == 1 and S.m_effective == m + 1
    assert np.max(np.abs(host(up.data) - host(nsk.apply(S, dev(taller)).data))) < 1e-12 * fro(a)
    # and the oracle's restatement agrees
    op = oracle.draw(kind, s, m, 45)
    ref = oracle.update_row(op, oracle.apply_state(op, a), row)
    assert np.max(np.abs(host(up.data) - ref)) < 1e-12 * fro(a)


def test_zero_rows_leave_sketch_unchanged(nsk, oracle):
    # test_sketch.cpp:259-268
    m, n, s = 24, 4, 10
    S = nsk.SketchOperator.draw("srft", s, m, 41)
    a = oracle.random_complex(m, n, 42)
    sa = nsk.apply(S, dev(a))
    up = nsk.update_row(sa, S, dev(np.zeros((1, n), dtype=np.complex128)))
    up = nsk.update_row(up, S, dev(np.zeros((1, n), dtype=np.complex128)))
    assert np.array_equal(host(up.data), host(sa.data))
    assert S.m_effective == m + 2 and up.data.shape[0] == s


@pytest.mark.parametrize("j", [0, 7, 39])
def test_gaussian_row_downdate_is_column_removal(nsk, oracle, j):
    # test_sketch.cpp:306-318: downdate equals drop_col(S, j) * drop_row(A, j)
    m, n, s = 40, 6, 25
    a = oracle.random_real(m, n, 61)
    S = nsk.SketchOperator.draw("gaussian", s, m, 62)
    sd = host(nsk.apply(S, dev(np.eye(m))).data)
    down = nsk.downdate_row(nsk.apply(S, dev(a)), S, j, dev(a[j:j + 1]))
    ref = np.delete(sd, j, axis=1) @ np.delete(a, j, axis=0)
    assert np.max(np.abs(host(down.data) - ref)) < 1e-13 * fro(a)
    assert S.live_rows == m - 1 and S.zeroed_rows == [j]
    # the zeroed G column no longer contributes to apply()
    assert np.max(np.abs(host(nsk.apply(S, dev(a)).data) - ref)) < 1e-13 * fro(a)


def test_downdate_errors(nsk, oracle):
    m, n, s = 40, 6, 25
    a = oracle.random_real(m, n, 61)
    S = nsk.SketchOperator.draw("gaussian", s, m, 64)
    sa = nsk.apply(S, dev(a))
    zero = nsk.downdate_row(sa, S, 3, dev(np.zeros((1, n))))
    assert np.array_equal(host(zero.data), host(sa.data))
    with pytest.raises(ValueError):
        nsk.downdate_row(zero, S, 3, dev(a[3:4]))
    with pytest.raises(IndexError):
        nsk.downdate_row(zero, S, m, dev(a[3:4]))


@pytest.mark.parametrize("kind,j", [("srft", 9), ("srdct", 0), ("srht", 5), ("countsketch", 11)])
def test_subsampled_row_downdate_matches_zeroed_row_oracle(nsk, oracle, kind, j):
    # test_sketch.cpp:320-337
    m, n, s = (32 if kind == "srht" else 36), 5, 14
    a = _mat(oracle, kind, m, n, 71)
    S = nsk.SketchOperator.draw(kind, s, m, 72)
    down = nsk.downdate_row(nsk.apply(S, dev(a)), S, j, dev(a[j:j + 1]))
    zeroed = a.copy()
    zeroed[j] = 0
    assert np.max(np.abs(host(down.data) - host(nsk.apply(S, dev(zeroed)).data))) < 1e-13 * fro(a)
    assert S.zeroed_rows == [j]


def test_downdating_an_appended_row_undoes_the_update(nsk, oracle):
    # test_sketch.cpp:338-346
    m, n, s = 36, 5, 14
    a = oracle.random_complex(m, n, 75)
    S = nsk.SketchOperator.draw("srft", s, m, 76)
    sa = nsk.apply(S, dev(a))
    row = oracle.random_complex(1, n, 77)
    back = nsk.downdate_row(nsk.update_row(sa, S, dev(row)), S, m, dev(row))
    assert np.max(np.abs(host(back.data) - host(sa.data))) < 1e-14 * fro(a)


def test_update_column_zeroes_removed_rows(nsk, oracle):
    # test_sketch.cpp:350-362
    m, n, s = 20, 3, 8
    a = oracle.random_complex(m, n, 81)
    S = nsk.SketchOperator.draw("srft", s, m, 82)
    sa = nsk.downdate_row(nsk.apply(S, dev(a)), S, 4, dev(a[4:5]))
    c = oracle.random_complex(m, 1, 83)
    up = nsk.update_column(sa, S, dev(c), n)
    c0 = c.copy()
    c0[4] = 0
    ref = host(nsk.apply(S, dev(c0)).data)
    assert np.max(np.abs(host(up.data)[:, n:] - ref)) < 1e-13 * fro(c)


def test_identical_call_sequences_bit_identical(nsk, oracle):
    # test_sketch.cpp:391-403
    m, n, s = 32, 4, 12
    a = oracle.random_complex(m, n, 101)
    r = oracle.random_complex(1, n, 103)

    def run():
        S = nsk.SketchOperator.draw("srft", s, m, 102)
        sa = nsk.apply(S, dev(a))
        sa = nsk.update_row(sa, S, dev(r))
        sa = nsk.downdate_row(sa, S, 5, dev(a[5:6]))
        sa = nsk.update_column(sa, S, dev(np.zeros((m + 1, 1), dtype=np.complex128)), 0)
        return host(sa.data)
    assert np.array_equal(run(), run())


@pytest.mark.parametrize("kind", KINDS3 + ["srht", "countsketch"])
def test_descriptor_replays_updates(nsk, oracle, kind):
    # test_sketch.cpp:405-428
    m, n, s = (32 if kind == "srht" else 28), 3, 10
    a = _mat(oracle, kind, m, n, 111)
    S = nsk.SketchOperator.draw(kind, s, m, 112)
    sa = nsk.apply(S, dev(a))
    sa = nsk.update_row(sa, S, dev(oracle.random_real(1, n, 113)))
    sa = nsk.update_row(sa, S, dev(oracle.random_real(1, n, 114)))
    sa = nsk.downdate_row(sa, S, 6, dev(a[6:7]))
    R = nsk.SketchOperator.from_descriptor(S.descriptor())
    assert (R.kind, R.m_effective, R.zeroed_rows, R.appended_count) == (S.kind, S.m_effective, S.zeroed_rows, 2)
    eye = np.eye(S.m_effective)
    assert np.array_equal(host(nsk.apply(R, dev(eye)).data), host(nsk.apply(S, dev(eye)).data))
    bad = ('{"format":1,"kind":"srft","s":4,"m":8,"seed":1,"appended":0,"zeroed_rows":[9]}')
    with pytest.raises(ValueError):
        nsk.SketchOperator.from_descriptor(bad)


def test_solve_after_updates_matches_oracle(nsk, oracle):
    m, n, s = 300, 12, 48
    a = oracle.random_real(m, n, 5)
    S = nsk.SketchOperator.draw("gaussian", s, m, 6)
    op = oracle.draw("gaussian", s, m, 6)
    row = oracle.random_real(1, n, 7)
    sa = nsk.update_row(nsk.apply(S, dev(a)), S, dev(row))
    ref = oracle.update_row(op, oracle.apply_state(op, a), row)
    sa = nsk.downdate_row(sa, S, 17, dev(a[17:18]))
    ref = oracle.downdate_row(op, ref, 17, a[17])
    assert np.max(np.abs(host(sa.data) - ref)) < 1e-13 * fro(a)
    taller = np.vstack([a, row])
    taller[17] = 0
    assert np.max(np.abs(host(nsk.apply(S, dev(taller)).data) - oracle.apply_state(op, taller))) < 1e-12 * fro(a)


# ----------------------------------------------------------------------------- TLS

def _tls_problem(oracle, m, n, k, noise, seed):
    A = oracle.random_real(m, n, seed)
    X = oracle.random_real(n, k, seed + 1)
    B = A @ X + noise * oracle.random_real(m, k, seed + 2)
    return A, B, X


@pytest.mark.parametrize("kind", ["gaussian", "srdct", "srht"])
def test_tls_recovers_consistent_problem(nsk, oracle, kind):
    # test_tls.cpp:135-150: zero noise -> sketched TLS recovers X to 1e-8
    m, n, k = 1024, 10, 2
    A, B, X = _tls_problem(oracle, m, n, k, 0.0, 3)
    S = nsk.SketchOperator.draw(kind, 4 * (n + k), m, 5)
    sol = nsk.tls_solve_sketched(dev(A), dev(B), S, allow_marginal=True)
    assert np.linalg.norm(host(sol.X) - X, 2) / np.linalg.norm(X, 2) < 1e-8


def test_tls_matches_oracle_under_noise(nsk, oracle):
    m, n, k = 4096, 20, 1
    A, B, X = _tls_problem(oracle, m, n, k, 1e-3, 11)
    S = nsk.SketchOperator.draw("gaussian", 2 * (n + k), m, 12)
    sol = nsk.tls_solve_sketched(dev(A), dev(B), S, certificate=True)
    Xr, Vr, svr, resr, condr = oracle.tls_solve_sketched(A, B, oracle.draw("gaussian", 2 * (n + k), m, 12))
    assert np.linalg.norm(host(sol.X) - Xr) <= 1e-9 * np.linalg.norm(Xr)
    assert oracle.sin_theta(host(sol.Vk), Vr) < 1e-10
    assert abs(sol.tls_residual - resr) <= 1e-10 * resr
    assert np.max(np.abs(host(sol.augmented_singular_values) - svr)) <= 1e-12 * svr[0]
    assert sol.residual_certificate is not None and sol.residual_certificate > 0
    # sketched TLS tracks the truth under noise (test_tls.cpp:152-174: 1e-2)
    assert np.linalg.norm(host(sol.X) - X) / np.linalg.norm(X) < 1e-2


def test_tls_validation(nsk, oracle):
    m, n, k = 200, 10, 2
    A, B, _ = _tls_problem(oracle, m, n, k, 1e-3, 21)
    S = nsk.SketchOperator.draw("gaussian", 4 * (n + k), m, 22)
    with pytest.raises(ValueError):
        nsk.tls_solve_sketched(dev(A[:, :1]), dev(B), S)  # n < k
    with pytest.raises(ValueError):
        nsk.tls_solve_sketched(dev(A), dev(B), nsk.SketchOperator.draw("gaussian", 4 * (n + k), m + 1, 22))
    with pytest.raises(ValueError):
        nsk.tls_solve_sketched(dev(A), dev(B), nsk.SketchOperator.draw("gaussian", n, m, 22))
    # rank-deficient A: sigma_n(SA) = 0 is not above sigma_{n+1}(S[A|B]) -> TlsExistenceError
    Adef = A.copy()
    Adef[:, -1] = 0.0
    with pytest.raises(nsk.TlsExistenceError):
        nsk.tls_solve_sketched(dev(Adef), dev(B), S)


# ---- exact TLS (tls.cpp:83-95) on the device: shifted CholeskyQR3 + SVD of R

@pytest.mark.parametrize("cplx", [False, True])
def test_tls_exact_matches_oracle(nsk, oracle, cplx):
    m, n, k = 3000, 24, 2
    A, B, X = _tls_problem(oracle, m, n, k, 1e-3, 31)
    if cplx:
        A = A + 1j * oracle.random_real(m, n, 41)
        B = A @ (X + 1j * oracle.random_real(n, k, 42)) + 1e-3 * oracle.random_real(m, k, 43)
    sol = nsk.tls_solve_exact(dev(A), dev(B), certificate=True)
    Xr, Vr, svr, resr, condr = oracle.tls_solve_exact(A, B)
    assert np.max(np.abs(host(sol.augmented_singular_values) - svr)) <= 1e-12 * svr[0]
    assert oracle.sin_theta(host(sol.Vk), Vr) < 1e-10
    assert np.linalg.norm(host(sol.X) - Xr) <= 1e-9 * np.linalg.norm(Xr)
    assert abs(sol.tls_residual - resr) <= 1e-10 * resr
    assert abs(sol.cond_Vk2 - condr) <= 1e-8 * condr
    # the certificate of the exact solution is its residual (||[A|B] Vk|| = sigma tail)
    assert abs(sol.residual_certificate - resr) <= 1e-8 * resr


def test_tls_exact_ill_conditioned(nsk, oracle):
    # kappa([A|B]) = 1e11 (plain CholeskyQR breaks down above ~1e8): the shift
    # keeps the first Cholesky alive, two more passes restore orthogonality;
    # sigma and the trailing subspace (gap 1e-8) match Householder.
    m, n, k = 2000, 16, 1
    sig = np.concatenate([np.logspace(0, -8, n), [1e-11]])
    C = oracle.make_test_matrix(m, n + k, sig, 51)
    A, B = C[:, :n], C[:, n:]
    sol = nsk.tls_solve_exact(dev(A), dev(B), allow_marginal=True)
    _, Vr, svr, _, _ = oracle.tls_solve_exact(A, B, allow_marginal=True)
    assert np.max(np.abs(host(sol.augmented_singular_values) - svr)) <= 1e-12 * svr[0]
    assert oracle.sin_theta(host(sol.Vk), Vr) < 1e-6


def test_tls_exact_validation_and_metrics(nsk, oracle):
    m, n, k = 400, 10, 1
    A, B, X = _tls_problem(oracle, m, n, k, 1e-4, 61)
    with pytest.raises(ValueError):
        nsk.tls_solve_exact(dev(A[:, :0]), dev(B))
    with pytest.raises(ValueError):
        nsk.tls_solve_exact(dev(A[: n, :]), dev(B[: n, :]))  # m < n + k
    Adef = A.copy()
    Adef[:, -1] = 0.0
    with pytest.raises(nsk.TlsExistenceError):
        nsk.tls_solve_exact(dev(Adef), dev(B))
    ex = nsk.tls_solve_exact(dev(A), dev(B))
    sk = nsk.tls_solve_sketched(dev(A), dev(B), nsk.SketchOperator.draw("gaussian", 8 * (n + k), m, 62))
    met = nsk.tls_error_metrics(ex, sk)
    assert 0 <= met.rel_err < 1e-2 and 0 <= met.sin_X <= 1 and 0 <= met.sin_Vk < 1e-2
    same = nsk.tls_error_metrics(ex, ex)
    assert same.rel_err == 0.0 and same.sin_X < 1e-12 and same.sin_Vk < 1e-12
