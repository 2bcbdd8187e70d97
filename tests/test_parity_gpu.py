"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Bars (stated per test): integer draws bit-exact; SA within 1e-12 relative
Frobenius of the oracle; trailing subspaces within a principal-angle bound
(complement projection, kernels.cpp:121-128); ||AW||_F within
1e-10 * max(||AW_ref||_F, 1e3 u ||A||_F).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SA_TOL = 1e-12
U = 2.220446049250313e-16


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


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def gpu_apply(nsk, kind, s, m, seed, A):
    S = nsk.SketchOperator.draw(kind, s, m, seed)
    return host(nsk.apply(S, dev(A)).data), S


# ----------------------------------------------------------------------------- apply parity

@pytest.mark.parametrize("s,m,n,seed", [(80, 2000, 20, 9000001), (400, 20000, 100, 9000001), (7, 333, 5, 3),
                                        (64, 4096, 300, 17), (1, 50, 3, 2), (33, 1000, 129, 4)])
def test_gaussian_apply_parity(nsk, oracle, s, m, n, seed):
    A = oracle.random_real(m, n, seed + 1)
    got, S = gpu_apply(nsk, "gaussian", s, m, seed, A)
    ref = oracle.apply(oracle.draw("gaussian", s, m, seed), A)
    assert rel(got, ref) <= SA_TOL


def test_gaussian_complex_apply_parity(nsk, oracle):
    A = oracle.random_complex(999, 13, 5)
    got, _ = gpu_apply(nsk, "gaussian", 50, 999, 77, A)
    ref = oracle.apply(oracle.draw("gaussian", 50, 999, 77), A)
    assert got.dtype == np.complex128
    assert rel(got, ref) <= SA_TOL


def test_gaussian_identity_known_answer(nsk, golden):
    # test_sketch.cpp:103-114: apply(S, I_4) == G/2 (1e-15 there; CUDA libm log/sincospi are
    # within 2 ulp of glibc, so the bound here is 4 ulp of the largest entry).
    G = golden["draws"]["G_4_4_42"]
    got, _ = gpu_apply(nsk, "gaussian", 4, 4, 42, np.eye(4))
    assert np.max(np.abs(got - G / 2.0)) <= 4 * U * np.max(np.abs(G))


@pytest.mark.parametrize("kind,s,m,n", [("srdct", 40, 2000, 20), ("srdct", 60, 60, 11), ("srdct", 17, 1000, 3),
                                        ("srdct", 256, 1 << 14, 64), ("srft", 64, 1000, 7), ("srft", 60, 60, 11),
                                        ("srft", 128, 1 << 13, 33)])
def test_srtt_apply_parity(nsk, oracle, kind, s, m, n):
    A = oracle.random_real(m, n, 11)
    got, _ = gpu_apply(nsk, kind, s, m, 21, A)
    ref = oracle.apply(oracle.draw(kind, s, m, 21), A)
    assert rel(got, ref) <= SA_TOL


@pytest.mark.parametrize("kind,s,m,n,cplx", [("srdct", 1024, 1 << 16, 8, False), ("srft", 1000, 1 << 15, 5, True),
                                             ("srft", 512, 3 << 12, 6, False), ("srdct", 300, 5 << 12, 4, False)])
def test_srtt_fast_path_parity(nsk, oracle, kind, s, m, n, cplx):
    """Blocked FFT path (m % 4096 == 0): sampled DFT / Makhoul DCT-III against scipy/numpy."""
    A = oracle.random_complex(m, n, 3) if cplx else oracle.random_real(m, n, 3)
    got, _ = gpu_apply(nsk, kind, s, m, 77, A)
    ref = oracle.apply(oracle.draw(kind, s, m, 77), A)
    assert rel(got, ref) <= SA_TOL


@pytest.mark.parametrize("s,m,n", [(256, 1 << 14, 5), (1000, 1 << 15, 3), (300, 3 << 14, 4), (2048, 1 << 18, 2),
                                   (1500, 1 << 16, 9), (1024, 1 << 17, 150), (4096, 1 << 14, 3), (1, 1 << 14, 1),
                                   (1 << 14, 1 << 14, 2), (7, 5 << 14, 149)])
def test_srdct_makhoul_parity(nsk, oracle, monkeypatch, s, m, n):
    """Register-streamed Makhoul tiles (srdct_stream.cu, the default for m % 16384 == 0) against
    scipy's DCT-III, and against the shared-memory tile path (srtt_tile.cu) and the strided FFT
    (srtt_fast.cu) on the same operator."""
    A = oracle.random_real(m, n, 13)
    got, _ = gpu_apply(nsk, "srdct", s, m, 91, A)
    ref = oracle.apply(oracle.draw("srdct", s, m, 91), A)
    assert rel(got, ref) <= SA_TOL
    for env in ("NSK_SRDCT_NOSTREAM", "NSK_SRTT_NOTILE"):  # cumulative: shared-memory tiles, then strided FFT
        monkeypatch.setenv(env, "1")
        other, _ = gpu_apply(nsk, "srdct", s, m, 91, A)
        assert rel(got, other) <= SA_TOL, env


@pytest.mark.parametrize("s,m,n", [(256, 1 << 14, 5), (1000, 1 << 15, 3), (300, 3 << 14, 4), (2048, 1 << 18, 2),
                                   (1500, 1 << 16, 9), (1024, 1 << 17, 150), (1, 1 << 14, 1), (1 << 14, 1 << 14, 2),
                                   (7, 5 << 14, 149)])
def test_srft_stream_parity(nsk, oracle, monkeypatch, s, m, n):
    """Warp-specialised srft tiles (srft_ws.cu, the default for real A with m % 16384 == 0)
    against numpy's inverse FFT, and against the shared-memory tile path (srtt_tile.cu) and the
    strided FFT (srtt_fast.cu) on the same operator."""
    A = oracle.random_real(m, n, 17)
    got, _ = gpu_apply(nsk, "srft", s, m, 93, A)
    ref = oracle.apply(oracle.draw("srft", s, m, 93), A)
    assert rel(got, ref) <= SA_TOL
    for env in ("NSK_SRFT_WS", "NSK_SRTT_NOTILE"):  # cumulative: shared-memory tiles, then strided FFT
        monkeypatch.setenv(env, "0" if env == "NSK_SRFT_WS" else "1")
        other, _ = gpu_apply(nsk, "srft", s, m, 93, A)
        assert rel(got, other) <= SA_TOL, env


def test_srft_complex_parity(nsk, oracle, golden):
    sa = golden["sa"]
    A = sa["A_srft"]
    got, _ = gpu_apply(nsk, "srft", 24, 300, 9000004, A)
    assert rel(got, sa["SA_srft"]) <= SA_TOL


@pytest.mark.parametrize("s,m,n", [(40, 2048, 20), (1024, 1 << 14, 8), (100, 1 << 12, 33), (16, 256, 5),
                                   (1000, 1 << 16, 3), (2048, 1 << 13, 4)])
def test_srht_apply_parity(nsk, oracle, s, m, n):
    A = oracle.random_real(m, n, 5)
    got, _ = gpu_apply(nsk, "srht", s, m, 9000002, A)
    ref = oracle.apply(oracle.draw("srht", s, m, 9000002), A)
    assert rel(got, ref) <= SA_TOL


@pytest.mark.parametrize("s,m,n", [(1024, 1 << 15, 7), (300, 1 << 13, 40), (2500, 1 << 16, 3)])
def test_srht_block_kernels_parity(nsk, oracle, monkeypatch, s, m, n):
    """Every SRHT block kernel against the oracle: 2048-row blocks by 16-byte loads (srht_kernel16, the
    default for 16-byte-aligned A with an even leading dimension), the 8-byte 2048-row kernel (reached by
    an odd leading dimension, by a base address that is 8 mod 16, and by NSK_SRHT_V16=0) and 1024-row
    blocks (NSK_SRHT_LB=10)."""
    import torch
    A = oracle.random_real(m, n, 21)
    ref = oracle.apply(oracle.draw("srht", s, m, 9000002), A)
    S = nsk.SketchOperator.draw("srht", s, m, 9000002)
    assert rel(host(nsk.apply(S, dev(A)).data), ref) <= SA_TOL
    buf = torch.zeros((n, m + 1), dtype=torch.float64, device="cuda").t()  # ld m + 1 (odd)
    buf[:m].copy_(torch.from_numpy(A))
    assert rel(host(nsk.apply(S, buf[:m]).data), ref) <= SA_TOL, "odd leading dimension"
    buf = torch.zeros((n, m + 2), dtype=torch.float64, device="cuda").t()  # ld m + 2, base 8 mod 16
    buf[1:m + 1].copy_(torch.from_numpy(A))
    assert rel(host(nsk.apply(S, buf[1:m + 1]).data), ref) <= SA_TOL, "base address 8 mod 16"
    monkeypatch.setenv("NSK_SRHT_V16", "0")
    assert rel(host(nsk.apply(S, dev(A)).data), ref) <= SA_TOL, "NSK_SRHT_V16=0"
    monkeypatch.setenv("NSK_SRHT_LB", "10")
    assert rel(host(nsk.apply(S, dev(A)).data), ref) <= SA_TOL, "NSK_SRHT_LB=10"


@pytest.mark.parametrize("s,m,n", [(400, 2000, 20), (4096, 100000, 8), (1024, 50000, 3), (64, 1000, 17),
                                   (30000, 70000, 2)])
def test_countsketch_apply_parity(nsk, oracle, s, m, n):
    A = oracle.random_real(m, n, 6)
    got, _ = gpu_apply(nsk, "countsketch", s, m, 9000003, A)
    ref = oracle.apply(oracle.draw("countsketch", s, m, 9000003), A)
    assert rel(got, ref) <= SA_TOL


@pytest.mark.parametrize("kind", ["gaussian", "srdct", "srht", "countsketch"])
def test_golden_fixture_sa(nsk, golden, kind):
    sa = golden["sa"]
    m = 2048 if kind == "srht" else 2000
    s = {"gaussian": 80, "srdct": 40, "srht": 40, "countsketch": 400}[kind]
    got, _ = gpu_apply(nsk, kind, s, m, 9000001, sa[f"A_{m}_20"])
    assert rel(got, sa[f"SA_{kind}"]) <= SA_TOL


@pytest.mark.parametrize("kind", ["gaussian", "srft", "srdct", "srht", "countsketch"])
def test_apply_bit_identical_reruns(nsk, oracle, kind):
    m = 4096
    A = dev(oracle.random_real(m, 40, 9))
    S = nsk.SketchOperator.draw(kind, 128, m, 5)
    a = host(nsk.apply(S, A).data)
    b = host(nsk.apply(S, A).data)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["gaussian", "srft", "srdct", "srht", "countsketch"])
def test_apply_is_linear(nsk, oracle, kind):
    # test_sketch.cpp:140-163: 1e-13 relative
    m = 2048
    a = oracle.random_real(m, 6, 13)
    b = oracle.random_real(m, 6, 14)
    S = nsk.SketchOperator.draw(kind, 64, m, 21)
    lhs = host(nsk.apply(S, dev(2 * a - 3 * b)).data)
    rhs = 2 * host(nsk.apply(S, dev(a)).data) - 3 * host(nsk.apply(S, dev(b)).data)
    assert np.max(np.abs(lhs - rhs)) < 1e-13 * np.linalg.norm(lhs)


@pytest.mark.parametrize("kind", ["srft", "srdct"])
def test_full_sampling_is_unitary(nsk, oracle, kind):
    # test_sketch.cpp:116-131: s = m preserves singular values to 1e-12 sigma_1
    m, n = 60, 11
    A = oracle.random_real(m, n, 5)
    got, _ = gpu_apply(nsk, kind, m, m, 7, A)
    sv, ref = np.linalg.svd(got, compute_uv=False), np.linalg.svd(A, compute_uv=False)
    assert np.max(np.abs(sv - ref)) < 1e-12 * ref[0]


def test_srht_full_sampling_is_unitary(nsk, oracle):
    m, n = 1 << 12, 9
    A = oracle.random_real(m, n, 5)
    got, _ = gpu_apply(nsk, "srht", m, m, 7, A)
    sv, ref = np.linalg.svd(got, compute_uv=False), np.linalg.svd(A, compute_uv=False)
    assert np.max(np.abs(sv - ref)) < 1e-12 * ref[0]


def test_zero_input_gives_zero(nsk):
    import torch
    S = nsk.SketchOperator.draw("srft", 8, 32, 3)
    Z = torch.zeros(32, 5, dtype=torch.complex128, device="cuda")
    assert torch.linalg.norm(nsk.apply(S, Z).data).item() == 0.0


def test_apply_validation(nsk, oracle):
    import torch
    S = nsk.SketchOperator.draw("srft", 8, 32, 3)
    with pytest.raises(ValueError):
        nsk.apply(S, torch.zeros(31, 5, dtype=torch.complex128, device="cuda"))
    D = nsk.SketchOperator.draw("srdct", 8, 32, 3)
    with pytest.raises(ValueError):
        nsk.apply(D, torch.zeros(32, 5, dtype=torch.complex128, device="cuda"))
    H = nsk.SketchOperator.draw("srht", 8, 32, 3)
    with pytest.raises(ValueError):
        nsk.apply(H, torch.zeros(32, 5, dtype=torch.complex128, device="cuda"))


def test_non_colmajor_and_ld_inputs(nsk, oracle):
    import torch
    m, n = 3000, 12
    A = oracle.random_real(m, n, 3)
    S = nsk.SketchOperator.draw("gaussian", 50, m, 4)
    ref = host(nsk.apply(S, dev(A)).data)
    rowmajor = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    assert np.array_equal(host(nsk.apply(S, rowmajor).data), ref)
    big = torch.zeros((n, m + 5), dtype=torch.float64, device="cuda")
    big[:, :m] = torch.from_numpy(A.T.copy()).cuda()
    view = big.t()[:m]  # column-major with lda = m + 5
    assert view.stride() == (1, m + 5)
    assert rel(host(nsk.apply(S, view).data), ref) <= 1e-15


@pytest.mark.parametrize("pad,off", [(16, 0), (5, 0), (16, 1)])
@pytest.mark.parametrize("kind", ["srft", "srdct", "srht", "countsketch", "gaussian"])
def test_padded_leading_dimension_tile_kernels(nsk, oracle, kind, pad, off):
    """lda = m + pad at m = 2^14 with the matrix starting `off` elements into the buffer: the
    tile kernels (even lda, 16-byte aligned A) and their fallbacks (odd lda, 8-byte aligned A),
    against the oracle on the unpadded matrix."""
    import torch
    m, n, s = 1 << 14, 7, 256
    A = oracle.random_real(m, n, 21)
    big = torch.zeros((n, m + pad + off), dtype=torch.float64, device="cuda")
    big[:, off:off + m] = torch.from_numpy(A.T.copy()).cuda()
    view = big.t()[off:off + m]
    assert view.stride() == (1, m + pad + off)
    S = nsk.SketchOperator.draw(kind, s, m, 9000011)
    got = host(nsk.apply(S, view).data)
    ref = oracle.apply(oracle.draw(kind, s, m, 9000011), A)
    assert rel(got, ref) <= SA_TOL


def test_host_entry_point_matches_device(nsk, oracle):
    m, n = 2000, 10
    A = oracle.random_real(m, n, 8)
    for kind in ("gaussian", "srdct", "srht", "countsketch", "srft"):
        mm = 2048 if kind == "srht" else m
        Ak = oracle.random_real(mm, n, 8)
        S = nsk.SketchOperator.draw(kind, 40, mm, 4)
        assert np.array_equal(nsk.apply(S, Ak).data, host(nsk.apply(S, dev(Ak)).data))


# ----------------------------------------------------------------------------- shards

@pytest.mark.parametrize("kind,m,splits", [("gaussian", 4000, [0, 1000, 2500, 4000]),
                                           ("srht", 1 << 14, [0, 4096, 8192, 16384]),
                                           ("countsketch", 1 << 14, [0, 2048, 10240, 16384])])
def test_row_shards_sum_to_apply(nsk, oracle, kind, m, splits):
    import torch
    A = oracle.random_real(m, 9, 3)
    S = nsk.SketchOperator.draw(kind, 100, m, 31)
    full = host(nsk.apply(S, dev(A)).data)
    acc = torch.zeros(100, 9, dtype=torch.float64, device="cuda")
    for a, b in zip(splits[:-1], splits[1:]):
        acc += nsk.apply_shard(S, dev(A[a:b]), a)
    assert rel(host(acc), full) <= 1e-13


@pytest.mark.parametrize("kind", ["srdct", "srft"])
def test_cyclic_shards_sum_to_apply(nsk, oracle, kind):
    import torch
    m, P = 3000, 4
    A = oracle.random_real(m, 7, 3)
    S = nsk.SketchOperator.draw(kind, 64, m, 31)
    full = host(nsk.apply(S, dev(A)).data)
    acc = None
    for g in range(P):
        part = nsk.apply_shard(S, dev(A[g::P]), g, P)
        acc = part if acc is None else acc + part
    assert rel(host(acc), full) <= 1e-13


# ----------------------------------------------------------------------------- solve

def _angle(W, Wref):
    from oracle import sketch_oracle as O
    return O.sin_theta(W, Wref)


def test_cfg1_solve_k_parity(nsk, oracle):
    """BASELINE configs[0]: m=20000, n=100, gaussian s=4n, sigma_n = 1e-10, k=1."""
    m, n = 20000, 100
    spec = np.concatenate([np.logspace(0, -3, n - 1), [1e-10]])
    A = oracle.make_test_matrix(m, n, spec, seed=1)
    S = nsk.SketchOperator.draw("gaussian", 4 * n, m, 9000001)
    res = nsk.solve_k(dev(A), 1, S)
    W, sig = host(res.W), host(res.sketched_singular_values)
    Wref, sref = oracle.solve_k(A, 1, oracle.draw("gaussian", 4 * n, m, 9000001))
    assert _angle(W, Wref) <= 1e-10
    # LAPACK/BDCSVD sigmas are accurate to O(n u sigma_1) absolutely (the 8.8e-11 trailing value
    # differs by ~2e-17 between the two backends), so the sigma bound is absolute: 1000 u sigma_1.
    assert np.max(np.abs(sig - sref)) <= 1000 * U * sref[0]
    r, rref = np.linalg.norm(A @ W), np.linalg.norm(A @ Wref)
    # 1e-10 relative, floored at the rounding level of evaluating ||A W||_F itself
    # (100 u ||A||_F): at configs[0] the reorder-only gap is ~3e-18.
    assert abs(r - rref) <= max(1e-10 * rref, 100 * U * np.linalg.norm(A))
    assert abs(nsk.residual_certificate(dev(A), res.W) - r) <= max(1e-12 * r, 100 * U * np.linalg.norm(A))
    # the sketched solution is near-optimal (Theorem 3): ||AW|| within factor 4 of sigma_n
    assert r < 4 * spec[-1]


@pytest.mark.parametrize("kind,s", [("srdct", 40), ("srht", 40), ("countsketch", 400), ("gaussian", 80)])
def test_solve_k_golden(nsk, golden, kind, s):
    sa = golden["sa"]
    m = 2048 if kind == "srht" else 2000
    A = sa[f"A_{m}_20"]
    S = nsk.SketchOperator.draw(kind, s, m, 9000001)
    res = nsk.solve_k(A, 1, S)  # host entry point
    assert _angle(res.W, sa[f"W_{kind}"]) <= 1e-10
    sref = sa[f"sigma_{kind}"]
    assert np.max(np.abs(res.sketched_singular_values - sref)) <= 1e-12 * sref[0]


def test_svd_trailing_contract(nsk, oracle):
    for (s, n, k) in [(40, 20, 3), (300, 150, 1), (1024, 256, 4), (64, 64, 5), (9, 1, 0)]:
        X = oracle.random_real(s, n, s + n)
        W, sig = nsk.svd_trailing(dev(X), k)
        W, sig = host(W), host(sig)
        _, sref, vh = np.linalg.svd(X, full_matrices=False)
        assert np.max(np.abs(sig - sref)) <= 1e-12 * sref[0]
        assert np.all(np.diff(sig) <= 0)
        if k:
            assert np.max(np.abs(W.T @ W - np.eye(k))) < 1e-12
            assert _angle(W, vh.T[:, n - k:]) < 1e-10


def test_svd_trailing_complex(nsk, oracle):
    X = oracle.random_complex(300, 150, 2)
    W, sig = nsk.svd_trailing(dev(X), 2)
    W, sig = host(W), host(sig)
    _, sref, vh = np.linalg.svd(X, full_matrices=False)
    assert np.max(np.abs(sig - sref)) <= 1e-12 * sref[0]
    assert _angle(W, vh.conj().T[:, -2:]) < 1e-10


def test_svd_complex_beyond_cluster_steep_spectrum(nsk):
    """Complex n = 400 (> 335: the global-memory block Jacobi, no preconditioning) with sigma
    logspaced 1 -> 1e-14: needs ~45 sweeps, above the former limit of 40."""
    rng = np.random.default_rng(5)
    s, n = 1200, 400
    U, _ = np.linalg.qr(rng.standard_normal((s, n)) + 1j * rng.standard_normal((s, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    sref = np.logspace(0, -14, n)
    X = (U * sref) @ V.conj().T
    W, sig = nsk.svd_trailing(dev(X), 1)
    W, sig = host(W), host(sig)
    assert np.max(np.abs(sig - sref)) <= 1e-12
    assert np.linalg.norm(X @ W) <= 1e-12


def test_exact_null_space_preserved(nsk, oracle):
    # test_nullspace.cpp:21-32
    m, n, k = 200, 20, 2
    spec = np.ones(n)
    spec[-k:] = 0.0
    A = oracle.make_test_matrix(m, n, spec, seed=1)
    S = nsk.SketchOperator.draw("srft", 2 * n, m, 2)
    res = nsk.solve_k(dev(A), k, S)
    assert nsk.residual_certificate(dev(A), res.W) < 1e-10
    exact = np.linalg.svd(A)[2].T[:, n - k:]
    assert _angle(host(res.W), exact) < 1e-10


def test_unitary_sketch_reproduces_exact_subspace(nsk, oracle):
    # test_nullspace.cpp:34-45
    m, n, k = 120, 12, 3
    spec = np.array([1.0 if i < n - k else 1e-2 * 10.0 ** (-(i - (n - k))) for i in range(n)])
    A = oracle.make_test_matrix(m, n, spec, seed=3)
    S = nsk.SketchOperator.draw("srft", m, m, 4)
    res = nsk.solve_k(dev(A), k, S)
    exact = np.linalg.svd(A)[2].T[:, n - k:]
    assert _angle(host(res.W), exact) < 1e-10
    ref = np.linalg.svd(A, compute_uv=False)
    assert np.max(np.abs(host(res.sketched_singular_values) - ref)) < 1e-12 * ref[0]


def test_trailing_residual_identity(nsk, oracle):
    # test_nullspace.cpp:47-57
    m, n, k = 150, 14, 4
    A = oracle.make_test_matrix(m, n, 10.0 ** (-0.5 * np.arange(n)), seed=5)
    S = nsk.SketchOperator.draw("srdct", 2 * n, m, 6)
    res = nsk.solve_k(dev(A), k, S)
    SA = host(nsk.apply(S, dev(A)).data)
    lhs = np.linalg.norm(SA @ host(res.W))
    rhs = math.sqrt(np.sum(host(res.sketched_singular_values)[-k:] ** 2))
    assert abs(lhs - rhs) <= 1e-10 * rhs


def test_solve_tol(nsk, oracle):
    # test_nullspace.cpp:95-135
    m, n = 90, 10
    A = oracle.make_test_matrix(m, n, 10.0 ** (-np.arange(n, dtype=float)), seed=7)
    S = nsk.SketchOperator.draw("srft", m, m, 8)
    assert nsk.solve_tol(dev(A), 3e-9, S).k == 1
    r0 = nsk.solve_tol(dev(A), 1e-12, S)
    assert r0.k == 0 and r0.W.shape == (n, 0)
    spec = np.ones(n)
    spec[-2:] = 0
    B = oracle.make_test_matrix(m, n, spec, seed=9)
    assert nsk.solve_tol(dev(B), 1e-14, S).k == 2
    with pytest.raises(ValueError):
        nsk.solve_tol(dev(A), 2.0, S)
    prev = 0
    for eps in (1e-11, 1e-7, 1e-4, 0.5):
        k = nsk.solve_tol(dev(A), eps, S).k
        assert k >= prev
        prev = k
    with pytest.raises(ValueError):
        nsk.solve_tol(dev(A), -1.0, S)
    kh = nsk.solve_tol(A, 3e-9, S)  # host entry point
    assert kh.k == 1


def test_solve_validation(nsk, oracle):
    # test_nullspace.cpp:160-170
    m, n = 64, 8
    A = dev(oracle.random_real(m, n, 10))
    S = nsk.SketchOperator.draw("srdct", 2 * n, m, 11)
    with pytest.raises(ValueError):
        nsk.solve_k(A, n, S)
    with pytest.raises(ValueError):
        nsk.solve_k(A, -1, S)
    with pytest.raises(ValueError):
        nsk.solve_k(A, 1, nsk.SketchOperator.draw("srdct", 2 * n, m + 1, 12))
    with pytest.raises(ValueError):
        nsk.solve_k(A, 1, nsk.SketchOperator.draw("srdct", n - 2, m, 13))


def test_residual_certificate_known_answer(nsk):
    a = np.zeros((3, 2))
    a[0, 0] = 3.0
    a[1, 1] = 1.0
    w = np.array([[1.0], [0.0]])
    assert abs(nsk.residual_certificate(dev(a), dev(w)) - 3.0) < 1e-15
    with pytest.raises(ValueError):
        nsk.residual_certificate(dev(a), dev(np.eye(3)[:, :1]))


# ----------------------------------------------------------------------------- full size

def test_cfg2_srht_full_size_properties(nsk, oracle):
    """BASELINE configs[1] at full size (m = 2^20, n = 256, s = 1024): linearity,
    bit-identical re-run and a column-sampled oracle check."""
    import torch
    m, n, s = 1 << 20, 256, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
    B = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
    S = nsk.SketchOperator.draw("srht", s, m, 9000002)
    sa = nsk.apply(S, A).data
    sb = nsk.apply(S, B).data
    sab = nsk.apply(S, (2 * A - 3 * B).t().contiguous().t()).data
    assert (torch.linalg.norm(sab - (2 * sa - 3 * sb)) / torch.linalg.norm(sab)).item() < 1e-13
    assert torch.equal(sa, nsk.apply(S, A).data)
    cols = [0, 77, 255]
    Ah = A[:, cols].cpu().numpy()
    ref = oracle.apply(oracle.draw("srht", s, m, 9000002), Ah)
    assert rel(sa[:, cols].cpu().numpy(), ref) <= SA_TOL


@pytest.mark.parametrize("kind", ["srdct", "srft"])
def test_cfg2_srtt_full_size_properties(nsk, oracle, kind):
    """configs[1] shape through the transform sketches: column sample vs scipy/numpy, re-run identity."""
    import torch
    m, n, s = 1 << 20, 64, 1024
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
    S = nsk.SketchOperator.draw(kind, s, m, 9000005)
    sa = nsk.apply(S, A).data
    assert torch.equal(sa, nsk.apply(S, A).data)
    cols = [0, 63]
    ref = oracle.apply(oracle.draw(kind, s, m, 9000005), A[:, cols].cpu().numpy())
    assert rel(sa[:, cols].cpu().numpy(), ref) <= SA_TOL


@pytest.mark.parametrize("kind", ["srdct", "srft"])
def test_srtt_stream_large_m(nsk, oracle, kind):
    """m = 2^24 + 2^14 (P = 16400 tile columns, not a power of two: exact-integer anchors with
    the FP64 quotient, 1025+ tiles per column) through the stream kernels, two columns vs the oracle."""
    import torch
    m, n, s = (1 << 24) + (1 << 14), 3, 1000
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
    S = nsk.SketchOperator.draw(kind, s, m, 9000007)
    sa = nsk.apply(S, A).data
    cols = [0, 2]
    ref = oracle.apply(oracle.draw(kind, s, m, 9000007), A[:, cols].cpu().numpy())
    assert rel(sa[:, cols].cpu().numpy(), ref) <= SA_TOL


def test_cfg5_loewner_complex_gaussian(nsk, oracle):
    """BASELINE configs[4]: complex128 Loewner matrix (m = 99850 active rows, n = 150),
    Gaussian sketch s = 2n on complex data, k = 1 trailing vector."""
    L = oracle.loewner_config5()
    m, n = L.shape
    S = nsk.SketchOperator.draw("gaussian", 2 * n, m, 9000005)
    res = nsk.solve_k(dev(L), 1, S)
    Wref, sref = oracle.solve_k(L, 1, oracle.draw("gaussian", 2 * n, m, 9000005))
    # L is numerically rank-deficient (trailing sigmas ~1e-12 ~ u ||L||): the trailing vector is
    # not unique, so parity is on the residual (rounding level, 100 u ||L||_F) and the sigmas.
    W = host(res.W)
    assert abs(np.linalg.norm(W) - 1.0) < 1e-12
    assert np.linalg.norm(L @ W) <= max(10 * np.linalg.norm(L @ Wref), 100 * U * np.linalg.norm(L))
    assert np.max(np.abs(host(res.sketched_singular_values) - sref)) <= 1000 * U * sref[0]
    SA = host(nsk.apply(S, dev(L)).data)
    assert rel(SA, oracle.apply(oracle.draw("gaussian", 2 * n, m, 9000005), L)) <= SA_TOL


@pytest.mark.parametrize("kind,s", [("gaussian", 64), ("srht", 256), ("countsketch", 4096)])
def test_host_pipelined_sketch(nsk, oracle, kind, s):
    """Host entry points on >= 256 MiB inputs copy A in row chunks and sketch each chunk as it
    lands (capi.cpp host_sketch): SA against the oracle, the unpipelined host path bit-identical
    to the device path, and solve_k through the host API against the oracle's W."""
    import os
    m, n = 1 << 21, 16
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    S = nsk.SketchOperator.draw(kind, s, m, 17)
    got = nsk.apply(S, A).data
    oref = oracle.apply(oracle.draw(kind, s, m, 17), A)
    assert rel(got, oref) <= SA_TOL
    ref = host(nsk.apply(S, dev(A)).data)
    assert rel(ref, oref) <= SA_TOL
    os.environ["NSK_NO_PIPELINE"] = "1"
    try:
        plain = nsk.apply(S, A).data
    finally:
        del os.environ["NSK_NO_PIPELINE"]
    assert np.array_equal(plain, ref)
    r_host = nsk.solve_k(A, 1, S)
    Wref, sref = oracle.from_sketch_svd(oref, 1)
    assert np.max(np.abs(np.asarray(r_host.sketched_singular_values) - sref)) <= 1000 * U * sref[0]
    assert _angle(np.asarray(r_host.W), Wref) <= 1e-10


@pytest.mark.parametrize("kind,s,m,n", [("srht", 512, 1 << 21, 40), ("countsketch", 2048, 1 << 21, 33),
                                        ("srdct", 256, 1 << 20, 9), ("srft", 128, 3 << 18, 5)])
def test_host_pageable_staging(nsk, oracle, kind, s, m, n):
    """Pageable host A (the reference callers' Eigen buffers) streams through the library's pinned
    staging ring (h2d.cpp): several slot-sized tiles per row chunk, a partial last tile, and the
    unpipelined copy (srdct/srft); SA against the oracle, and pinned input gives the same bytes."""
    import torch
    rng = np.random.default_rng(9)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    S = nsk.SketchOperator.draw(kind, s, m, 23)
    got = nsk.apply(S, A).data
    assert rel(got, oracle.apply(oracle.draw(kind, s, m, 23), A)) <= SA_TOL
    pinned = torch.empty((n, m), dtype=torch.float64, pin_memory=True).t()
    pinned.copy_(torch.from_numpy(A))
    out = np.empty_like(got, order="F")
    from paper_2206_00975_b200 import _lib
    import ctypes
    _lib.check(_lib.load().nsk_apply_host(S.handle, 0, m, n, ctypes.c_void_p(pinned.data_ptr()), m,
                                          out.ctypes.data_as(ctypes.c_void_p), s))
    assert np.array_equal(out, got)


# ----------------------------------------------------------------------------- general m and cyclic shards

@pytest.mark.parametrize("kind,m,s,n,cplx", [("srft", 20000, 400, 7, False), ("srdct", 20000, 400, 7, False),
                                             ("srft", 100000, 300, 5, True), ("srdct", 100000, 300, 5, False),
                                             ("srft", 99850, 300, 4, True), ("srdct", 99850, 300, 4, False),
                                             ("srft", 1009, 64, 3, False), ("srdct", 1009, 64, 3, False),
                                             ("srdct", 840, 840, 2, False), ("srft", 3 * 7 * 5 * 64, 2500, 3, False),
                                             ("srft", 1000000, 1000, 2, False), ("srdct", 1000000, 1000, 2, False)])
def test_srtt_general_length(nsk, oracle, kind, m, s, n, cplx):
    """Exact-length transforms at m not a multiple of 4096 (FFTW transforms any m with no padding,
    transforms.cpp:17-64, sketch.hpp:34-35): the mixed-radix engine (srtt_general.cu) against
    numpy/scipy at 1e-12 -- m = 20000, 100000 and 10^6 (the reference's AAA default, aaa.cpp:254-258),
    99850 = 2 5^2 1997 (the Loewner row count), the prime 1009, s > 2048 (two slot chunks)."""
    A = oracle.random_complex(m, n, 4) if cplx else oracle.random_real(m, n, 4)
    got, _ = gpu_apply(nsk, kind, s, m, 41, A)
    ref = oracle.apply(oracle.draw(kind, s, m, 41), A)
    assert rel(got, ref) <= SA_TOL


@pytest.mark.parametrize("kind,m,P", [("srft", 1 << 17, 4), ("srdct", 1 << 17, 8), ("srft", 20000, 4),
                                      ("srdct", 20000, 8), ("srdct", 3 << 14, 2), ("srft", 99850, 2)])
def test_cyclic_shard_partials(nsk, oracle, kind, m, P):
    """Multi-GPU srft/srdct rows: rank g holds rows g, g+P, ...; its partial is the
    local length-m/P transform, twiddled and gathered (decimation in time).  Every partial against
    the oracle applied to A with the other ranks' rows zeroed, and their sum against the full apply."""
    import torch
    n, s = 5, 256
    A = oracle.random_real(m, n, 8)
    S = nsk.SketchOperator.draw(kind, s, m, 55)
    op = oracle.draw(kind, s, m, 55)
    acc = None
    for g in range(P):
        part = nsk.apply_shard(S, dev(A[g::P]), g, P)
        Am = np.zeros_like(A)
        Am[g::P] = A[g::P]
        assert rel(host(part), oracle.apply(op, Am)) <= SA_TOL
        acc = part if acc is None else acc + part
    assert rel(host(acc), oracle.apply(op, A)) <= SA_TOL


@pytest.mark.parametrize("splits", [[0, 12288 * 3, 12288 * 7, 100000], [0, 512 * 5, 4096 * 9, 4096 * 9 + 512, 100000]])
def test_countsketch_shard_windows(nsk, oracle, splits):
    """CountSketch shards build tables for their own rows only (a tile-aligned window, operator.cpp
    tables(lo, hi)): each shard's partial against the oracle on A with the other rows zeroed, fresh
    operators per shard order (first use builds the window), and the sum against the full apply."""
    m, n, s = 100000, 6, 2048
    A = oracle.random_real(m, n, 12)
    op = oracle.draw("countsketch", s, m, 77)
    for order in (list(range(len(splits) - 1)), list(reversed(range(len(splits) - 1)))):
        S = nsk.SketchOperator.draw("countsketch", s, m, 77)
        acc = np.zeros((s, n))
        for i in order:
            a, b = splits[i], splits[i + 1]
            part = host(nsk.apply_shard(S, dev(A[a:b]), a))
            Am = np.zeros_like(A)
            Am[a:b] = A[a:b]
            assert rel(part, oracle.apply(op, Am)) <= SA_TOL
            acc += part
        assert rel(acc, oracle.apply(op, A)) <= SA_TOL
        assert rel(host(nsk.apply(S, dev(A)).data), oracle.apply(op, A)) <= SA_TOL


@pytest.mark.parametrize("kind,cyclic", [("srht", False), ("countsketch", False), ("gaussian", False),
                                         ("srdct", True), ("srft", True)])
def test_nccl_entry_points_single_rank(nsk, oracle, kind, cyclic):
    """The multi-GPU C ABI (nsk_apply_allreduce / nsk_solve_k_sharded, nccl_shard.cpp) on a
    one-rank NCCL communicator made by the library (nsk_nccl_unique_id / nsk_nccl_comm_init):
    NCCL is dlopened, the partial is all-reduced in place, the SVD runs; results against the
    oracle.  (One GPU per process: the world-size > 1 reduce is the same call.)"""
    from paper_2206_00975_b200.distributed import NcclComm, RowShard, sharded_apply_nccl, sharded_solve_k_nccl
    m = 1 << 16
    n, s = 8, (4096 if kind == "countsketch" else 64)
    A = oracle.random_real(m, n, 21)
    S = nsk.SketchOperator.draw(kind, s, m, 61)
    comm = NcclComm()
    try:
        shard = RowShard(0, 1, m)
        SA = host(sharded_apply_nccl(S, dev(A), shard, comm))
        ref = oracle.apply(oracle.draw(kind, s, m, 61), A)
        assert rel(SA, ref) <= SA_TOL
        W, sig = sharded_solve_k_nccl(S, dev(A), 2, shard, comm)
        Wref, sref = oracle.from_sketch_svd(ref, 2)
        assert np.max(np.abs(host(sig) - sref)) <= 1000 * U * sref[0]
        assert _angle(host(W), Wref) <= 1e-8
    finally:
        comm.close()


@pytest.mark.parametrize("kind,m,row0,mloc", [("gaussian", 50000, 16000, 20000), ("srht", 1 << 17, 1 << 15, 1 << 15),
                                              ("countsketch", 4 * 12288, 12288, 2 * 12288),
                                              ("gaussian", 1 << 21, 0, 1 << 21)])
def test_nccl_host_shard_single_rank(nsk, oracle, kind, m, row0, mloc):
    """nsk_solve_k_sharded_host on a contiguous shard from host memory (a one-rank communicator, so
    the all-reduce is the identity): the partial sketch S[:, rows] A_rows (the library's host
    pipeline with the shard's global row offset; the 2^21 x 16 case is big enough to stream in row
    chunks) and its SVD against the oracle applied to A zero outside the shard."""
    from paper_2206_00975_b200.distributed import NcclComm, RowShard, sharded_solve_k_host_nccl
    n = 16 if m == 1 << 21 else 8
    s = 4096 if kind == "countsketch" else 64
    A_loc = oracle.random_real(mloc, n, 23)
    A_full = np.zeros((m, n))
    A_full[row0:row0 + mloc] = A_loc
    S = nsk.SketchOperator.draw(kind, s, m, 62)
    comm = NcclComm()
    try:
        W, sig = sharded_solve_k_host_nccl(S, A_loc, 2, RowShard(row0, 1, mloc), comm)
        ref = oracle.apply(oracle.draw(kind, s, m, 62), A_full)
        Wref, sref = oracle.from_sketch_svd(ref, 2)
        assert np.max(np.abs(sig - sref)) <= 1000 * U * sref[0]
        assert _angle(W, Wref) <= 1e-8
    finally:
        comm.close()


def test_tls_complex_many_rhs_and_release(nsk, oracle):
    """Complex sketched TLS with k = 60 right-hand sides (the corner solve needs 57.6 KiB of
    dynamic shared memory, above the 48 KiB default) against the oracle, k = 65 rejected before
    any work, and nsk_release_scratch trims the library's private pool."""
    from paper_2206_00975_b200 import _lib
    rng = np.random.default_rng(3)
    m, n, k, s = 600, 64, 60, 300
    A = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    X0 = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    B = A @ X0 + 1e-6 * (rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)))
    S = nsk.SketchOperator.draw("gaussian", s, m, 5)
    sol = nsk.tls_solve_sketched(dev(A), dev(B), S, allow_marginal=True)
    Xr, Vr, sr, _, _ = oracle.tls_solve_sketched(A, B, oracle.draw("gaussian", s, m, 5), allow_marginal=True)
    assert np.max(np.abs(host(sol.augmented_singular_values) - sr)) <= 1000 * U * sr[0]
    assert rel(host(sol.X), Xr) <= 1e-8
    with pytest.raises(ValueError):
        nsk.tls_solve_sketched(dev(np.hstack([A, A[:, :1]])), dev(np.hstack([B, B[:, :5]])), S)
    _lib.check(_lib.load().nsk_release_scratch())
    # the host-buffer path reallocates what the release freed (pageable input > 4 MiB: staging ring)
    A2 = np.asfortranarray(rng.standard_normal((1 << 16, 12)))
    S2 = nsk.SketchOperator.draw("srht", 64, 1 << 16, 3)
    assert rel(np.asarray(nsk.apply(S2, A2).data), oracle.apply(oracle.draw("srht", 64, 1 << 16, 3), A2)) <= SA_TOL


@pytest.mark.parametrize("k", [2, 7, 24])
def test_tls_multi_rhs_real(nsk, oracle, k):
    """X = -V_k1 V_k2^{-1} for several right-hand sides (the corner LU needs its row interchanges
    applied before the forward substitution) against the oracle (tls.cpp:26-43)."""
    rng = np.random.default_rng(k)
    m, n, s = 500, 40, 200
    A = rng.standard_normal((m, n))
    B = A @ rng.standard_normal((n, k)) + 1e-5 * rng.standard_normal((m, k))
    S = nsk.SketchOperator.draw("srdct", s, m, 12)
    sol = nsk.tls_solve_sketched(dev(A), dev(B), S, allow_marginal=True)
    Xr, Vr, sr, _, _ = oracle.tls_solve_sketched(A, B, oracle.draw("srdct", s, m, 12), allow_marginal=True)
    assert _angle(host(sol.Vk), Vr) <= 1e-10
    assert rel(host(sol.X), Xr) <= 1e-10


@pytest.mark.parametrize("kind,s,m,n,pinned", [("srht", 256, 1 << 20, 33, False), ("gaussian", 96, 300000, 40, False),
                                               ("countsketch", 2048, 600000, 17, True), ("srdct", 128, 1 << 18, 9, False),
                                               ("srft", 64, 20000, 3, True)])
def test_host_strided_input(nsk, oracle, kind, s, m, n, pinned):
    """Host A with a leading dimension larger than m (a block of a bigger Eigen matrix): the staged and
    pinned copies honour lda, pipelined (>= 256 MiB) or not, against the oracle on the same rows."""
    import ctypes
    import torch
    from paper_2206_00975_b200 import _lib
    lda = m + 37
    rng = np.random.default_rng(m % 1000)
    big = rng.standard_normal((lda, n))
    if pinned:
        buf = torch.empty((n, lda), dtype=torch.float64, pin_memory=True).t()
        buf.copy_(torch.from_numpy(big))
        ptr = buf.data_ptr()
    else:
        big = np.asfortranarray(big)
        ptr = big.ctypes.data
    A = np.asfortranarray(big[:m])
    S = nsk.SketchOperator.draw(kind, s, m, 71)
    cplx_out = kind == "srft"
    SA = np.empty((s, n), dtype=np.complex128 if cplx_out else np.float64, order="F")
    _lib.check(_lib.load().nsk_apply_host(S.handle, 0, m, n, ctypes.c_void_p(ptr), lda,
                                          SA.ctypes.data_as(ctypes.c_void_p), s))
    assert rel(SA, oracle.apply(oracle.draw(kind, s, m, 71), A)) <= SA_TOL


def test_nccl_empty_shard(nsk, oracle):
    """A rank with no rows contributes zeros (nsk_apply_allreduce with mloc = 0)."""
    from paper_2206_00975_b200.distributed import NcclComm, RowShard, sharded_apply_nccl
    import torch
    S = nsk.SketchOperator.draw("gaussian", 32, 1000, 3)
    comm = NcclComm()
    try:
        A = torch.empty((0, 4), dtype=torch.float64, device="cuda")
        SA = host(sharded_apply_nccl(S, A, RowShard(500, 1, 0), comm))
        assert np.array_equal(SA, np.zeros((32, 4)))
    finally:
        comm.close()


def test_host_staging_complex_and_tls_pipeline(nsk, oracle):
    """Complex pageable input through the staging ring (16-byte entries, chunk-major device copy), and
    sketched TLS from pageable host buffers large enough for the chunked pipeline with the B block
    copied first (capi.cpp host_sketch with kb > 0) against the device-buffer TLS on the same data."""
    import ctypes
    import torch
    from paper_2206_00975_b200 import _lib
    rng = np.random.default_rng(21)
    m, n = 300000, 6
    A = np.asfortranarray(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    S = nsk.SketchOperator.draw("gaussian", 48, m, 5)
    got = np.asarray(nsk.apply(S, A).data)
    assert rel(got, oracle.apply(oracle.draw("gaussian", 48, m, 5), A)) <= SA_TOL
    # TLS: [A | b] 2^21 x 32 real = 512 MiB -> pipelined host path
    m2, n2 = 1 << 21, 31
    A2 = np.asfortranarray(rng.standard_normal((m2, n2)))
    b2 = np.asfortranarray(A2 @ rng.standard_normal((n2, 1)) + 1e-4 * rng.standard_normal((m2, 1)))
    for kind, s in (("gaussian", 64), ("srht", 128), ("countsketch", 1024)):
        S2 = nsk.SketchOperator.draw(kind, s, m2, 8)
        L = _lib.load()
        X = np.empty((n2, 1), order="F")
        Vk = np.empty((n2 + 1, 1), order="F")
        sg = np.empty(n2 + 1)
        info = np.zeros(4)
        _lib.check(L.nsk_tls_solve_sketched_host(S2.handle, 0, m2, n2, 1, A2.ctypes.data_as(ctypes.c_void_p), m2,
                                                 b2.ctypes.data_as(ctypes.c_void_p), m2, 1e12, 1,
                                                 X.ctypes.data_as(ctypes.c_void_p), n2,
                                                 Vk.ctypes.data_as(ctypes.c_void_p), n2 + 1,
                                                 sg.ctypes.data_as(ctypes.c_void_p),
                                                 info.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        ref = nsk.tls_solve_sketched(dev(A2), dev(b2), S2, allow_marginal=True)
        assert np.max(np.abs(sg - host(ref.augmented_singular_values))) <= 1e-12 * sg[0], kind
        assert rel(X, host(ref.X)) <= 1e-10, kind
