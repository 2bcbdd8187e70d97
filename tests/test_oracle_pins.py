"""Pin the CPU oracle before trusting it (CPU only).

* Philox4x32-10 known answer (Random123 KAT, key 0 / counter 0).
* Every draw of the restatement equals the reference's own rng.hpp output,
  recorded by tests/golden/make_golden.py (and, where the reference tree is
  present, re-derived live from oracle/_ref).
* Transform conventions: the oracle's srdct / srft equal the reference's
  closed-form entries (transforms.cpp:66-80) and the dense definitions of
  test_transforms.cpp:13-38.
"""
import math

import numpy as np
import pytest


def test_philox_known_answer(oracle):
    import ctypes
    out = (ctypes.c_uint32 * 4)()
    key = (ctypes.c_uint32 * 2)(0, 0)
    oracle.lib().nsko_philox.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint64,
                                         ctypes.POINTER(ctypes.c_uint32)]
    oracle.lib().nsko_philox(key, 0, out)
    assert [hex(x) for x in out] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]


@pytest.mark.parametrize("seed,stream", [(0, 0), (42, 0), (42, 1), (9000001, 0), (2**64 - 1, 77), (123456789, 2)])
def test_words_gaussians_match_reference(oracle, golden, seed, stream):
    d = golden["draws"]
    assert np.array_equal(oracle.words(seed, stream, 0, 64), d[f"words_{seed}_{stream}"])
    assert np.array_equal(oracle.gaussians(seed, stream, 0, 64), d[f"gauss_{seed}_{stream}"])


@pytest.mark.parametrize("s,m,seed", [(4, 4, 42), (6, 16, 123), (7, 9, 5)])
def test_gaussian_operator_matrix(oracle, golden, s, m, seed):
    G = golden["draws"][f"G_{s}_{m}_{seed}"]
    assert np.array_equal(oracle.gaussian_block(seed, s, 0, m, nthreads=2), G)


def test_gaussian_identity_known_answer(oracle, golden):
    # test_sketch.cpp:103-114: apply(S, I_4) == G / 2 within 1e-15.
    G = golden["draws"]["G_4_4_42"]
    op = oracle.draw("gaussian", 4, 4, 42)
    assert np.max(np.abs(oracle.apply(op, np.eye(4)) - G / 2.0)) < 1e-15


@pytest.mark.parametrize("m,s,seed", [(16, 6, 123), (1000, 64, 7), (1 << 20, 1024, 9000002),
                                      (1000003, 512, 9000077), (20000, 400, 11), (60, 60, 7)])
def test_srtt_draw_matches_reference(oracle, golden, m, s, seed):
    d = golden["draws"]
    op = oracle.draw("srdct", s, m, seed)
    assert np.array_equal(op.idx, d[f"idx_{m}_{s}_{seed}"])
    assert np.array_equal(np.packbits((op.signs > 0).astype(np.uint8)), d[f"signbits_{m}_{s}_{seed}"])


@pytest.mark.parametrize("m,s,seed", [(1000, 64, 3), (1 << 16, 4096, 9000003)])
def test_countsketch_draw_matches_reference(oracle, golden, m, s, seed):
    d = golden["draws"]
    b, g = oracle.countsketch_draw(seed, m, s)
    assert np.array_equal(b, d[f"csbucket_{m}_{s}_{seed}"])
    assert np.array_equal(np.packbits((g > 0).astype(np.uint8)), d[f"cssignbits_{m}_{s}_{seed}"])


def test_update_stream_gaussians(oracle, golden):
    ug = golden["draws"]["update_gauss_45_10_3"]
    assert np.array_equal(oracle.gaussians(45, 1, 0, 30).reshape(3, 10).T, ug)


def test_live_reference_if_present(oracle):
    R = oracle.ref_lib()
    if R is None:
        pytest.skip("reference tree not present (GPU box): fixtures above carry the pin")
    w = np.empty(4096, np.uint32)
    R.nskref_words(777, 3, 4096, w.ctypes.data_as(oracle._u32p))
    assert np.array_equal(w, oracle.words(777, 3, 0, 4096))
    g = np.empty(4096)
    R.nskref_gaussians(777, 3, 4096, g.ctypes.data_as(oracle._dp))
    assert np.array_equal(g, oracle.gaussians(777, 3, 0, 4096))


def _dense_dct3(m):
    # test_transforms.cpp:26-37
    a = np.arange(m)[:, None]
    j = np.arange(m)[None, :]
    c = np.where(j == 0, math.sqrt(1.0 / m), math.sqrt(2.0 / m))
    return c * np.cos(np.pi * j * (2 * a + 1) / (2 * m))


def _dense_idft(m):
    a = np.arange(m)[:, None]
    b = np.arange(m)[None, :]
    return np.exp(2j * np.pi * (a * b % m) / m) / math.sqrt(m)


@pytest.mark.parametrize("m", [1, 2, 7, 12, 16, 100])
def test_transform_conventions(oracle, m):
    # test_transforms.cpp:86-141 tolerances: 1e-12 * ||x||
    import scipy.fft
    x = oracle.random_real(m, 3, 600 + m)
    y = scipy.fft.dct(x, type=3, norm="ortho", axis=0)
    assert np.max(np.abs(y - _dense_dct3(m) @ x)) <= 1e-12 * np.linalg.norm(x)
    z = oracle.random_complex(m, 3, 500 + m)
    w = np.fft.ifft(z, axis=0, norm="ortho")
    assert np.max(np.abs(w - _dense_idft(m) @ z)) <= 1e-12 * np.linalg.norm(z)


@pytest.mark.parametrize("kind", ["srft", "srdct"])
def test_oracle_apply_equals_dense_operator(oracle, kind):
    m, s, n = 48, 16, 5
    op = oracle.draw(kind, s, m, 21)
    A = oracle.random_real(m, n, 13)
    T = _dense_idft(m) if kind == "srft" else _dense_dct3(m)
    dense = math.sqrt(m / s) * (T[op.idx] * op.signs[None, :])
    assert np.max(np.abs(oracle.apply(op, A) - dense @ A)) < 1e-13 * np.linalg.norm(A)


def test_srht_oracle_equals_dense():
    from oracle import sketch_oracle as O
    m, s, n = 64, 16, 3
    op = O.draw("srht", s, m, 5)
    A = O.random_real(m, n, 3)
    H = np.array([[(-1) ** bin(r & j).count("1") for j in range(m)] for r in range(m)]) / math.sqrt(m)
    dense = math.sqrt(m / s) * (H[op.idx] * op.signs[None, :])
    assert np.max(np.abs(O.apply(op, A) - dense @ A)) < 1e-13


def test_countsketch_oracle_equals_dense():
    from oracle import sketch_oracle as O
    m, s, n = 500, 32, 4
    op = O.draw("countsketch", s, m, 8)
    D = np.zeros((s, m))
    D[op.bucket, np.arange(m)] = op.signs
    A = O.random_real(m, n, 4)
    assert np.max(np.abs(O.apply(op, A) - D @ A)) < 1e-13


def test_golden_sa_reproduces(oracle, golden):
    sa = golden["sa"]
    A = sa["A_2000_20"]
    op = oracle.draw("gaussian", 80, 2000, 9000001)
    assert np.array_equal(oracle.apply(op, A), sa["SA_gaussian"])


def test_angles_complement_projection(oracle):
    # kernels.cpp:121-128: tiny angles stay accurate (test_kernels.cpp:180-189)
    n = 6
    U = np.linalg.qr(oracle.random_real(n, 1, 3))[0]
    e = np.zeros((n, 1))
    e[1] = 1e-12
    ep = e - U @ (U.T @ e)
    V = (U + ep) / np.linalg.norm(U + ep)
    expect = np.linalg.norm(ep) / math.sqrt(1 + np.linalg.norm(ep) ** 2)
    assert abs(oracle.sin_theta(U, V) - expect) < 1e-3 * expect


def test_tls_exact_oracle_equals_svd_of_augmented(oracle):
    # tls.cpp:83-95: the R factor of [A|B] shares singular values and right
    # singular vectors with [A|B]; X = -V_k1 V_k2^{-1} of the trailing subspace.
    rng = np.random.default_rng(3)
    m, n, k = 300, 8, 2
    A = rng.standard_normal((m, n))
    X = rng.standard_normal((n, k))
    B = A @ X + 1e-3 * rng.standard_normal((m, k))
    Xo, Vo, so, res, cond = oracle.tls_solve_exact(A, B)
    _, s, vh = np.linalg.svd(np.concatenate([A, B], axis=1))
    v = vh.T[:, n:]
    assert np.max(np.abs(so - s)) <= 1e-13 * s[0]
    assert oracle.sin_theta(Vo, v) < 1e-12
    assert np.linalg.norm(Xo - np.linalg.solve(v[n:].T, -v[:n].T).T) <= 1e-10 * np.linalg.norm(Xo)
    assert abs(res - math.sqrt(np.sum(s[n:] ** 2))) <= 1e-12 * res
    assert np.linalg.norm(Xo - X) / np.linalg.norm(X) < 1e-2
