"""The Gaussian sketch's TMA A-tile paths (real 2-D boxes, complex boxes with permuted fragment
columns, contiguous [A | B]) against its cp.async path and the oracle, and the register-resident
look-ahead QR against the column-in-memory one.

Both Gaussian paths feed the same DMMAs in the same order, so SA must agree bit for bit
(NSK_GAUSS_TMA=0 selects the cp.async path); the QR kernels sum in different orders, so their
SVDs agree to rounding (sigma within 1e3 u sigma_1, trailing vectors within 1e-12).
"""
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


def sketch_both(nsk, monkeypatch, S, Ad):
    monkeypatch.delenv("NSK_GAUSS_TMA", raising=False)
    tma = host(nsk.apply(S, Ad).data)
    monkeypatch.setenv("NSK_GAUSS_TMA", "0")
    cpa = host(nsk.apply(S, Ad).data)
    monkeypatch.delenv("NSK_GAUSS_TMA")
    return tma, cpa


# n = 200 / 300 real columns: the BN = 256 and BN = 512 tiles; m = 1003 leaves a partial last chunk
# (TMA zero-fills the rows past m); s = 300 leaves a partial s-tile.
@pytest.mark.parametrize("s,m,n", [(256, 4096, 200), (300, 1003, 300), (1024, 20000, 512), (64, 777, 129)])
def test_gaussian_tma_real_bit_identical(nsk, oracle, monkeypatch, s, m, n):
    A = oracle.random_real(m, n, 41)
    S = nsk.SketchOperator.draw("gaussian", s, m, 4242)
    tma, cpa = sketch_both(nsk, monkeypatch, S, dev(A))
    assert np.array_equal(tma, cpa)
    assert rel(tma, oracle.apply(oracle.draw("gaussian", s, m, 4242), A)) <= SA_TOL


# complex: 150 and 100 complex columns (300 / 200 logical columns: BN = 512 / 256 tiles)
@pytest.mark.parametrize("s,m,n", [(300, 5003, 150), (128, 2048, 100), (40, 999, 7)])
def test_gaussian_tma_complex_bit_identical(nsk, oracle, monkeypatch, s, m, n):
    A = oracle.random_complex(m, n, 43)
    S = nsk.SketchOperator.draw("gaussian", s, m, 4343)
    tma, cpa = sketch_both(nsk, monkeypatch, S, dev(A))
    assert np.array_equal(tma, cpa)
    assert rel(tma, oracle.apply(oracle.draw("gaussian", s, m, 4343), A)) <= SA_TOL


def test_tls_contiguous_block_matches_separate(nsk, oracle):
    """[A | b] in one buffer (one tensor map) and A, b in separate buffers (cp.async for the
    straddling tile) give the same sketch, hence the same X, V_k and sigma, bit for bit."""
    import torch
    m, n = 6000, 255
    C = oracle.random_real(m, n + 1, 47)
    S = nsk.SketchOperator.draw("gaussian", 4 * (n + 1), m, 4747)
    Cd = dev(C)
    one = nsk.tls_solve_sketched(Cd[:, :n], Cd[:, n:], S, allow_marginal=True)
    Ad, bd = dev(C[:, :n]), dev(C[:, n:])  # two allocations: not back to back
    two = nsk.tls_solve_sketched(Ad, bd, S, allow_marginal=True)
    torch.cuda.synchronize()
    assert np.array_equal(host(one.X), host(two.X))
    assert np.array_equal(host(one.augmented_singular_values), host(two.augmented_singular_values))


@pytest.mark.parametrize("s,n,cplx", [(1024, 256, False), (1024, 512, False), (600, 300, True), (300, 64, False)])
def test_qr_register_kernel_matches_memory_kernel(nsk, oracle, monkeypatch, s, n, cplx):
    spec = np.concatenate([np.logspace(0, -3, n - 4), np.full(4, 1e-12)])
    X = oracle.make_test_matrix(s, n, spec, seed=5)
    if cplx:
        X = X + 1j * oracle.make_test_matrix(s, n, spec, seed=6)
    Xd = dev(X)
    monkeypatch.delenv("NSK_SVD_QR_OLD", raising=False)
    W1, s1 = nsk.svd_trailing(Xd, 4)
    monkeypatch.setenv("NSK_SVD_QR_OLD", "1")
    W2, s2 = nsk.svd_trailing(Xd, 4)
    monkeypatch.delenv("NSK_SVD_QR_OLD")
    s1, s2 = host(s1), host(s2)
    assert np.max(np.abs(s1 - s2)) <= 1e3 * U * s1[0]
    assert oracle.sin_theta(host(W1), host(W2)) <= 1e-10


# Row shards of a Gaussian operator through the TMA tiles (n = 200 / 300: the 256- and 384-wide
# tiles): the shard partials sum to the whole sketch, and each matches the oracle on A zero
# outside the shard (the tensor map covers the local rows; S is regenerated for the global ones).
@pytest.mark.parametrize("n,cplx", [(200, False), (300, False), (150, True)])
def test_gaussian_tma_row_shards(nsk, oracle, n, cplx):
    m, s = 9000, 320
    A = oracle.random_complex(m, n, 51) if cplx else oracle.random_real(m, n, 51)
    S = nsk.SketchOperator.draw("gaussian", s, m, 5151)
    op = oracle.draw("gaussian", s, m, 5151)
    cuts = [0, 2000, 5120, m]
    total = None
    for a, b in zip(cuts[:-1], cuts[1:]):
        part = host(nsk.apply_shard(S, dev(A[a:b]), a))
        Az = np.zeros_like(A)
        Az[a:b] = A[a:b]
        assert rel(part, oracle.apply(op, Az)) <= SA_TOL
        total = part if total is None else total + part
    assert rel(total, oracle.apply(op, A)) <= SA_TOL
