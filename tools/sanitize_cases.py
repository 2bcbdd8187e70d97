"""Small cases that walk every kernel family once, each checked against the oracle: the quick
whole-library sanity pass (`python tools/sanitize_cases.py [family ...]`).  Sizes are the smallest
that still take the tile / TMA / cluster kernels rather than their fallbacks.  (Written for
compute-sanitizer, which is closed on this GPU pool; the oracle comparison is what remains.)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_00975_b200 as nsk  # noqa: E402
from oracle import sketch_oracle as O  # noqa: E402

only = set(sys.argv[1:])
torch.cuda.set_device(0)


def want(name):
    return not only or name in only


def dev(A):
    return torch.from_numpy(np.asfortranarray(A)).cuda()


def check_apply(kind, s, A, tag):
    m = A.shape[0]
    S = nsk.SketchOperator.draw(kind, s, m, 7000003)
    SA = nsk.apply(S, dev(A)).data.cpu().numpy()
    ref = O.apply(O.draw(kind, s, m, 7000003), A)
    err = np.linalg.norm(SA - ref) / np.linalg.norm(ref)
    print(f"{tag}: {kind} {A.shape} s={s} rel err {err:.2e}", flush=True)
    assert err <= 1e-12, (tag, err)
    return S


if want("srht"):
    check_apply("srht", 64, O.random_real(8192, 8, 1), "srht blocked 2048-row warps")
    check_apply("srht", 64, O.random_real(1024, 5, 2), "srht 1024-row warps")
if want("countsketch"):
    check_apply("countsketch", 256, O.random_real(70000, 16, 3), "countsketch owner kernel")
if want("gaussian"):
    check_apply("gaussian", 64, O.random_real(5000, 24, 4), "gaussian real (TMA tiles need 16-byte rows)")
    check_apply("gaussian", 64, O.random_real(4099, 7, 5), "gaussian real, odd shape")
    Z = O.random_real(3000, 20, 6) + 1j * O.random_real(3000, 20, 7)
    check_apply("gaussian", 48, Z, "gaussian complex")
if want("srft"):
    check_apply("srft", 64, O.random_real(1 << 15, 6, 8), "srft warp-specialised tiles")
    check_apply("srft", 64, O.random_real(20000, 4, 9), "srft general length")
    Z = O.random_real(1 << 14, 3, 10) + 1j * O.random_real(1 << 14, 3, 11)
    check_apply("srft", 32, Z, "srft complex")
if want("srdct"):
    check_apply("srdct", 64, O.random_real(1 << 15, 6, 12), "srdct stream kernel")
    check_apply("srdct", 64, O.random_real(9985, 4, 13), "srdct general length")
if want("svd"):
    for (s, n) in ((128, 32), (400, 100), (640, 300)):
        M = O.random_real(s, n, 14 + n)
        W, sig = nsk.svd_trailing(dev(M), 2)
        sref = np.linalg.svd(M, compute_uv=False)
        err = np.max(np.abs(sig.cpu().numpy() - sref)) / sref[0]
        print(f"svd {s}x{n}: sigma err {err:.2e}", flush=True)
        assert err <= 1e-12
    Mc = O.random_real(300, 150, 40) + 1j * O.random_real(300, 150, 41)
    W, sig = nsk.svd_trailing(dev(Mc), 1)
    sref = np.linalg.svd(Mc, compute_uv=False)
    assert np.max(np.abs(sig.cpu().numpy() - sref)) / sref[0] <= 1e-12
    print("svd complex 300x150 ok", flush=True)
if want("solve"):
    m, n = 4096, 16
    spec = np.concatenate([np.logspace(0, -3, n - 1), [1e-10]])
    A = O.make_test_matrix(m, n, spec, seed=1)
    S = nsk.SketchOperator.draw("gaussian", 4 * n, m, 9000001)
    res = nsk.solve_k(dev(A), 1, S)
    Wref, _ = O.solve_k(A, 1, O.draw("gaussian", 4 * n, m, 9000001))
    ang = O.sin_theta(res.W.cpu().numpy(), Wref)
    cert = nsk.residual_certificate(dev(A), res.W)
    print(f"solve_k angle {ang:.2e} certificate {cert:.2e}", flush=True)
    assert ang <= 1e-10
if want("tls"):
    m, n = 6000, 12
    A = O.random_real(m, n, 50)
    x = O.random_real(n, 1, 51)
    B = A @ x + 1e-3 * O.random_real(m, 1, 52)
    S = nsk.SketchOperator.draw("gaussian", 4 * (n + 1), m, 11)
    sol = nsk.tls_solve_sketched(dev(A), dev(B), S)
    ex = nsk.tls_solve_exact(dev(A), dev(B))
    X = sol.X.cpu().numpy() if hasattr(sol.X, "cpu") else np.asarray(sol.X)
    print("tls |X - x| / |x| =", np.linalg.norm(X - x) / np.linalg.norm(x), flush=True)
    assert np.linalg.norm(X - x) / np.linalg.norm(x) < 5e-2
if want("updates"):
    m, n = 5000, 10
    A = O.random_real(m, n, 60)
    for kind in ("gaussian", "srdct", "srft"):
        S = nsk.SketchOperator.draw(kind, 40, m, 13)
        sa = nsk.apply(S, dev(A))
        col = O.random_real(m, 1, 61)[:, 0]
        sa2 = nsk.update_column(sa, S, dev(col), 3)
        sa3 = nsk.downdate_column(sa2, 3)
        err = (sa3.data - sa.data).abs().max().item()
        assert err <= 1e-12, (kind, err)
        row = O.random_real(1, n, 62)[0]
        sa4 = nsk.update_row(sa, S, dev(row))
        assert sa4.data.shape[1] == n
    print("updates ok", flush=True)
torch.cuda.synchronize()
print("sanitize cases ok")
