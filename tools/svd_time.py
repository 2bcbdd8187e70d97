"""Time and check svd_trailing on graded / random s x n inputs (real and complex).

Usage: python tools/svd_time.py [n ...]; env NSK_SVD_NORT=1 selects the
unpreconditioned path, NSK_SVD_DEBUG=1 prints the sweep counts.
Prints one line per case: ms per call, max relative sigma error against
torch.linalg.svdvals, and the trailing-subspace residual ||A W|| / sigma_1.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402


def make(s, n, kind, cplx, g):
    dt = torch.complex128 if cplx else torch.float64
    U, _ = torch.linalg.qr(torch.randn(s, n, dtype=dt, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=dt, device="cuda", generator=g))
    if kind == "graded":
        sig = torch.cat([torch.logspace(0, -3, n - 4, dtype=torch.float64, device="cuda"),
                         torch.full((4,), 1e-12, dtype=torch.float64, device="cuda")])
    elif kind == "steep":
        sig = torch.logspace(0, -14, n, dtype=torch.float64, device="cuda")
    else:
        return torch.randn(n, s, dtype=dt, device="cuda", generator=g).t()
    X = (U * sig.to(dt)) @ V.mH
    return X.t().contiguous().t()


def main():
    ns = [int(a) for a in sys.argv[1:]] or [64, 128, 256]
    for n in ns:
        s = 4 * n
        for cplx in (False, True):
            for kind in ("random", "graded", "steep"):
                g = torch.Generator(device="cuda").manual_seed(n)
                X = make(s, n, kind, cplx, g)
                k = 4
                W, sv = nsk.svd_trailing(X, k)
                torch.cuda.synchronize()
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 5
                t0.record()
                for _ in range(reps):
                    W, sv = nsk.svd_trailing(X, k)
                t1.record()
                torch.cuda.synchronize()
                ms = t0.elapsed_time(t1) / reps
                ref = torch.linalg.svdvals(X)
                err = ((sv - ref).abs() / ref[0]).max().item()
                res = (torch.linalg.norm(X @ W) / ref[0]).item()
                orth = torch.linalg.norm(W.mH @ W - torch.eye(k, dtype=W.dtype, device="cuda")).item()
                print(f"n={n} {'c' if cplx else 'r'} {kind:7s} {ms:8.3f} ms  sigma_err/s1={err:.2e} "
                      f"||AW||/s1={res:.2e} (ref {ref[-1].item() / ref[0].item():.1e}) orth={orth:.1e}", flush=True)


if __name__ == "__main__":
    main()
