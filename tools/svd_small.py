"""SVD time at the small BASELINE shapes (configs[0] 400 x 100, configs[2] 4096 x 64, configs[4]
300 x 150 complex) and configs[1] 1024 x 256: whole call (CUDA events, median of 7) and, with
NSK_SVD_DEBUG=1, the cluster stage's own phase stamps.  `--once` runs each shape once (for an
ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402

SHAPES = ((400, 100, False), (4096, 64, False), (300, 150, True), (1024, 256, False), (1024, 512, False))


def make(s, n, cplx):
    dt = torch.complex128 if cplx else torch.float64
    g = torch.Generator(device="cuda").manual_seed(n)
    U, _ = torch.linalg.qr(torch.randn(s, n, dtype=dt, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=dt, device="cuda", generator=g))
    sig = torch.cat([torch.logspace(0, -3, n - 1, dtype=torch.float64, device="cuda"),
                     torch.full((1,), 1e-10, dtype=torch.float64, device="cuda")])
    X = (U * sig.to(dt)) @ V.mH
    return X.t().contiguous().t()


def main():
    once = "--once" in sys.argv
    for s, n, cplx in SHAPES:
        X = make(s, n, cplx)
        if once:
            nsk.svd_trailing(X, 1)
            torch.cuda.synchronize()
            continue
        for _ in range(2):
            nsk.svd_trailing(X, 1)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nsk.svd_trailing(X, 1)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"svd {s} x {n} {'c128' if cplx else 'f64'}: {ts[3]:.3f} ms (min {ts[0]:.3f})", flush=True)
        os.environ["NSK_SVD_DEBUG"] = "1"
        nsk.svd_trailing(X, 1)
        torch.cuda.synchronize()
        del os.environ["NSK_SVD_DEBUG"]


if __name__ == "__main__":
    main()
