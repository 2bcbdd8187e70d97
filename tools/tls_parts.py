"""Device-time breakdown of sketched TLS at configs[3] (m = 2^22, n = 511, k = 1, Gaussian s = 1024):
the one-pass apply of S [A | b], the two SVDs of tls.cpp:110-111, and the whole call."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


m, n, s = 1 << 22, 511, 1024
g = torch.Generator(device="cuda").manual_seed(1)
C = torch.randn(n + 1, m, dtype=torch.float64, device="cuda", generator=g).t()
A, b = C[:, :n], C[:, n:]
S = nsk.SketchOperator.draw("gaussian", s, m, 3)
SA = nsk.apply(S, C).data
print("apply [A b] (512 cols)  %.2f ms" % t(lambda: nsk.apply(S, C)))
print("svd 1024 x 512 (k=1)    %.2f ms" % t(lambda: nsk.svd_trailing(SA, 1)))
print("svd 1024 x 511 (k=0)    %.2f ms" % t(lambda: nsk.svd_trailing(SA[:, :n], 0)))
print("tls_solve_sketched      %.2f ms" % t(lambda: nsk.tls_solve_sketched(A, b, S, allow_marginal=True)))
