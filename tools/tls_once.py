"""One sketched TLS call at configs[3] (for an ncu launch list of its kernels)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402

m, n, s = 1 << 22, 511, 1024
g = torch.Generator(device="cuda").manual_seed(1)
C = torch.randn(n + 1, m, dtype=torch.float64, device="cuda", generator=g).t()
S = nsk.SketchOperator.draw("gaussian", s, m, 3)
for _ in range(2):
    nsk.tls_solve_sketched(C[:, :n], C[:, n:], S, allow_marginal=True)
torch.cuda.synchronize()
