"""One sketched-TLS call at configs[3] (m = 2^22, n = 511, k = 1) after a warm-up, for a launch list
(ncu --metrics gpu__time_duration.sum) and the SVD stages' globaltimer stamps (NSK_SVD_DEBUG=1)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402

m = int(os.environ.get("TLS_M", 1 << 22))
n, s = 511, 1024
g = torch.Generator(device="cuda").manual_seed(1)
C = torch.randn(n + 1, m, dtype=torch.float64, device="cuda", generator=g).t()
A, b = C[:, :n], C[:, n:]
S = nsk.SketchOperator.draw("gaussian", s, m, 3)
nsk.tls_solve_sketched(A, b, S, allow_marginal=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
nsk.tls_solve_sketched(A, b, S, allow_marginal=True)
e1.record()
torch.cuda.synchronize()
print("tls_solve_sketched %.2f ms" % e0.elapsed_time(e1), flush=True)
