"""Where the SVD time goes (1024 x 512, 1024 x 256): whole call vs the cluster stage's own clock
stamps (NSK_SVD_DEBUG=1 prints QRCP / transpose / sweep milliseconds)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402

for s, n in ((1024, 512), (1024, 256)):
    X = torch.randn(n, s, dtype=torch.float64, device="cuda").t()
    for _ in range(2):
        nsk.svd_trailing(X, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nsk.svd_trailing(X, 1)
    e1.record()
    torch.cuda.synchronize()
    print(f"svd {s} x {n}: {e0.elapsed_time(e1):.2f} ms", flush=True)
    os.environ["NSK_SVD_DEBUG"] = "1"
    nsk.svd_trailing(X, 1)
    torch.cuda.synchronize()
    del os.environ["NSK_SVD_DEBUG"]
