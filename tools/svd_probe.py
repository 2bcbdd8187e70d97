"""Time the on-device SVD (svd_trailing) at the BASELINE shapes; prints ms per call."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk
for (s, n) in [(1024, 256), (1024, 512), (4096, 64), (400, 100)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(n, s, dtype=torch.float64, device="cuda", generator=g).t()
    nsk.svd_trailing(X, 1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); W, sig = nsk.svd_trailing(X, 1); e1.record(); torch.cuda.synchronize()
    ref = np.linalg.svd(X.cpu().numpy(), compute_uv=False)
    print(f"svd {s}x{n}: {e0.elapsed_time(e1):.3f} ms  max|dsig|/s1 = {np.max(np.abs(sig.cpu().numpy()-ref))/ref[0]:.2e}", flush=True)
