"""Time svd_trailing on random s x n inputs: python tools/svd_shape.py s n [s n ...] (NSK_SVD_DEBUG=1 for phases)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402

args = [int(a) for a in sys.argv[1:]] or [4096, 64]
for s, n in zip(args[::2], args[1::2]):
    g = torch.Generator(device="cuda").manual_seed(s + n)
    X = torch.randn(n, s, dtype=torch.float64, device="cuda", generator=g).t()
    nsk.svd_trailing(X, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        nsk.svd_trailing(X, 1)
    e1.record()
    torch.cuda.synchronize()
    print(f"s={s} n={n}: {e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
