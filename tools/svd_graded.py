"""SVD of a graded s x n test matrix (sigma logspaced 1 -> 1e-3, trailing k = 1e-12), NSK_SVD_DEBUG prints sweeps."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk
s, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 4
g = torch.Generator(device="cuda").manual_seed(1)
U, _ = torch.linalg.qr(torch.randn(s, n, dtype=torch.float64, device="cuda", generator=g))
V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
sig = torch.cat([torch.logspace(0, -3, n - k, dtype=torch.float64, device="cuda"),
                 torch.full((k,), 1e-12, dtype=torch.float64, device="cuda")])
X = (U * sig) @ V.t()
X = X.t().contiguous().t()
for _ in range(2):
    W, sv = nsk.svd_trailing(X, k)
torch.cuda.synchronize()
ang = torch.linalg.norm(V[:, n - k:].t() @ W).item() ** 2 / k
print("ok", sv[:2].tolist(), sv[-k:].tolist(), "subspace cos2 mean", ang)
