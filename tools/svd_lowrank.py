import sys, torch
sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk
for n, s, r in [(64, 256, 2), (256, 1024, 2), (512, 1024, 2), (512, 1024, 1), (300, 1200, 5), (512, 2048, 100), (16, 64, 0)]:
    g = torch.Generator(device="cuda").manual_seed(n + r)
    if r == 0:
        X = torch.zeros(s, n, dtype=torch.float64, device="cuda")
    else:
        X = torch.randn(s, r, dtype=torch.float64, device="cuda", generator=g) @ torch.randn(r, n, dtype=torch.float64, device="cuda", generator=g)
    X = X.t().contiguous().t()
    try:
        W, sv = nsk.svd_trailing(X, 2)
        ref = torch.linalg.svdvals(X)
        print(n, s, r, "ok", float((sv - ref).abs().max() / max(ref[0].item(), 1e-300)), float(torch.linalg.norm(X @ W)), float(torch.linalg.norm(W.T @ W - torch.eye(2, device="cuda", dtype=torch.float64))))
    except Exception as e:
        print(n, s, r, "FAIL", e)
