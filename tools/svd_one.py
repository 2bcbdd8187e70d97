import sys, torch
sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk
s, n = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(n, s, dtype=torch.float64, device="cuda", generator=g).t()
for _ in range(2):
    W, sig = nsk.svd_trailing(X, 1)
torch.cuda.synchronize()
print("ok", sig[:3].tolist())
