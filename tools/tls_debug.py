import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2206_00975_b200 as nsk
from oracle import sketch_oracle as O
for cplx, k in ((True, 60), (False, 60), (True, 20), (True, 40), (True, 33), (True, 32)):
    rng = np.random.default_rng(3)
    m, n, s = 600, 64, 300
    A = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
    X0 = rng.standard_normal((n, k)) + (1j * rng.standard_normal((n, k)) if cplx else 0)
    B = A @ X0 + 1e-6 * (rng.standard_normal((m, k)) + (1j * rng.standard_normal((m, k)) if cplx else 0))
    S = nsk.SketchOperator.draw("gaussian", s, m, 5)
    sol = nsk.tls_solve_sketched(torch.from_numpy(np.asfortranarray(A)).cuda(), torch.from_numpy(np.asfortranarray(B)).cuda(), S, allow_marginal=True)
    Xr, Vr, sr, _, _ = O.tls_solve_sketched(A, B, O.draw("gaussian", s, m, 5), allow_marginal=True)
    V = sol.Vk.cpu().numpy(); X = sol.X.cpu().numpy()
    v1, v2 = V[:n], V[n:]
    Xv = np.linalg.solve(v2.T, -v1.T).T
    print(cplx, k, "sinV", O.sin_theta(V, Vr), "X vs oracle", np.linalg.norm(X - Xr) / np.linalg.norm(Xr), "X from gpu V", np.linalg.norm(Xv - Xr) / np.linalg.norm(Xr), "orth", np.abs(V.conj().T @ V - np.eye(k)).max())
