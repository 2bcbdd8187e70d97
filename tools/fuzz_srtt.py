"""Random-shape parity sweep of the srft / srdct paths (general-length engine, tiles, shards) against
the oracle.  python tools/fuzz_srtt.py [cases] -- prints the worst relative error per path."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402
from oracle import sketch_oracle as O  # noqa: E402

rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
worst = {}
for c in range(cases):
    kind = rng.choice(["srft", "srdct"])
    m = int(rng.choice([rng.integers(2, 3000), rng.integers(3000, 300000), 4096 * int(rng.integers(1, 40))]))
    s = int(rng.integers(1, min(m, 3000) + 1))
    n = int(rng.integers(1, 7))
    cplx = kind == "srft" and rng.random() < 0.4
    A = O.random_complex(m, n, c) if cplx else O.random_real(m, n, c)
    seed = int(rng.integers(1, 1 << 30))
    S = nsk.SketchOperator.draw(kind, s, m, seed)
    op = O.draw(kind, s, m, seed)
    ref = O.apply(op, A)
    got = nsk.apply(S, torch.from_numpy(np.asfortranarray(A)).cuda()).data.cpu().numpy()
    e = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    key = f"{kind}{'-c' if cplx else ''} full"
    worst[key] = max(worst.get(key, 0.0), e)
    if e > 1e-12:
        print("FAIL", kind, m, s, n, cplx, e, flush=True)
    # cyclic shards when P | m
    for P in (2, 3, 4, 8):
        if m % P or m // P < 1 or cplx:
            continue
        acc = None
        for g in range(P):
            part = nsk.apply_shard(S, torch.from_numpy(np.ascontiguousarray(A[g::P])).cuda().t().contiguous().t()
                                   if A.ndim > 1 else None, g, P).cpu().numpy()
            acc = part if acc is None else acc + part
        e2 = np.linalg.norm(acc - ref) / max(np.linalg.norm(ref), 1e-300)
        key2 = f"{kind} shards"
        worst[key2] = max(worst.get(key2, 0.0), e2)
        if e2 > 1e-12:
            print("FAIL shard", kind, m, s, n, P, e2, flush=True)
        break
for k, v in sorted(worst.items()):
    print(f"{k:14s} worst rel err {v:.3e}")
