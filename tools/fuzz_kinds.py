"""Random-shape parity sweep of gaussian / srht / countsketch: device apply, host (pageable) apply and
contiguous row shards against the oracle.  python tools/fuzz_kinds.py [cases] [seed]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402
from oracle import sketch_oracle as O  # noqa: E402

rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
worst = {}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def note(key, e, info):
    worst[key] = max(worst.get(key, 0.0), e)
    if e > 1e-12:
        print("FAIL", key, info, e, flush=True)


for c in range(cases):
    kind = str(rng.choice(["gaussian", "srht", "countsketch"]))
    if kind == "srht":
        m = 1 << int(rng.integers(4, 19))
    else:
        m = int(rng.choice([rng.integers(2, 5000), rng.integers(5000, 400000)]))
    s = int(rng.integers(1, (min(m, 1024) if kind == "srht" else 2048) + 1))
    if kind == "countsketch":
        s = int(rng.integers(1, 5000))
    n = int(rng.integers(1, 9))
    cplx = kind == "gaussian" and rng.random() < 0.3
    A = O.random_complex(m, n, c) if cplx else O.random_real(m, n, c)
    seed = int(rng.integers(1, 1 << 30))
    S = nsk.SketchOperator.draw(kind, s, m, seed)
    ref = O.apply(O.draw(kind, s, m, seed), A)
    info = (kind, m, s, n, cplx)
    got = nsk.apply(S, torch.from_numpy(np.asfortranarray(A)).cuda()).data.cpu().numpy()
    note(kind + " device", rel(got, ref), info)
    note(kind + " host", rel(np.asarray(nsk.apply(S, A).data), ref), info)
    align = {"srht": 2048, "countsketch": 512}.get(kind, 1)
    if m >= 4 * align and not cplx:
        cuts = sorted(set(int(x) // align * align for x in rng.integers(1, m, size=2)))
        cuts = [0] + [x for x in cuts if 0 < x < m] + [m]
        acc = 0
        for a, b in zip(cuts[:-1], cuts[1:]):
            acc = acc + nsk.apply_shard(S, torch.from_numpy(np.asfortranarray(A[a:b])).cuda(), a).cpu().numpy()
        note(kind + " shards", rel(acc, ref), info + (cuts,))
for k, v in sorted(worst.items()):
    print(f"{k:20s} worst rel err {v:.3e}")
