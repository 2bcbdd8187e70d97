"""Device time of the general-length / cyclic-shard srft and srdct engine (srtt_general.cu)
against the tuned stream kernels at the configs[1] shape.  Prints ms and GB/s of A read."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402


def t_apply(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n, s = 256, 1024
for kind in ("srft", "srdct"):
    for m, P in ((1 << 20, 1), (1 << 20, 8), (1000000, 1), (1 << 23, 8), (20000 * 50, 1)):
        mloc = m // P
        A = torch.randn(n, mloc, dtype=torch.float64, device="cuda").t()
        S = nsk.SketchOperator.draw(kind, s, m, 5)
        if P == 1:
            ms = t_apply(lambda: nsk.apply(S, A))
        else:
            ms = t_apply(lambda: nsk.apply_shard(S, A, 3, P))
        print(f"{kind:6s} m={m:9d} P={P} rows/rank={mloc:8d} n={n} s={s}: {ms:8.3f} ms  "
              f"{mloc * n * 8 / ms / 1e6:7.1f} GB/s", flush=True)
        del A
