"""Stress the warp-specialised / stream transform kernels: repeated applies must be bit-identical
(a race in the mbarrier / named-barrier hand-offs would show up as a differing rerun).

usage: python tools/stress_stream.py [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    g = torch.Generator(device="cuda").manual_seed(3)
    bad = 0
    for kind in ("srft", "srdct"):
        for (m, n, s) in [(1 << 14, 3, 1), (1 << 16, 150, 1024), (1 << 20, 64, 1024), (5 << 14, 7, 1500),
                          (1 << 18, 257, 333)]:
            A = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
            S = nsk.SketchOperator.draw(kind, s, m, 77)
            ref = nsk.apply(S, A).data.clone()
            diff = 0
            for _ in range(reps):
                if not torch.equal(nsk.apply(S, A).data, ref):
                    diff += 1
            bad += diff
            print(f"{kind:5s} m={m:8d} n={n:4d} s={s:5d}: {reps} reruns, {diff} differ", flush=True)
    print("stress ok" if bad == 0 else f"stress FAILED ({bad} differing reruns)")


if __name__ == "__main__":
    main()
