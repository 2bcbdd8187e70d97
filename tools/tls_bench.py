"""Exact vs sketched total least squares on the device (the reference's `tls`
bench recipe, bench.cpp:240-310, and PAPER.md Table 1): device-resident
A (m x n, N(0,1)), B = A x_true + noise N(0,1), both solvers timed end to end
(median of 5, CUDA events), plus the error metrics of tls.cpp:115-131.

Usage: python tools/tls_bench.py [--m 4194304] [--n 511] [--k 1] [--noise 1e-3]
                                 [--kinds gaussian,srht,countsketch] [--reps 5]
Prints one JSON line per sketch kind.
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402


def timed(fn, reps):
    ts, out = [], None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2], out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1 << 22)
    ap.add_argument("--n", type=int, default=511)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--noise", type=float, default=1e-3)
    ap.add_argument("--kinds", default="gaussian,srht,countsketch")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(a.seed)
    m, n, k = a.m, a.n, a.k
    A = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()  # column-major
    xt = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g)
    B = (A @ xt + a.noise * torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g))
    B = B.t().contiguous().t()
    t_exact, ex = timed(lambda: nsk.tls_solve_exact(A, B, allow_marginal=True), a.reps)
    cert = nsk.tls_solve_exact(A, B, allow_marginal=True, certificate=True).residual_certificate
    for kind in a.kinds.split(","):
        s = {"gaussian": 2 * (n + k), "srht": 4 * (n + k), "countsketch": 8 * (n + k)}[kind]
        S = nsk.SketchOperator.draw(kind, s, m, a.seed + 1)
        t_sk, sk = timed(lambda: nsk.tls_solve_sketched(A, B, S, allow_marginal=True), a.reps)
        skc = nsk.tls_solve_sketched(A, B, S, allow_marginal=True, certificate=True)
        met = nsk.tls_error_metrics(ex, sk)
        print(json.dumps({
            "m": m, "n": n, "k": k, "noise": a.noise, "sketch": kind, "s": s,
            "time_exact_ms": round(t_exact, 3), "time_sketched_ms": round(t_sk, 3),
            "speedup": round(t_exact / t_sk, 3),
            "residual_exact": ex.tls_residual, "residual_exact_certified": cert,
            "residual_ratio": skc.residual_certificate / ex.tls_residual,
            "rel_err": met.rel_err, "sin_X": met.sin_X, "sin_vk": met.sin_Vk,
            "x_err_vs_truth": float(torch.linalg.norm(sk.X - xt) / torch.linalg.norm(xt)),
        }), flush=True)


if __name__ == "__main__":
    main()
