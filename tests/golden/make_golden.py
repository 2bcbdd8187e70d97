"""Generate the golden fixtures in tests/golden/ from the REFERENCE's own RNG.

Runs only where /root/reference exists (this container): it compiles the
reference header proj/include/nullsketch/rng.hpp unmodified into oracle/_ref/
(oracle/Makefile) and records the exact call sequences the reference library
issues:
  * PhiloxStream::next_u32 / next_gaussian / next_double (rng.hpp:25-54)
  * SketchOperator::draw for gaussian  -> G column-major (sketch.cpp:117-121)
  * SketchOperator::draw for srft/srdct -> m signs + sorted Fisher-Yates sample
    (sketch.cpp:122-126, rng.hpp:108-121)
  * the CountSketch protocol defined on the same stream (m next_sign, then
    m next_below(s))
  * row-update Gaussians of stream (seed, 1) (sketch.cpp:273-275)
Also records the Random123 Philox4x32-10 known answer (key 0, counter 0).
The SA/W golden vectors are computed by the oracle restatement on these
pinned draws (tests/golden/sa_*.npz).

Usage: python tests/golden/make_golden.py
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import sketch_oracle as O  # noqa: E402


def main():
    O.build()
    R = O.ref_lib()
    if R is None:
        raise SystemExit("oracle/_ref/libnsk_ref.so missing: the reference tree is needed to pin fixtures")
    dp, ip, i32p, u32p = O._dp, O._ip, O._i32p, O._u32p
    out = {}
    # Philox word streams and Gaussians for assorted (seed, stream)
    cases = [(0, 0), (42, 0), (42, 1), (9000001, 0), (2**64 - 1, 77), (123456789, 2)]
    for seed, stream in cases:
        w = np.empty(64, np.uint32)
        R.nskref_words(seed, stream, 64, w.ctypes.data_as(u32p))
        g = np.empty(64)
        R.nskref_gaussians(seed, stream, 64, g.ctypes.data_as(dp))
        d = np.empty(16)
        R.nskref_doubles(seed, stream, 16, d.ctypes.data_as(dp))
        out[f"words_{seed}_{stream}"] = w
        out[f"gauss_{seed}_{stream}"] = g
        out[f"double_{seed}_{stream}"] = d
    # gaussian operator matrix G (test_sketch.cpp:103-114 uses s = m = 4, seed 42)
    for s, m, seed in [(4, 4, 42), (6, 16, 123), (7, 9, 5)]:
        G = np.empty(s * m)
        R.nskref_gaussian_G(seed, s, m, G.ctypes.data_as(dp))
        out[f"G_{s}_{m}_{seed}"] = G.reshape(m, s).T.copy()
    # srft/srdct draws (also SRHT's protocol)
    for m, s, seed in [(16, 6, 123), (1000, 64, 7), (1 << 20, 1024, 9000002), (1000003, 512, 9000077),
                       (20000, 400, 11), (60, 60, 7)]:
        sg = np.empty(m)
        idx = np.empty(s, np.int64)
        R.nskref_srtt_draw(seed, m, s, sg.ctypes.data_as(dp), idx.ctypes.data_as(ip))
        out[f"idx_{m}_{s}_{seed}"] = idx
        out[f"signbits_{m}_{s}_{seed}"] = np.packbits((sg > 0).astype(np.uint8))
    # CountSketch draw protocol
    for m, s, seed in [(1000, 64, 3), (1 << 16, 4096, 9000003)]:
        b = np.empty(m, np.int32)
        sg = np.empty(m)
        R.nskref_countsketch_draw(seed, m, s, b.ctypes.data_as(i32p), sg.ctypes.data_as(dp))
        out[f"csbucket_{m}_{s}_{seed}"] = b
        out[f"cssignbits_{m}_{s}_{seed}"] = np.packbits((sg > 0).astype(np.uint8))
    # row-update Gaussians, stream (seed, 1)
    ug = np.empty(10 * 3)
    R.nskref_update_gaussians(45, 10, 3, ug.ctypes.data_as(dp))
    out["update_gauss_45_10_3"] = ug.reshape(3, 10).T.copy()
    np.savez_compressed(os.path.join(HERE, "draws_ref.npz"), **out)
    print("wrote draws_ref.npz with", len(out), "arrays")

    # SA / W / sigma golden vectors from the oracle restatement, small shapes.
    sa = {}
    spec = np.concatenate([np.logspace(0, -3, 19), [1e-10]])
    A = O.make_test_matrix(2000, 20, spec, seed=1)
    sa["A_2000_20"] = A
    for kind, s in [("gaussian", 80), ("srdct", 40), ("srht", 40), ("countsketch", 400)]:
        m = 2048 if kind == "srht" else 2000
        Ak = O.make_test_matrix(m, 20, spec, seed=1) if m != 2000 else A
        op = O.draw(kind, s, m, 9000001)
        SA = O.apply(op, Ak)
        W, sv = O.solve_k(Ak, 1, op)
        sa[f"SA_{kind}"] = SA
        sa[f"W_{kind}"] = W
        sa[f"sigma_{kind}"] = sv
        if m != 2000:
            sa[f"A_{m}_20"] = Ak
    Ac = O.random_complex(300, 12, 5)
    op = O.draw("srft", 24, 300, 9000004)
    sa["A_srft"] = Ac
    sa["SA_srft"] = O.apply(op, Ac)
    np.savez_compressed(os.path.join(HERE, "sa_oracle.npz"), **sa)
    print("wrote sa_oracle.npz")


if __name__ == "__main__":
    main()
