"""C-ABI library: loads, exports every declared symbol, host-side logic (CPU only).

No compute entry point is called here (no GPU in this container); the draw,
descriptor and validation paths run on the host.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2206_00975_b200 import _lib
from paper_2206_00975_b200.sketch import SketchOperator, default_sketch_size

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2206_00975_b200 import build
    build.build()


def declared_symbols():
    syms = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", f)).read()
            syms |= set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(nsk_\w+)\s*\(", txt, re.M))
    return syms


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 17
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in sorted(syms):
        assert hasattr(L, s), s
    assert set(_lib.EXPORTS) == syms


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kind,m,s,seed", [("srdct", 16, 6, 123), ("srft", 1000, 64, 7), ("srht", 1 << 20, 1024, 9000002),
                                           ("srdct", 1000003, 512, 9000077), ("srdct", 20000, 400, 11)])
def test_sample_indices_bit_exact(golden, kind, m, s, seed):
    S = SketchOperator.draw(kind, s, m, seed)
    assert np.array_equal(S.sample_indices(), golden["draws"][f"idx_{m}_{s}_{seed}"])


def test_draw_validation_matches_reference():
    # test_sketch.cpp:91-101
    with pytest.raises(ValueError):
        SketchOperator.draw("srft", 10, 8, 1)
    with pytest.raises(ValueError):
        SketchOperator.draw("srdct", 10, 8, 1)
    with pytest.raises(ValueError):
        SketchOperator.draw("gaussian", 0, 8, 1)
    SketchOperator.draw("gaussian", 10, 8, 1)  # taller than m is allowed
    with pytest.raises(ValueError):
        SketchOperator.draw("srht", 4, 12, 1)   # no zero padding: m must be 2^p
    with pytest.raises(ValueError):
        SketchOperator.draw("nope", 4, 12, 1)
    assert default_sketch_size("srft", 50) == 100
    assert default_sketch_size("srdct", 50) == 100
    assert default_sketch_size("gaussian", 50) == 200


def test_descriptor_round_trip():
    for kind in ("gaussian", "srft", "srdct", "srht", "countsketch"):
        m = 64
        S = SketchOperator.draw(kind, 10, m, 112)
        d = S.descriptor()
        assert d == ('{"appended":0,"format":1,"kind":"%s","m":64,"s":10,"seed":112,"zeroed_rows":[]}' % kind)
        R = SketchOperator.from_descriptor(d)
        assert (R.kind, R.s, R.m, R.seed) == (S.kind, S.s, S.m, S.seed)
        assert R.id != S.id
        if kind in ("srft", "srdct", "srht"):
            assert np.array_equal(R.sample_indices(), S.sample_indices())
    # sketch.cpp:315-337 error paths (test_sketch.cpp:424-427)
    with pytest.raises(ValueError):
        SketchOperator.from_descriptor("{}")
    with pytest.raises(ValueError):
        SketchOperator.from_descriptor('{"format":1,"kind":"srft","s":4,"m":8,"seed":1,"appended":0,'
                                       '"zeroed_rows":[9]}')


def test_draw_is_deterministic_and_seeded():
    a = SketchOperator.draw("srdct", 6, 16, 123).sample_indices()
    b = SketchOperator.draw("srdct", 6, 16, 123).sample_indices()
    c = SketchOperator.draw("srdct", 6, 16, 124).sample_indices()
    assert np.array_equal(a, b) and not np.array_equal(a, c)
