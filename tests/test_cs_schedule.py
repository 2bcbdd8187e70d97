"""CountSketch owner schedule (cs_schedule.cpp), checked on the host.

The schedule is a pure function of the operator's buckets and signs; these
tests call the library's test hook on synthetic tables and check that every
row is scheduled exactly once, to the thread that owns its bucket, with its
slot and sign, that no half-warp iteration reads a shared-memory bank pair
more than twice (idle lanes only unused ones), and that the iteration count
of every warp is the Koenig optimum of the split-bank graphs.
"""
import ctypes

import numpy as np
import pytest

from paper_2206_00975_b200 import _lib

T, THREADS, WARPS = 4096, 1024, 32


@pytest.fixture(scope="module")
def hook():
    from paper_2206_00975_b200 import build
    build.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    f = L.nsk_internal_cs_schedule
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p,
                  ctypes.c_void_p]
    f.gmax = L.nsk_internal_cs_gmax()
    return f


def run(hook, table, s, T=T):
    ntiles = table.size // T
    ent = np.zeros((ntiles, WARPS, hook.gmax, 32), dtype=np.uint64)
    cnt = np.zeros((ntiles, WARPS), dtype=np.uint8)
    assert hook(table.ctypes.data, ntiles, T, s, ent.ctypes.data, cnt.ctypes.data) == 0
    return ent, cnt


def check(table, s, ent, cnt, T=T):
    ntiles = table.size // T
    for t in range(ntiles):
        tab = table[t * T:(t + 1) * T]
        b_all = tab & 0xFFFF
        seen = np.zeros(T, dtype=np.int64)
        for w in range(WARPS):
            n = int(cnt[t, w])
            for it in range(n):
                col = (ent[t, w, it // 4, :] >> np.uint64(16 * (it % 4))) & np.uint64(0xFFFF)
                for h in range(2):
                    e = col[16 * h:16 * h + 16].astype(np.int64)
                    valid = (e & 0x4000) != 0
                    r = e & 0xFFF
                    uses = np.bincount(r[valid] & 15, minlength=16)
                    assert uses.max(initial=0) <= 2  # at most a 2-way bank conflict
                    assert np.all(uses[r[~valid] & 15] == 0)  # idle lanes read unused bank pairs
                    assert len(set((r[~valid] & 15).tolist())) == int((~valid).sum())
                    assert np.all(e[~valid] < 16)
                    for lane in np.nonzero(valid)[0]:
                        row = int(r[lane])
                        b = int(b_all[row])
                        assert b % THREADS == 32 * w + 16 * h + lane
                        assert (int(e[lane]) >> 12) & 3 == b // THREADS
                        assert (int(e[lane]) >> 15) & 1 == 1 - ((int(tab[row]) >> 16) & 1)  # negative flag
                        seen[row] += 1
            # Koenig optimum: iterations = max(lane degree, ceil(bank-pair degree / 2)) over both halves
            mine = np.nonzero((b_all % THREADS) // 32 == w)[0]
            deg = 0
            for h in range(2):
                sub = mine[((b_all[mine] % 32) >> 4) == h]
                if sub.size:
                    deg = max(deg, np.bincount(b_all[sub] % 16, minlength=16).max(),
                              (np.bincount(sub & 15, minlength=16).max() + 1) // 2)
            assert n == deg
        assert np.all(seen == 1)


@pytest.mark.parametrize("s,ntiles,seed,tile", [(4096, 2, 1, 3072), (3000, 1, 2, 3072), (1024, 1, 3, 3072),
                                                (2048, 1, 4, 3072), (4096, 1, 5, 3072)])
def test_schedule_covers_rows_once_conflict_free_and_optimal(hook, s, ntiles, seed, tile):
    rng = np.random.default_rng(seed)
    b = rng.integers(0, s, size=ntiles * tile, dtype=np.uint32)
    sg = rng.integers(0, 2, size=ntiles * tile, dtype=np.uint32)
    table = (b | (sg << 16)).astype(np.uint32)
    ent, cnt = run(hook, table, s, tile)
    check(table, s, ent, cnt, tile)


def test_schedule_from_operator_draw(hook, oracle):
    """Buckets/signs of a real draw (oracle protocol, bit-exact with the device table)."""
    s, m = 4096, 2 * T
    op = oracle.draw("countsketch", s, m, 9000003)
    table = (op.bucket.astype(np.uint32) | ((op.signs > 0).astype(np.uint32) << 16)).astype(np.uint32)
    ent, cnt = run(hook, table, s)
    check(table, s, ent, cnt)


def test_schedule_rejects_oversized_s(hook):
    table = np.zeros(T, dtype=np.uint32)
    assert hook(table.ctypes.data, 1, T, 5000, None, None) == -1
    assert hook(table.ctypes.data, 1, 4100, 4096, None, None) == -1  # rows beyond the 12-bit field


def test_degenerate_tile_falls_back(hook):
    # every row in one bucket: one lane would need 4096 iterations -> no schedule (stream kernel instead)
    table = np.full(T, 7, dtype=np.uint32)
    assert hook(table.ctypes.data, 1, T, 4096, None, None) == -1
