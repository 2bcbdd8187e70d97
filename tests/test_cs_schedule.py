"""CountSketch owner schedule (cs_schedule.cpp), checked on the host.

The schedule is a pure function of the operator's buckets and signs; these
tests call the library's test hook on synthetic tables and check that every
row is scheduled exactly once, to the thread that owns its bucket, with its
slot and sign, that every half-warp iteration reads 16 distinct shared-memory
bank pairs, and that the iteration count of every warp is the Koenig optimum
(the largest vertex degree of its two half-warp graphs).
"""
import ctypes

import numpy as np
import pytest

from paper_2206_00975_b200 import _lib

T, THREADS, WARPS = 3072, 1024, 32


@pytest.fixture(scope="module")
def hook():
    from paper_2206_00975_b200 import build
    build.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    f = L.nsk_internal_cs_schedule
    f.restype = ctypes.c_longlong
    f.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_longlong,
                  ctypes.c_void_p]
    return f


def run(hook, table, s, T=T):
    ntiles = table.size // T
    off = np.zeros(ntiles + 1, dtype=np.uint64)
    size = hook(table.ctypes.data, ntiles, T, s, None, 0, off.ctypes.data)
    assert size > 0
    sec = np.zeros(size, dtype=np.uint8)
    assert hook(table.ctypes.data, ntiles, T, s, sec.ctypes.data, size, off.ctypes.data) == size
    return sec, off


def check(table, s, sec, off, T=T):
    ntiles = table.size // T
    for t in range(ntiles):
        tab = table[t * T:(t + 1) * T]
        b_all = tab & 0xFFFF
        part = sec[int(off[t]):int(off[t + 1])].view(np.uint16)
        assert part.size % 8 == 0  # 16-byte multiple
        hdr = part[:64].astype(np.int64)
        total = hdr[WARPS]
        ent = part[64:].reshape(total, 32)
        seen = np.zeros(T, dtype=np.int64)
        for w in range(WARPS):
            i0, i1 = hdr[w], (hdr[w + 1] if w + 1 < WARPS else total)
            blk = ent[i0:i1]
            for it in range(blk.shape[0]):
                for h in range(2):
                    e = blk[it, 16 * h:16 * h + 16]
                    valid = (e & 0x8000) != 0
                    r = (e & 0xFFF).astype(np.int64)
                    assert len(set((r[valid] & 15).tolist())) == int(valid.sum())  # distinct bank pairs
                    assert len(set((r & 15).tolist())) == 16  # idle lanes read unused bank pairs
                    assert np.all(e[~valid] < 16)
                    for lane in np.nonzero(valid)[0]:
                        row = int(r[lane])
                        b = int(b_all[row])
                        assert b % THREADS == 32 * w + 16 * h + lane
                        assert (int(e[lane]) >> 12) & 3 == b // THREADS
                        assert (int(e[lane]) >> 14) & 1 == 1 - ((int(tab[row]) >> 16) & 1)  # negative flag
                        seen[row] += 1
            # Koenig optimum: iterations = max degree over both half-warp graphs
            mine = np.nonzero((b_all % THREADS) // 32 == w)[0]
            deg = 0
            for h in range(2):
                sub = mine[((b_all[mine] % 32) >> 4) == h]
                if sub.size:
                    deg = max(deg, np.bincount(b_all[sub] % 16, minlength=16).max(),
                              np.bincount(sub & 15, minlength=16).max())
            assert i1 - i0 == deg
        assert np.all(seen == 1)


@pytest.mark.parametrize("s,ntiles,seed,tile", [(4096, 2, 1, 3072), (3000, 1, 2, 3072), (1024, 1, 3, 3072),
                                                (2048, 1, 4, 3072), (4096, 1, 5, 4096)])
def test_schedule_covers_rows_once_conflict_free_and_optimal(hook, s, ntiles, seed, tile):
    rng = np.random.default_rng(seed)
    b = rng.integers(0, s, size=ntiles * tile, dtype=np.uint32)
    sg = rng.integers(0, 2, size=ntiles * tile, dtype=np.uint32)
    table = (b | (sg << 16)).astype(np.uint32)
    sec, off = run(hook, table, s, tile)
    check(table, s, sec, off, tile)


def test_schedule_from_operator_draw(hook, oracle):
    """Buckets/signs of a real draw (oracle protocol, bit-exact with the device table)."""
    s, m = 4096, 2 * T
    op = oracle.draw("countsketch", s, m, 9000003)
    table = (op.bucket.astype(np.uint32) | ((op.signs > 0).astype(np.uint32) << 16)).astype(np.uint32)
    sec, off = run(hook, table, s)
    check(table, s, sec, off)


def test_schedule_rejects_oversized_s(hook):
    table = np.zeros(T, dtype=np.uint32)
    assert hook(table.ctypes.data, 1, T, 5000, None, 0, None) == -1
    assert hook(table.ctypes.data, 1, 4100, 4096, None, 0, None) == -1  # rows beyond the 12-bit field


def test_degenerate_tile_falls_back(hook):
    # every row in one bucket: one lane would need 4096 iterations -> no schedule (stream kernel instead)
    table = np.full(T, 7, dtype=np.uint32)
    assert hook(table.ctypes.data, 1, T, 4096, None, 0, None) == -1
