"""Host-buffer end-to-end pieces (default configs[1]: m = 2^20, n = 256, SRHT s = 1024): wall time of
nsk_apply_host / nsk_solve_k_host from pageable and pinned memory, and of the draw alone.
usage: python tools/e2e_parts.py [kind m n s]"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_00975_b200 as nsk  # noqa: E402
from paper_2206_00975_b200 import _lib  # noqa: E402

L = _lib.load()
kind = sys.argv[1] if len(sys.argv) > 1 else "srht"
m, n, s = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (1 << 20, 256, 1024)
k = 1
pin = torch.empty((n, m), dtype=torch.float64, pin_memory=True).t()
pin.copy_(torch.randn(n, m, dtype=torch.float64, device="cuda").t())
page = np.asfortranarray(pin.numpy().copy())
SA = np.empty((s, n), order="F")
W = np.empty((n, k), order="F")
sig = np.empty(n)


def wall(fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


S = nsk.SketchOperator.draw(kind, s, m, 9)
for name, ptr in (("pageable", page.ctypes.data), ("pinned", pin.data_ptr())):
    ta = wall(lambda: _lib.check(L.nsk_apply_host(S.handle, 0, m, n, ctypes.c_void_p(ptr), m,
                                                  SA.ctypes.data_as(ctypes.c_void_p), s)))
    ts = wall(lambda: _lib.check(L.nsk_solve_k_host(S.handle, 0, m, n, ctypes.c_void_p(ptr), m, k,
                                                    W.ctypes.data_as(ctypes.c_void_p), n,
                                                    sig.ctypes.data_as(ctypes.c_void_p))))
    print(f"{kind} {name:9s} apply_host {ta:8.2f} ms   solve_k_host {ts:8.2f} ms", flush=True)
d = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
torch.cuda.synchronize()
print(f"{kind} torch pinned copy alone {wall(lambda: (d.copy_(pin, non_blocking=True), torch.cuda.synchronize())):.2f} ms")
