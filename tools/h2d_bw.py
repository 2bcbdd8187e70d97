"""Pinned host -> device copy bandwidth (2 GiB), single copy vs 4 concurrent chunks."""
import time
import torch
n = 1 << 28
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print("single copy GB/s", n * 8 / dt / 1e9, "ms", dt * 1e3)
ss = [torch.cuda.Stream() for _ in range(4)]
t = time.perf_counter()
for _ in range(3):
    q = n // 4
    for i, s in enumerate(ss):
        with torch.cuda.stream(s):
            d[i * q:(i + 1) * q].copy_(h[i * q:(i + 1) * q], non_blocking=True)
    torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print("4 streams GB/s", n * 8 / dt / 1e9, "ms", dt * 1e3)
