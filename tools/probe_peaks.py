"""Measure FP64 peaks on the B200 box: cuBLAS DGEMM (torch.matmul fp64) and copy bandwidth.

Writes gpurun_out/fp64_peaks.json. Used once to fill the FP64 roofline denominator
(MEASURED_PEAKS.json has only HBM and bf16)."""
import json, os, time, torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda:0")
out = {"gpu": torch.cuda.get_device_name(0), "sm_count": torch.cuda.get_device_properties(0).multi_processor_count,
       "cpu_count": os.cpu_count()}
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best
for N in (4096, 8192):
    a = torch.randn(N, N, dtype=torch.float64, device=dev); b = torch.randn(N, N, dtype=torch.float64, device=dev)
    t = timeit(lambda: torch.matmul(a, b))
    out[f"dgemm_{N}_tflops"] = 2 * N**3 / t / 1e12
# tall-skinny shaped like the sketch: (s x m) @ (m x n)
for (s, m, n) in ((1024, 1 << 20, 512), (400, 20000, 100)):
    g = torch.randn(s, m, dtype=torch.float64, device=dev); a = torch.randn(m, n, dtype=torch.float64, device=dev)
    t = timeit(lambda: torch.matmul(g, a))
    out[f"dgemm_{s}x{m}x{n}_tflops"] = 2 * s * m * n / t / 1e12
    del g, a
x = torch.empty(1 << 30, dtype=torch.float64, device=dev); y = torch.empty_like(x)
t = timeit(lambda: y.copy_(x))
out["copy_gbs"] = 2 * x.numel() * 8 / t / 1e9
t = timeit(lambda: x.sum())
out["read_gbs"] = x.numel() * 8 / t / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
print(json.dumps(out))
