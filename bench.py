"""bench.py -- sketch throughput of the B200 hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--kind srht|srdct|srft|countsketch|gaussian|cfg0|cfg4]

Default workload = BASELINE.json configs[1] (the config the metric is quoted
on that fits one GPU): SRHT, A fp64 m = 2^20 x n = 256, U diag(sigma) V^T with
sigma logspaced 1 -> 1e-3 and the trailing k = 4 values 1e-12, s = 4n = 1024.
Other kinds: configs[2] (countsketch), configs[3] (gaussian, one GPU's share of
[A b]), configs[0] (cfg0), configs[4] (cfg4, complex Loewner), and the
configs[1] shape through the reference's own transform kinds (srdct, srft).

A "step" is one application of the sketch to the whole resident A (S A -> SA,
s x n).  value = rows of A sketched per second, whole job (N GPUs row-shard A:
weak scaling, m per GPU fixed; the s x n partials are summed with an NCCL
all-reduce, the only exchange the path has).  A is >= 2 GiB per GPU at the
HBM-bound configs, far above the 126 MB L2, so no flush is needed between
steps (cfg0/cfg4 are FP64-tensor bound and L2-resident by construction).

Keys beyond the base contract:
  roofline      dominant kernel (name reported by the library): algorithmic
                bytes (read A once + write SA) or flops (2 s m n, x2 complex)
                / its CUDA-event time inside the timed steps, against
                MEASURED_PEAKS.json hbm_gbs, or the measured FP64 DMMA peak
  e2e           the user's call, per step: nsk_op_draw + nsk_solve_k_host +
                nsk_op_destroy with A in pinned host memory (the bench
                contract): draw, H2D, sketch, SVD, D2H of W and sigma.
                e2e.pageable repeats it from ordinary malloc'd memory (the
                reference's callers hold plain Eigen buffers).
  cpu_baseline  the oracle port (oracle/, C + NumPy/SciPy) on this host's
                cores: draw / apply / SVD separately, median of 5, all cores
                and 1 thread (bench.cpp:78-88)
  breakdown     apply / SVD device milliseconds
--impl reference times the reference's CPU path (the oracle restatement of
draw + apply + LAPACK SVD; the reference itself needs Eigen/FFTW and cannot be
built here) on the same config, every step in full, and prints the same line
with "impl": "reference".
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 36.86   # profiles/fp64_peaks_r01.json: DMMA-only microbenchmark (burst)
FP64_DGEMM_TFLOPS = 35.47       # cuBLAS DGEMM 8192^3 on the same box

CONFIGS = {
    # key: sketch kind, m per GPU, n, s, k, complex input, description
    "srht": dict(kind="srht", m=1 << 20, n=256, s=1024, k=4, cplx=False,
                 desc="BASELINE configs[1]: SRHT m=2^20 n=256 s=4n=1024 k=4"),
    "srdct": dict(kind="srdct", m=1 << 20, n=256, s=1024, k=4, cplx=False,
                  desc="configs[1] shape, reference-pinned analogue: SRDCT m=2^20 n=256 s=1024 k=4"),
    "srft": dict(kind="srft", m=1 << 20, n=256, s=1024, k=4, cplx=False,
                 desc="configs[1] shape, SRFT (complex output) m=2^20 n=256 s=1024 k=4"),
    "countsketch": dict(kind="countsketch", m=1 << 24, n=64, s=4096, k=1, cplx=False,
                        desc="BASELINE configs[2]: CountSketch m=2^24 n=64 s=n^2=4096 k=1"),
    "gaussian": dict(kind="gaussian", m=1 << 22, n=512, s=1024, k=1, cplx=False,
                     desc="BASELINE configs[3] per GPU: Gaussian on [A b], m=2^22 n=512 s=1024 k=1"),
    "cfg0": dict(kind="gaussian", m=20000, n=100, s=400, k=1, cplx=False,
                 desc="BASELINE configs[0]: Gaussian m=20000 n=100 s=4n=400 k=1 (CPU-runnable parity config)"),
    "cfg4": dict(kind="gaussian", m=99850, n=150, s=300, k=1, cplx=True,
                 desc="BASELINE configs[4]: complex128 Loewner m=99850 (100000 - 150 support rows) n=150, "
                      "Gaussian s=2n=300 k=1"),
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _poll(self):
        while True:
            self._sample()
            if self._stop.wait(0.01):
                break

    def _sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()
        self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def make_input(key, m, n, k, seed, device):
    """Synthetic A with the config's construction (generated on the device; not timed)."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    if key == "countsketch":
        # configs[2]: A = G P + 1e-14 E, P = I - p p^T (rank n-1), true null vector p.
        p = torch.randn(n, dtype=torch.float64, device=device, generator=g)
        p /= torch.linalg.norm(p)
        A = torch.empty((n, m), dtype=torch.float64, device=device).t()
        P = torch.eye(n, dtype=torch.float64, device=device) - torch.outer(p, p)
        step = 1 << 22
        for r0 in range(0, m, step):
            r1 = min(m, r0 + step)
            G = torch.randn(r1 - r0, n, dtype=torch.float64, device=device, generator=g)
            E = torch.randn(r1 - r0, n, dtype=torch.float64, device=device, generator=g)
            A[r0:r1] = G @ P + 1e-14 * E
        return A
    if key == "gaussian":
        # configs[3]: C = [A b], A ~ N(0,1) (n-1 cols), b = A x + 1e-3 noise.
        A = torch.empty((n, m), dtype=torch.float64, device=device).t()
        x = torch.randn(n - 1, dtype=torch.float64, device=device, generator=g)
        step = 1 << 20
        for r0 in range(0, m, step):
            r1 = min(m, r0 + step)
            blk = torch.randn(r1 - r0, n - 1, dtype=torch.float64, device=device, generator=g)
            A[r0:r1, :n - 1] = blk
            A[r0:r1, n - 1] = blk @ x + 1e-3 * torch.randn(r1 - r0, dtype=torch.float64, device=device,
                                                           generator=g)
        return A
    if key == "cfg4":
        # configs[4]: z on the unit circle (seeded uniform angles), f(z) = 1/(1.1 - z) + e^z, support
        # z_j = every (M/n)-th sample, L_ij = (F_i - f_j) / (Z_i - z_j) over the M - n active rows.
        M = m + n
        theta = 2 * math.pi * torch.rand(M, dtype=torch.float64, device=device, generator=g)
        z = torch.polar(torch.ones_like(theta), theta)
        f = 1.0 / (1.1 - z) + torch.exp(z)
        support = (torch.arange(n, device=device) * M) // n
        mask = torch.ones(M, dtype=torch.bool, device=device)
        mask[support] = False
        Z, F = z[mask], f[mask]
        L = (F[:, None] - f[None, support]) / (Z[:, None] - z[None, support])
        return L.t().contiguous().t()
    # configs[1] / configs[0]: U diag(sigma) V^T; configs[1]: logspaced 1 -> 1e-3 with the trailing k
    # at 1e-12; configs[0]: logspaced 1 -> 1e-3 over n-1 values and sigma_n = 1e-10.
    G = torch.randn((n, m), dtype=torch.float64, device=device, generator=g).t()
    U, _ = torch.linalg.qr(G)
    del G
    V, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device=device, generator=g))
    if key == "cfg0":
        sig = torch.cat([torch.logspace(0, -3, n - 1, dtype=torch.float64, device=device),
                         torch.full((1,), 1e-10, dtype=torch.float64, device=device)])
    else:
        sig = torch.cat([torch.logspace(0, -3, n - k, dtype=torch.float64, device=device),
                         torch.full((k,), 1e-12, dtype=torch.float64, device=device)])
    A = ((U * sig) @ V.t()).t().contiguous().t()
    del U
    return A


def algorithmic(cfg, m):
    """(bytes, flops) per apply: read A once + write SA; S is regenerated (0 bytes);
    flops 2 s m n for the Gaussian GEMM, x2 for complex A against the real G."""
    kind, n, s, cplx = cfg["kind"], cfg["n"], cfg["s"], cfg["cplx"]
    elem_in = 16 if cplx else 8
    out_elem = 16 if (kind == "srft" or cplx) else 8
    byts = m * n * elem_in + s * n * out_elem
    flops = 2 * s * m * n * (2 if cplx else 1) if kind == "gaussian" else 0
    return byts, flops


# ----------------------------------------------------------------------------- CPU side (oracle port)

def _median5(fn, reps=5):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def cpu_leg(cfg, A, threads, reps=5, ncols=None):
    """Oracle port of the reference's draw, apply and SVD (bench.cpp:78-88 median of 5) on `threads`
    host threads over A (m_sample x ncols).  Returns seconds for draw, apply, SVD."""
    import numpy as np
    from oracle import sketch_oracle as O
    kind, s, k = cfg["kind"], cfg["s"], cfg["k"]
    m = A.shape[0]
    ncols = ncols or A.shape[1]
    Ac = A[:, :ncols]
    box = {}

    def draw():
        box["op"] = O.draw(kind, s, m, 9000002)

    def apply():
        op = box["op"]
        if kind == "srht":
            SA = np.zeros((s, ncols), order="F")
            O.lib().nsko_srht_apply(O._p(op.signs, O._dp), O._p(op.idx, O._ip), s, m, ncols, O._p(Ac, O._dp), m,
                                    O._p(SA, O._dp), s, 0, ncols, threads)
        elif kind == "countsketch":
            SA = np.zeros((s, ncols), order="F")
            O.lib().nsko_countsketch_apply_tables(O._p(op.bucket, O._i32p), O._p(op.signs, O._dp), s, m, ncols,
                                                  O._p(Ac, O._dp), m, O._p(SA, O._dp), s, threads)
        elif kind == "srdct":
            import scipy.fft
            SA = math.sqrt(m / s) * scipy.fft.dct(op.signs[:, None] * Ac, type=3, norm="ortho", axis=0,
                                                  workers=threads)[op.idx]
        elif kind == "srft":
            import scipy.fft
            SA = math.sqrt(m / s) * scipy.fft.ifft(op.signs[:, None] * Ac.astype(np.complex128), axis=0,
                                                   norm="ortho", workers=threads)[op.idx]
        else:  # gaussian: G regenerated by column blocks on `threads` threads, BLAS GEMM
            SA = np.zeros((s, ncols), dtype=Ac.dtype)
            blk = max(1, min(m, (1 << 24) // s))
            for j0 in range(0, m, blk):
                j1 = min(m, j0 + blk)
                G = O.gaussian_block(9000002, s, j0, j1, nthreads=threads)
                if np.iscomplexobj(Ac):
                    SA += G @ Ac[j0:j1].real + 1j * (G @ Ac[j0:j1].imag)
                else:
                    SA += G @ Ac[j0:j1]
            SA /= math.sqrt(s)
        box["SA"] = SA

    def svd():
        O.from_sketch_svd(box["SA"], k)

    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=threads)
    except Exception:
        limiter = None
    try:
        t_draw = _median5(draw, reps)
        t_apply = _median5(apply, reps)
        t_svd = _median5(svd, reps) if ncols == cfg["n"] else None
    finally:
        if limiter is not None:
            limiter.restore_original_limits()
    return t_draw, t_apply, t_svd


def cpu_plan(key, cfg):
    """Bounded sample per host-thread count (~10-30 s of CPU work in total): (m_sample, ncols_all, ncols_one)."""
    m, n = cfg["m"], cfg["n"]
    if key == "srht":
        return m, n, n                   # full config on both legs (1 thread ~5 s per apply)
    if key in ("srdct", "srft"):
        return m, n, 32                  # 1 thread: 32 of the n columns (columns are independent)
    if key == "countsketch":
        return m, n, 16
    if key == "gaussian":
        return 1 << 15, n, n             # G regeneration + GEMM are linear in m: 2^15-row sample
    return m, n, n                       # cfg0 / cfg4: full


def cpu_baseline(key, cfg):
    import numpy as np
    threads = os.cpu_count() or 1
    m_s, nc_all, nc_one = cpu_plan(key, cfg)
    rng = np.random.default_rng(7)
    if cfg["cplx"]:
        A = np.asfortranarray(rng.standard_normal((m_s, cfg["n"])) + 1j * rng.standard_normal((m_s, cfg["n"])))
    else:
        A = np.asfortranarray(rng.standard_normal((m_s, cfg["n"])))
    out = {}
    for label, th, nc in (("all_cores", threads, nc_all), ("one_thread", 1, nc_one)):
        d, a, v = cpu_leg(cfg, A, th, ncols=nc)
        rows_per_s = m_s / a * (nc / cfg["n"])   # apply is column-separable: rate for all n columns
        out[label] = {"threads": th, "rows": m_s, "columns": nc, "draw_s": round(d, 5), "apply_s": round(a, 5),
                      "svd_s": None if v is None else round(v, 5), "apply_rows_per_s": rows_per_s}
    al = out["all_cores"]
    sample = (f"oracle port, median of 5: draw + apply + SVD of {al['rows']} x {al['columns']} rows x columns on "
              f"{threads} threads; 1 thread on {out['one_thread']['rows']} x {out['one_thread']['columns']}"
              + (" (column sample: rows/s scaled by n / columns)" if out["one_thread"]["columns"] < cfg["n"] else "")
              + (f" (row sample of the m = {cfg['m']} config)" if m_s < cfg["m"] else ""))
    return {"value": al["apply_rows_per_s"], "unit": "rows/s", "cores": threads, "kind": "port",
            "sample": sample, **out}


# ----------------------------------------------------------------------------- GPU arm

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2206_00975_b200 as nsk
    from paper_2206_00975_b200 import _lib

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    key = args.kind
    cfg = CONFIGS[key]
    kind, mloc, n, s, k = cfg["kind"], cfg["m"], cfg["n"], cfg["s"], cfg["k"]
    m_glob = mloc * world
    L = _lib.load()
    S = nsk.SketchOperator.draw(kind, s, m_glob, 9000002)
    A = make_input(key, mloc, n, k, 1234 + rank, dev)
    stream = torch.cuda.current_stream()
    comm = shard = None
    # N > 1 (or NSK_BENCH_SHARDED=1 on one GPU, to exercise it): the library's own NCCL path
    # (nsk_apply_allreduce: partial + ncclAllReduce in one call)
    sharded = world > 1 or os.environ.get("NSK_BENCH_SHARDED") == "1"
    if sharded:
        from paper_2206_00975_b200.distributed import NcclComm, RowShard, sharded_apply_nccl
        comm = NcclComm()
        # srft / srdct: cyclic shards (decimation in time); the others: contiguous row blocks
        shard = RowShard(rank, world, mloc) if kind in ("srft", "srdct") else RowShard(rank * mloc, 1, mloc)

    def step():
        if not sharded:
            return nsk.apply(S, A).data
        return sharded_apply_nccl(S, A, shard, comm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps, barrier + sync on both sides, max over ranks.
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.nsk_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # dominant-kernel time: the library records CUDA events around that kernel
    # only, on the stream it launches on, during these same K timed steps
    L.nsk_timing_collect(None, None)
    L.nsk_timing_enable(1)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            SA = step()
        e1.record(stream)
        torch.cuda.synchronize()
    L.nsk_timing_enable(0)
    launches = L.nsk_kernel_launches() - launches0
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = tt.item()
        dist.barrier()
    ms_per_step = t_ms / args.steps
    value = m_glob * args.steps / (t_ms / 1e3)

    tot = np.zeros(1)
    cnt = np.zeros(1, dtype=np.int64)
    L.nsk_timing_collect(tot.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                         cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    kname = (L.nsk_timing_kernel() or b"").decode()
    kernel_ms = float(tot[0] / max(cnt[0], 1))
    kernels_per_step = float(cnt[0]) / args.steps
    byts, flops = algorithmic(cfg, mloc)
    # per launch: a step may run the dominant kernel more than once (e.g. the pipelined chunks)
    byts_l, flops_l = byts / max(kernels_per_step, 1.0), flops / max(kernels_per_step, 1.0)
    hbm_peak, peak_src = measured_peaks()
    if kind == "gaussian":
        achieved = flops_l / (kernel_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_DMMA_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": round(achieved / FP64_DMMA_PEAK_TFLOPS, 4),
                "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peaks_r01.json); "
                               f"cuBLAS DGEMM {FP64_DGEMM_TFLOPS} TF/s"}
    else:
        achieved = byts_l / (kernel_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
    roof.update({"kernel": kname, "kernel_ms": round(kernel_ms, 4), "kernels_per_step": kernels_per_step,
                 "algorithmic_bytes": int(byts_l), "algorithmic_flops": int(flops_l),
                 "traffic": traffic_from_profiles(key, kname)})

    # ---- breakdown: SVD device time (rank 0's view).
    SA = step()
    nsk.svd_trailing(SA, k)  # warm: first-launch module loading and scratch-pool growth stay out
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    W, sig = nsk.svd_trailing(SA, k)
    t1.record(stream)
    torch.cuda.synchronize()
    svd_ms = t0.elapsed_time(t1)

    # ---- e2e through the C ABI with host buffers (rank-local shard on N > 1).
    e2e = e2e_measure(nsk, cfg, A, args, world, rank, mloc, comm)
    del A
    torch.cuda.empty_cache()

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline(key, cfg)
        clocks = clk.summary()
        result = {
            "metric": "rows of A sketched/s", "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cfg["cplx"] else "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "kind": kind, "m_per_gpu": mloc, "m_total": m_glob, "n": n, "s": s,
                       "k": k, "l2": ("A is %.2f GiB per GPU (%s 126 MB L2)%s" % (
                           byts / 2**30, ">" if byts > 126e6 else "<",
                           ": no flush needed" if byts > 126e6 else
                           ": L2-resident; FP64-tensor bound, S regenerated per tile")),
                       "parallelism": f"row-shard x{world}" + (" + NCCL all-reduce of s x n" if world > 1 else "")},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks,
            "breakdown": {"apply_ms": round(ms_per_step, 4), "svd_ms": round(svd_ms, 3),
                          "hbm_gbs_step": round(byts / (ms_per_step / 1e3) / 1e9, 1)},
        }
    if comm is not None:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def e2e_measure(nsk, cfg, A, args, world, rank, mloc, comm=None):
    """The user's call per step: nsk_op_draw + nsk_solve_k_host + nsk_op_destroy, A in host memory
    (pinned; and pageable, the reference callers' Eigen buffers, as a sub-key), W and sigma back in host memory."""
    import numpy as np
    import torch
    from paper_2206_00975_b200 import _lib
    L = _lib.load()
    kind, n, s, k = cfg["kind"], cfg["n"], cfg["s"], cfg["k"]
    steps = max(1, min(args.steps, args.e2e_steps))
    dt = torch.complex128 if cfg["cplx"] else torch.float64
    Ah_pin = torch.empty((n, mloc), dtype=dt, pin_memory=True).t()
    Ah_pin.copy_(A)
    if comm is not None:
        return e2e_sharded(nsk, cfg, Ah_pin, steps, rank, mloc, comm)
    Ah_page = np.asfortranarray(Ah_pin.numpy().copy())  # ordinary malloc'd host memory
    cplx_out = kind == "srft" or cfg["cplx"]
    W = np.empty((n, k), dtype=np.complex128 if cplx_out else np.float64, order="F")
    sig = np.empty(n)
    scalar = 1 if cfg["cplx"] else 0

    def one(ptr):
        h = ctypes.c_void_p()
        _lib.check(L.nsk_op_draw(_lib.KIND_CODES[kind], s, mloc, 9000002, ctypes.byref(h)))
        try:
            _lib.check(L.nsk_solve_k_host(h, scalar, mloc, n, ctypes.c_void_p(ptr), mloc, k,
                                          W.ctypes.data_as(ctypes.c_void_p), n, sig.ctypes.data_as(ctypes.c_void_p)))
        finally:
            L.nsk_op_destroy(h)

    def timed(ptr):
        one(ptr)  # warm: staging ring, scratch pool, module load
        t0 = time.perf_counter()
        for _ in range(steps):
            one(ptr)
        return (time.perf_counter() - t0) / steps

    t_page = timed(Ah_page.ctypes.data)
    t_pin = timed(Ah_pin.data_ptr())
    bi = mloc * n * (16 if cfg["cplx"] else 8)
    bo = W.nbytes + sig.nbytes
    tls = None
    if kind == "gaussian" and not cfg["cplx"] and n == 512:
        # configs[3] is a total-least-squares problem: the same call as the reference's tls command
        # (tls_solve_sketched, tls.cpp:97-113) on [A | b] = the first 511 and the last column
        X = np.empty((n - 1, 1), order="F")
        Vk = np.empty((n, 1), order="F")
        sg = np.empty(n)
        info = np.zeros(4)

        def tls_one(ptr):
            h = ctypes.c_void_p()
            _lib.check(L.nsk_op_draw(_lib.KIND_CODES[kind], s, mloc, 9000002, ctypes.byref(h)))
            try:
                _lib.check(L.nsk_tls_solve_sketched_host(
                    h, 0, mloc, n - 1, 1, ctypes.c_void_p(ptr), mloc, ctypes.c_void_p(ptr + 8 * mloc * (n - 1)), mloc,
                    1e12, 1, X.ctypes.data_as(ctypes.c_void_p), n - 1, Vk.ctypes.data_as(ctypes.c_void_p), n,
                    sg.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
            finally:
                L.nsk_op_destroy(h)
        tls_one(Ah_page.ctypes.data)
        t0 = time.perf_counter()
        for _ in range(steps):
            tls_one(Ah_page.ctypes.data)
        t_tls = (time.perf_counter() - t0) / steps
        tls = {"value": mloc / t_tls, "unit": "rows/s", "ms": round(t_tls * 1e3, 3),
               "api": "nsk_op_draw + nsk_tls_solve_sketched_host + nsk_op_destroy on [A | b] in pageable memory "
                      "(one-pass S [A | b], both SVDs, X = -V_k1 V_k2^{-1})"}
    # headline: A in pinned host memory (the bench contract's e2e); the same call from pageable
    # memory (the reference callers' Eigen buffers) is reported beside it
    return {"value": mloc / t_pin, "unit": "rows/s", "ms": round(t_pin * 1e3, 3), "steps": steps,
            "api": "nsk_op_draw + nsk_solve_k_host + nsk_op_destroy (draw and device tables, H2D of A from "
                   "pinned (cudaHostAlloc) host memory in row chunks, each chunk sketched as it lands, "
                   "QR + Jacobi SVD, D2H of W and sigma); host wall clock",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
            "pageable": {"value": mloc / t_page, "unit": "rows/s", "ms": round(t_page * 1e3, 3),
                         "api": "same call with A in ordinary malloc'd host memory (packed into the library's "
                                "pinned staging ring by host threads, then the same pipeline)"},
            **({"tls": tls} if tls else {})}


def e2e_sharded(nsk, cfg, Ah, steps, rank, mloc, comm):
    """N > 1: the user's call on every rank, per step: nsk_op_draw + nsk_solve_k_sharded_host on the
    rank's row shard in host memory (pinned, and pageable as a sub-key) -- the library's pipelined
    host path (row chunks sketched as they land), then ncclAllReduce of the s x n partials and the
    Jacobi SVD on every rank, W and sigma back in host memory; host wall clock, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2206_00975_b200 import _lib
    from paper_2206_00975_b200.distributed import RowShard
    L = _lib.load()
    kind, n, s, k = cfg["kind"], cfg["n"], cfg["s"], cfg["k"]
    world = dist.get_world_size() if dist.is_initialized() else 1
    shard = RowShard(rank, world, mloc) if kind in ("srft", "srdct") else RowShard(rank * mloc, 1, mloc)
    Ah_page = np.asfortranarray(Ah.numpy().copy())
    cplx_out = kind == "srft" or cfg["cplx"]
    W = np.empty((n, k), dtype=np.complex128 if cplx_out else np.float64, order="F")
    sig = np.empty(n)
    scalar = 1 if cfg["cplx"] else 0

    def one(ptr):
        h = ctypes.c_void_p()
        _lib.check(L.nsk_op_draw(_lib.KIND_CODES[kind], s, world * mloc, 9000002, ctypes.byref(h)))
        try:
            _lib.check(L.nsk_solve_k_sharded_host(h, scalar, shard.row0, shard.rstep, mloc, n, ctypes.c_void_p(ptr),
                                                  mloc, k, W.ctypes.data_as(ctypes.c_void_p), n,
                                                  sig.ctypes.data_as(ctypes.c_void_p), comm.handle))
        finally:
            L.nsk_op_destroy(h)

    def timed(ptr):
        one(ptr)  # warm: staging ring, scratch pool, tables
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one(ptr)
        dt = (time.perf_counter() - t0) / steps
        t = torch.tensor([dt], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    t_page = timed(Ah_page.ctypes.data)
    t_pin = timed(Ah.data_ptr())
    api = ("nsk_op_draw + nsk_solve_k_sharded_host on the rank's row shard (H2D of the shard in row chunks "
           "in row chunks, each chunk sketched as it lands, ncclAllReduce of the s x n partials, "
           "Jacobi SVD on every rank, D2H of W and sigma); host wall clock, max over ranks")
    return {"value": world * mloc / t_pin, "unit": "rows/s", "ms": round(t_pin * 1e3, 3), "steps": steps,
            "api": api + " -- the shard in pinned (cudaHostAlloc) host memory",
            "h2d_bytes_per_step": world * mloc * n * Ah.element_size(),
            "d2h_bytes_per_step": int(W.nbytes + sig.nbytes),
            "pageable": {"value": world * mloc / t_page, "unit": "rows/s", "ms": round(t_page * 1e3, 3),
                         "api": "same call with the shard in ordinary malloc'd host memory"}}


def traffic_from_profiles(key, kname):
    """DRAM bytes (read + write) per launch of the dominant kernel from the newest committed
    `ncu --set full` capture of this config (profiles/r*_<key>_ncu.json) when it profiled the same
    kernel, else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{key}_ncu.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        d = json.load(f)
    e = d[0] if isinstance(d, list) and d else d
    if kname and e.get("kernel") and kname not in str(e["kernel"]):
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def nbytes(v):  # ncu_summary stores [value, unit]
        if isinstance(v, (list, tuple)):
            return float(v[0]) * scale.get(v[1], 1.0)
        return float(v)
    try:
        return int(nbytes(e["dram__bytes_read.sum"]) + nbytes(e["dram__bytes_write.sum"]))
    except (KeyError, TypeError, ValueError):
        return None


# ----------------------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's CPU path on this host: each step is the reference's solve with its draw
    (SketchOperator::draw + solve_k = apply + SVD, nullsketch_main.cpp:134-163) in full, on all host
    threads (the restatement, oracle/: Eigen/FFTW are absent)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return None
    key = args.kind
    cfg = CONFIGS[key]
    kind, n, s, k = cfg["kind"], cfg["n"], cfg["s"], cfg["k"]
    import numpy as np
    from oracle import sketch_oracle as O
    threads = os.cpu_count() or 1
    O.build()
    # the gaussian configs[3] step is ~20 s of CPU work: a 2^18-row sample per step (rate is linear in m)
    m = cfg["m"] if key != "gaussian" else 1 << 18
    rng = np.random.default_rng(7)
    if cfg["cplx"]:
        A = np.asfortranarray(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    else:
        A = np.asfortranarray(rng.standard_normal((m, n)))
    times = {"draw": [], "apply": [], "svd": []}

    def step(record):
        t0 = time.perf_counter()
        d, a, v = cpu_leg(cfg, A, threads, reps=1)
        if record:
            times["draw"].append(d)
            times["apply"].append(a)
            times["svd"].append(v)

    for _ in range(args.warmup):
        step(False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(True)
    wall = time.perf_counter() - t0
    apply_s = statistics.mean(times["apply"])
    total_s = statistics.mean(a + b + c for a, b, c in zip(times["draw"], times["apply"], times["svd"]))
    value = m / apply_s
    sample = (f"oracle port of draw + apply ({kind}) + LAPACK SVD, m={m} x n={n}, every step in full, "
              f"{threads} threads" + (f" (row sample of m = {cfg['m']})" if m < cfg["m"] else ""))
    return {"metric": "rows of A sketched/s", "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": apply_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cfg["cplx"] else "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg["desc"], "kind": kind, "m_per_gpu": cfg["m"], "m_timed": m, "n": n, "s": s,
                       "k": k},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": m / total_s, "unit": "rows/s", "ms": round(total_s * 1e3, 3),
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "api": "draw + apply + SVD (the reference's nullspace path), host memory"},
            "breakdown": {"draw_ms": round(statistics.mean(times["draw"]) * 1e3, 3),
                          "apply_ms": round(apply_s * 1e3, 3),
                          "svd_ms": round(statistics.mean(times["svd"]) * 1e3, 3),
                          "timed_region_s": round(wall, 3)},
            "note": "reference C++ needs Eigen 3.4 + FFTW3 (absent): its restatement (oracle/) is timed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="srht", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
