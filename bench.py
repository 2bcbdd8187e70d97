"""bench.py -- sketch throughput of the B200 hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--kind srht|srdct|srft|gaussian|countsketch]

Default workload = BASELINE.json configs[1] (the config the metric is quoted
on that fits one GPU): SRHT, A fp64 m = 2^20 x n = 256, U diag(sigma) V^T with
sigma logspaced 1 -> 1e-3 and the trailing k = 4 values 1e-12, s = 4n = 1024.
A "step" is one application of the sketch to the whole resident A (S A ->
SA, s x n).  value = rows of A sketched per second, whole job (N GPUs row-
shard A: weak scaling, m per GPU fixed; the s x n partials are summed with an
NCCL all-reduce, the only exchange the path has).  A is 2 GiB per GPU, far
above the 126 MB L2, so no L2 flush is needed between steps.

Keys beyond the base contract:
  roofline      dominant kernel: algorithmic bytes (read A once + write SA)
                / CUDA-event kernel time, against MEASURED_PEAKS.json hbm_gbs
                (FP64 TF/s against the measured DMMA peak for gaussian)
  cpu_baseline  the oracle port (oracle/, C + NumPy) on this host's cores
  e2e           solve_k through the C ABI with host buffers: pinned H2D of A,
                sketch, on-device Jacobi SVD, D2H of W and sigma, per step
  breakdown     apply / SVD / solve_k device milliseconds
--impl reference times the reference's CPU path (the oracle restatement of
apply + LAPACK SVD; the reference itself needs Eigen/FFTW and cannot be
built here) on the same config and prints the same line with "impl".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 36.86   # profiles/fp64_peaks_r01.json: DMMA-only microbenchmark (burst)
FP64_DGEMM_TFLOPS = 35.47       # cuBLAS DGEMM 8192^3 on the same box

CONFIGS = {
    # kind: (m per GPU, n, s, k, description)
    "srht": (1 << 20, 256, 1024, 4, "BASELINE configs[1]: SRHT m=2^20 n=256 s=4n=1024 k=4"),
    "srdct": (1 << 20, 256, 1024, 4, "configs[1] shape, pinned analogue: SRDCT m=2^20 n=256 s=1024 k=4"),
    "srft": (1 << 20, 256, 1024, 4, "configs[1] shape, SRFT (complex output) m=2^20 n=256 s=1024 k=4"),
    "countsketch": (1 << 24, 64, 4096, 1, "BASELINE configs[2]: CountSketch m=2^24 n=64 s=n^2=4096 k=1"),
    "gaussian": (1 << 22, 512, 1024, 1, "BASELINE configs[3] per GPU: Gaussian on [A b], m=2^22 n=512 s=1024 k=1"),
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


def make_input(kind, m, n, k, seed, device):
    """Synthetic A with the config's construction (generated on the device; not timed)."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    if kind == "countsketch":
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
    if kind == "gaussian":
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
    # configs[1]: U diag(sigma) V^T, trailing k singular values 1e-12.
    G = torch.randn((n, m), dtype=torch.float64, device=device, generator=g).t()
    U, _ = torch.linalg.qr(G)
    del G
    V, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device=device, generator=g))
    sig = torch.logspace(0, -3, n - k, dtype=torch.float64, device=device)
    sig = torch.cat([sig, torch.full((k,), 1e-12, dtype=torch.float64, device=device)])
    A = ((U * sig) @ V.t()).t().contiguous().t()
    del U
    if kind == "srft":
        return A
    return A


def algorithmic(kind, m, n, s):
    """(bytes, flops) per apply: read A once + write SA; S is regenerated (0 bytes)."""
    elem_in = 8
    out_elem = 16 if kind == "srft" else 8
    byts = m * n * elem_in + s * n * out_elem
    flops = 2 * s * m * n if kind == "gaussian" else 0
    return byts, flops


# ----------------------------------------------------------------------------- CPU side

def cpu_time_apply(kind, m, n, s, k, seed, budget_s=12.0, ncols=None, threads=None):
    """Oracle port of the reference's apply (+ LAPACK SVD) on this host's cores.

    Returns (rows_per_s, seconds_per_full_step, sample description, cores)."""
    import numpy as np
    from oracle import sketch_oracle as O
    threads = threads or os.cpu_count()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    ncols = ncols or n
    rng = np.random.default_rng(seed)
    op = O.draw(kind, s, m, 9000002)
    A = np.asfortranarray(rng.standard_normal((m, ncols)))
    reps, t_tot = 0, 0.0
    while t_tot < budget_s and reps < 50:
        t0 = time.perf_counter()
        if kind == "srht":
            SA = np.zeros((s, ncols), order="F")
            O.lib().nsko_srht_apply(O._p(op.signs, O._dp), O._p(op.idx, O._ip), s, m, ncols, O._p(A, O._dp), m,
                                    O._p(SA, O._dp), s, 0, ncols, threads)
        else:
            SA = O.apply(op, A)
        t_tot += time.perf_counter() - t0
        reps += 1
        if t_tot > budget_s / 2 and reps >= 1:
            break
    per_rep = t_tot / reps
    full = per_rep * (n / ncols)
    sample = f"{kind} apply, m={m}, {ncols} of {n} columns, {reps} reps, {threads} threads"
    return m / full, full, sample, threads


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
    kind = args.kind
    mloc, n, s, k, desc = CONFIGS[kind]
    m_glob = mloc * world
    L = _lib.load()
    S = nsk.SketchOperator.draw(kind, s, m_glob, 9000002)
    A = make_input(kind, mloc, n, k, 1234 + rank, dev)
    stream = torch.cuda.current_stream()
    out_dtype = torch.complex128 if kind == "srft" else torch.float64

    def step():
        if world == 1:
            return nsk.apply(S, A).data
        part = nsk.apply_shard(S, A, rank * mloc)
        dist.all_reduce(part)
        return part

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
    import ctypes
    L.nsk_timing_collect(tot.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                         cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    kernel_ms = float(tot[0] / max(cnt[0], 1))
    byts, flops = algorithmic(kind, mloc, n, s)
    hbm_peak, peak_src = measured_peaks()
    if kind == "gaussian":
        achieved = flops / (kernel_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_DMMA_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": round(achieved / FP64_DMMA_PEAK_TFLOPS, 4),
                "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peaks_r01.json); "
                               f"cuBLAS DGEMM {FP64_DGEMM_TFLOPS} TF/s"}
    else:
        achieved = byts / (kernel_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
    roof.update({"kernel": {"srht": "srht_kernel", "srdct": "srdct_tile_kernel", "srft": "srtt_tile_kernel",
                            "countsketch": "countsketch_owner_kernel", "gaussian": "gaussian_sketch_kernel"}[kind],
                 "kernel_ms": round(kernel_ms, 4), "algorithmic_bytes": byts, "algorithmic_flops": flops,
                 "traffic": traffic_from_profiles(kind)})

    # ---- breakdown: SVD and solve_k device time (rank 0's view).
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
    e2e = e2e_measure(nsk, S, A, k, kind, args, world, rank, mloc)

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            rps, full, sample, cores = cpu_time_apply(kind, mloc, n, s, k, 7, ncols=min(n, 64))
            cpu = {"value": rps, "unit": "rows/s", "cores": cores, "kind": "port", "sample": sample,
                   "seconds_per_full_step": round(full, 4)}
        clocks = clk.summary()
        result = {
            "metric": "rows of A sketched/s", "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "kind": kind, "m_per_gpu": mloc, "m_total": m_glob, "n": n, "s": s,
                       "k": k, "l2": "A is %.1f GiB per GPU (> 126 MB L2): no flush needed" % (mloc * n * 8 / 2**30),
                       "parallelism": f"row-shard x{world}" + (" + NCCL all-reduce of s x n" if world > 1 else "")},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks,
            "breakdown": {"apply_ms": round(ms_per_step, 4), "svd_ms": round(svd_ms, 3),
                          "hbm_gbs_step": round(byts / (ms_per_step / 1e3) / 1e9, 1)},
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def e2e_measure(nsk, S, A, k, kind, args, world, rank, mloc):
    """solve_k through nsk_solve_k_host: pinned host A in, W and sigma out, each step."""
    import ctypes

    import numpy as np
    import torch
    from paper_2206_00975_b200 import _lib
    L = _lib.load()
    n = A.shape[1]
    Ah = torch.empty((n, mloc), dtype=torch.float64, pin_memory=True).t()
    Ah.copy_(A)
    W = np.empty((n, k), dtype=np.complex128 if kind == "srft" else np.float64, order="F")
    sig = np.empty(n)
    steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        return e2e_sharded(nsk, S, Ah, k, kind, steps, rank, mloc)

    def one():
        rc = L.nsk_solve_k_host(S.handle, 0, mloc, n, ctypes.c_void_p(Ah.data_ptr()), mloc, k,
                                W.ctypes.data_as(ctypes.c_void_p), n, sig.ctypes.data_as(ctypes.c_void_p))
        _lib.check(rc)

    one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    bi = mloc * n * 8
    bo = W.nbytes + sig.nbytes
    return {"value": mloc / dt, "unit": "rows/s", "ms": round(dt * 1e3, 3), "steps": steps,
            "api": "nsk_solve_k_host (H2D of A from pinned memory, sketch, Jacobi SVD, D2H of W and sigma)",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo}


def e2e_sharded(nsk, S, Ah, k, kind, steps, rank, mloc):
    """N > 1: every rank copies its pinned host shard in, sketches it, the partials are
    all-reduced, rank 0 runs the SVD and W / sigma are broadcast and copied out
    (paper_2206_00975_b200.distributed.sharded_solve_k); device time, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2206_00975_b200.distributed import RowShard, sharded_solve_k
    dev = torch.device("cuda", torch.cuda.current_device())
    n = Ah.shape[1]
    Ad = torch.empty((n, mloc), dtype=torch.float64, device=dev).t()
    shard = RowShard(rank * mloc, 1, mloc)

    def one():
        Ad.copy_(Ah, non_blocking=True)
        W, sig = sharded_solve_k(S, Ad, k, shard)
        return W.cpu(), sig.cpu()

    one()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        W, sig = one()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = t.item() / 1e3
    world = dist.get_world_size()
    return {"value": world * mloc / dt, "unit": "rows/s", "ms": round(dt * 1e3, 3), "steps": steps,
            "api": "distributed.sharded_solve_k (pinned H2D of each shard, apply_shard, NCCL all-reduce, "
                   "Jacobi SVD on rank 0, broadcast, D2H of W and sigma)",
            "h2d_bytes_per_step": world * mloc * n * 8, "d2h_bytes_per_step": int(W.numel() * W.element_size()
                                                                                 + sig.numel() * 8)}


def traffic_from_profiles(kind):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    `ncu --set full` capture of this kind (profiles/r01_<kind>_ncu.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{kind}_ncu.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        d = json.load(f)
    e = d[0] if isinstance(d, list) and d else d
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
    rank, world, _ = env_rank()
    if rank != 0:
        return None
    kind = args.kind
    mloc, n, s, k, desc = CONFIGS[kind]
    import numpy as np
    from oracle import sketch_oracle as O
    threads = os.cpu_count()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    O.build()
    # bounded sample per step: ncols columns of the full m rows (the apply cost is linear in n)
    ncols = max(1, min(n, args.ref_cols))
    rng = np.random.default_rng(7)
    A = np.asfortranarray(rng.standard_normal((mloc, ncols)))
    op = O.draw(kind, s, mloc, 9000002)

    def step():
        if kind == "srht":
            SA = np.zeros((s, ncols), order="F")
            O.lib().nsko_srht_apply(O._p(op.signs, O._dp), O._p(op.idx, O._ip), s, mloc, ncols, O._p(A, O._dp),
                                    mloc, O._p(SA, O._dp), s, 0, ncols, threads)
        else:
            O.apply(op, A)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    full = dt * n / ncols
    value = mloc / full
    sample = (f"oracle port of apply ({kind}), m={mloc}, {ncols} of {n} columns per step "
              f"(rows/s scaled to all {n} columns), {threads} threads")
    return {"metric": "rows of A sketched/s", "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": full * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": desc, "kind": kind, "m_per_gpu": mloc, "n": n, "s": s, "k": k},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference C++ needs Eigen 3.4 + FFTW3 (absent): its restatement (oracle/) is timed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="srht", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-cols", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
