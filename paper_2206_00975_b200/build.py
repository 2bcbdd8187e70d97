"""Build libnullsketch_b200.so in-tree for sm_100a (nvcc; no JIT cache).

Usage: python -m paper_2206_00975_b200.build  [--force]
The library is self-contained (static cudart); nothing is installed outside
the package directory, so the built .so travels with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libnullsketch_b200.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]

SOURCES = ["operator.cpp", "capi.cpp", "gaussian_sketch.cu", "srht_sketch.cu", "countsketch.cu",
           "srtt_sketch.cu", "srtt_fast.cu", "srtt_general.cu", "jacobi_svd.cu", "residual.cu", "instrument.cpp", "updates.cu",
           "cs_schedule.cpp", "h2d.cpp", "nccl_shard.cpp", "cluster_jacobi.cu", "srtt_tile.cu", "tall_qr.cu", "srdct_stream.cu", "srft_ws.cu"]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "nullsketch_b200.h")]


def _nccl_dirs():
    """nccl.h (types only; the library is dlopened at run time) from the torch-bundled NCCL wheel."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
    except Exception:
        base = "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"
    return os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")


def _compile(src):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    lang = ["-x", "cu"] if src.endswith(".cpp") else []
    extra = []
    if src == "nccl_shard.cpp":
        inc, lib = _nccl_dirs()
        extra = ["-I", inc, f'-DNSK_NCCL_PATH="{lib}"']
    cmd = [NVCC, *ARCH, *FLAGS, *lang, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in _deps() if os.path.exists(d))


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, SOURCES))
    for obj, err in results:
        if verbose and err.strip():
            print(err, file=sys.stderr)
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *[o for o, _ in results], "-lcublas", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return OUT


CLI_SRC = os.path.join(HERE, "..", "tools", "cli", "nullsketch_main.cpp")
CLI_OUT = os.path.join(HERE, "nullsketch_b200")


def build_cli(force=False):
    """The reference-compatible command-line tool (tools/cli), linked against the library."""
    lib = build()
    if not force and os.path.exists(CLI_OUT) and os.path.getmtime(CLI_OUT) >= max(
            os.path.getmtime(CLI_SRC), os.path.getmtime(lib),
            os.path.getmtime(os.path.join(HERE, "..", "include", "nullsketch_b200.hpp"))):
        return CLI_OUT
    cmd = ["g++", "-O2", "-std=c++17", "-I", os.path.join(HERE, "..", "include"), CLI_SRC, "-o", CLI_OUT,
           "-L", HERE, "-lnullsketch_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    return CLI_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_cli(force="--force" in sys.argv))
