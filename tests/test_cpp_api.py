"""Build tests/cpp/test_cpp_api.cpp against include/nullsketch_b200.hpp and the
in-tree library; the compile runs everywhere, the binary runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2206_00975_b200")


def _build(tmp_path):
    from paper_2206_00975_b200 import build
    build.build()
    exe = str(tmp_path / "test_cpp_api")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", LIBDIR, "-lnullsketch_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_api_compiles(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
