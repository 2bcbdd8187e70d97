"""The reference-compatible CLI (tools/cli/nullsketch_main.cpp; reference
tools/nullsketch_main.cpp:134-290): argument handling and file IO on the CPU,
`nullspace` / `tls` results against the Python API on the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    from paper_2206_00975_b200 import build
    return build.build_cli()


def run(cli, *args, cwd=None):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=300, cwd=cwd)


def write_mm(path, a):
    a = np.asarray(a)
    cplx = np.iscomplexobj(a)
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix array {'complex' if cplx else 'real'} general\n")
        f.write("% written by the test\n")
        f.write(f"{a.shape[0]} {a.shape[1]}\n")
        for v in a.T.reshape(-1):
            f.write(f"{float(v.real)!r} {float(v.imag)!r}\n" if cplx else f"{float(v)!r}\n")


def read_mm(path):
    with open(path) as f:
        head = f.readline().split()
        rows, cols = map(int, f.readline().split())
        vals = [list(map(float, line.split())) for line in f if line.strip()]
    v = np.array(vals)
    x = v[:, 0] + 1j * v[:, 1] if head[3] == "complex" else v[:, 0]
    return x.reshape(cols, rows).T


def test_cli_usage_and_errors(cli, tmp_path):
    r = run(cli, "--help")
    assert r.returncode == 0 and "nullspace" in r.stdout and "tls" in r.stdout
    assert run(cli).returncode == 2
    r = run(cli, "nullspace", "--in", tmp_path / "missing.mtx")
    assert r.returncode == 1 and "cannot open" in r.stderr
    r = run(cli, "frobnicate")
    assert r.returncode == 1 and "unknown command" in r.stderr
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n")
    r = run(cli, "nullspace", "--in", bad)
    assert r.returncode == 1 and "only dense 'array' format" in r.stderr
    short = tmp_path / "short.mtx"
    short.write_text("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n")
    r = run(cli, "nullspace", "--in", short)
    assert r.returncode == 1 and "unexpected end of file" in r.stderr
    ragged = tmp_path / "ragged.csv"
    ragged.write_text("1,2,3\n4,5\n")
    r = run(cli, "nullspace", "--in", ragged)
    assert r.returncode == 1 and "row has 2 entries, expected 3" in r.stderr
    r = run(cli, "nullspace", "--in", short, "--k", "1", "--tol", "1e-3")
    assert r.returncode == 1 and "excludes" in r.stderr
    r = run(cli, "--format", "xml", "nullspace", "--in", short)
    assert r.returncode == 1
    r = run(cli, "tls", "--a", short)
    assert r.returncode == 1 and "--b are required" in r.stderr


@pytest.mark.gpu
def test_cli_nullspace_matches_api(cli, tmp_path, oracle):
    import paper_2206_00975_b200 as nsk
    m, n = 2000, 12
    A = oracle.make_test_matrix(m, n, np.concatenate([np.logspace(0, -3, n - 1), [1e-10]]), 3)
    write_mm(tmp_path / "A.mtx", A)
    out = tmp_path / "out"
    r = run(cli, "--seed", 9, "--out", out, "nullspace", "--in", tmp_path / "A.mtx", "--k", 1, "--sketch", "gaussian",
            "--certificate")
    assert r.returncode == 0, r.stderr
    sm = json.loads(r.stdout)
    assert sm["command"] == "nullspace" and sm["m"] == m and sm["n"] == n and sm["k"] == 1
    assert sm["sketch"]["kind"] == "gaussian" and sm["sketch"]["size"] == 4 * n and sm["sketch"]["seed"] == 9
    W = read_mm(sm["w_path"])
    ref = nsk.solve_k(A, 1, nsk.SketchOperator.draw("gaussian", 4 * n, m, 9))
    assert np.array_equal(W, np.asarray(ref.W))  # same C ABI, same draws: bit-identical
    assert np.allclose(sm["sketched_singular_values"], ref.sketched_singular_values, rtol=0, atol=0)
    assert sm["residual_fro"] > 0
    # --tol picks k from the sketched spectrum; csv flattens the same summary
    r = run(cli, "--format", "csv", "--out", out, "nullspace", "--in", tmp_path / "A.mtx", "--tol", 1e-6)
    assert r.returncode == 0, r.stderr
    rows = dict(line.split(",", 1) for line in r.stdout.strip().splitlines()[1:])
    assert rows["command"] == "nullspace" and rows["k"] == "1" and rows["sketch.kind"] == "srft"


@pytest.mark.gpu
def test_cli_tls_with_exact_baseline(cli, tmp_path, oracle):
    m, n, k = 3000, 8, 1
    A = oracle.random_real(m, n, 5)
    X = oracle.random_real(n, k, 6)
    B = A @ X + 1e-4 * oracle.random_real(m, k, 7)
    write_mm(tmp_path / "A.mtx", A)
    np.savetxt(tmp_path / "B.csv", B, delimiter=",", fmt="%.17g")
    r = run(cli, "--out", tmp_path, "tls", "--a", tmp_path / "A.mtx", "--b", tmp_path / "B.csv", "--sketch",
            "gaussian", "--exact-baseline")
    assert r.returncode == 0, r.stderr
    sm = json.loads(r.stdout)
    Xs = read_mm(sm["x_path"])
    assert np.linalg.norm(Xs - X) / np.linalg.norm(X) < 1e-2
    assert sm["exact"]["tls_residual"] > 0 and sm["residual_ratio"] >= 1.0 - 1e-9
    assert 0 <= sm["metrics"]["rel_err"] < 1e-2 and "exact_seconds" in sm["timings"]
