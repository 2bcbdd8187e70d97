"""CPU restatement (oracle) of the reference's sketch-and-solve hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs import this module,
and only as the checker or the CPU baseline.  The product package
``paper_2206_00975_b200`` never imports it and fails loudly when its CUDA
library is missing.

What it restates (file:line relative to /root/reference):

* draws                 proj/src/sketch.cpp:103-128, proj/include/nullsketch/rng.hpp
                        (bit-exact, via the plain-C restatement nsk_oracle.c,
                        itself pinned against the compiled reference header)
* apply, gaussian       proj/src/sketch.cpp:195-205 (+ real_times_complex 18-25)
* apply, srft           proj/src/sketch.cpp:206-217 + transforms.cpp:17-36
                        (FFTW_BACKWARD then 1/sqrt(m)  ==  numpy.fft.ifft(norm="ortho"))
* apply, srdct          proj/src/sketch.cpp:218-229 + transforms.cpp:38-64
                        (pre-scaled REDFT01  ==  scipy.fft.dct(type=3, norm="ortho"))
* solve_k / solve_tol   proj/src/nullspace.cpp:10-53 (Eigen BDCSVD -> LAPACK gesdd)
* residual_certificate  proj/src/nullspace.cpp:55-62
* canonical angles      proj/src/kernels.cpp:121-167 (complement projection)
* make_test_matrix      proj/src/kernels.cpp:169-203

Kinds with no reference implementation (SPEC.md:15,210 list them as
non-goals) -- parity for these is *unpinned* beyond their draws:

* srht         SA = sqrt(m/s) R H D A, H the normalised Sylvester Hadamard
               matrix, m a power of two, draws identical to srdct.
* countsketch  SA[h(i), :] += sigma(i) A[i, :]; sigma(i) = next_sign() #i and
               h(i) = next_below(s) #i issued after the m signs on stream
               (seed, 0).

Third-party arithmetic the reference delegates (absent here, so restated by
its published definition): Eigen >= 3.4 (GEMM, BDCSVD, HouseholderQR) and FFTW3
(REDFT01, BACKWARD DFT) -- CMakeLists.txt:131,133, versions unpinned upstream.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

KINDS = ("gaussian", "srft", "srdct", "srht", "countsketch")

c_u64 = ctypes.c_uint64
c_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build():
    """Compile the C restatement (and the reference RNG harness where possible)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libnsk_oracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.nsko_words.argtypes = [c_u64, c_u64, c_u64, c_u64, _u32p]
        L.nsko_gaussians.argtypes = [c_u64, c_u64, c_u64, c_u64, _dp]
        L.nsko_signs.argtypes = [c_u64, c_i64, _dp]
        L.nsko_sample_indices.argtypes = [c_u64, c_i64, c_i64, _ip]
        L.nsko_sample_indices.restype = ctypes.c_int
        L.nsko_countsketch_draw.argtypes = [c_u64, c_i64, c_i64, _i32p, _dp]
        L.nsko_countsketch_apply.argtypes = [c_u64, c_i64, c_i64, c_i64, _dp, c_i64, _dp, c_i64]
        L.nsko_gaussian_block.argtypes = [c_u64, c_u64, c_i64, c_i64, c_i64, _dp, ctypes.c_int]
        L.nsko_srht_apply.argtypes = [_dp, _ip, c_i64, c_i64, c_i64, _dp, c_i64, _dp, c_i64,
                                      c_i64, c_i64, ctypes.c_int]
        L.nsko_fwht.argtypes = [_dp, c_i64]
        L.nsko_gaussian_rows.argtypes = [c_u64, c_u64, c_i64, _ip, c_i64, c_i64, c_i64, _dp, ctypes.c_int]
        L.nsko_countsketch_apply_tables.argtypes = [_i32p, _dp, c_i64, c_i64, c_i64, _dp, c_i64, _dp, c_i64,
                                                    ctypes.c_int]
        _LIB = L
    return _LIB


def ref_lib():
    """The reference's own rng.hpp compiled unmodified (oracle/_ref), or None."""
    global _REF
    if _REF is None:
        path = os.path.join(_HERE, "_ref", "libnsk_ref.so")
        if not os.path.exists(path):
            return None
        L = ctypes.CDLL(path)
        L.nskref_words.argtypes = [c_u64, c_u64, c_u64, _u32p]
        L.nskref_gaussians.argtypes = [c_u64, c_u64, c_u64, _dp]
        L.nskref_doubles.argtypes = [c_u64, c_u64, c_u64, _dp]
        L.nskref_gaussian_G.argtypes = [c_u64, c_i64, c_i64, _dp]
        L.nskref_srtt_draw.argtypes = [c_u64, c_i64, c_i64, _dp, _ip]
        L.nskref_countsketch_draw.argtypes = [c_u64, c_i64, c_i64, _i32p, _dp]
        L.nskref_update_gaussians.argtypes = [c_u64, c_i64, c_i64, _dp]
        _REF = L
    return _REF


def _p(a, t):
    return a.ctypes.data_as(t)


# ----------------------------------------------------------------------------- draws

def words(seed, stream, first, count):
    out = np.empty(count, dtype=np.uint32)
    lib().nsko_words(seed, stream, first, count, _p(out, _u32p))
    return out


def gaussians(seed, stream, first, count):
    out = np.empty(count, dtype=np.float64)
    lib().nsko_gaussians(seed, stream, first, count, _p(out, _dp))
    return out


def signs(seed, m):
    out = np.empty(m, dtype=np.float64)
    lib().nsko_signs(seed, m, _p(out, _dp))
    return out


def sample_indices(seed, m, s):
    out = np.empty(s, dtype=np.int64)
    rc = lib().nsko_sample_indices(seed, m, s, _p(out, _ip))
    if rc != 0:
        raise ValueError("sample_indices: need 0 <= s <= m")
    return out


def countsketch_draw(seed, m, s):
    b = np.empty(m, dtype=np.int32)
    g = np.empty(m, dtype=np.float64)
    lib().nsko_countsketch_draw(seed, m, s, _p(b, _i32p), _p(g, _dp))
    return b, g


def gaussian_block(seed, s, j0, j1, stream=0, nthreads=None):
    """Columns j0..j1-1 of the s x m Gaussian G (sketch.cpp:117-121), s x (j1-j0)."""
    out = np.empty((j1 - j0) * s, dtype=np.float64)
    lib().nsko_gaussian_block(seed, stream, s, j0, j1, _p(out, _dp), nthreads or os.cpu_count())
    return out.reshape(j1 - j0, s).T


def gaussian_rows(seed, s, rows, j0, j1, stream=0, nthreads=None):
    """Rows `rows` of the s x m Gaussian G over columns j0..j1-1 (sketch.cpp:117-121):
    out[r, j - j0] = Gaussian #(j*s + rows[r]) of stream (seed, stream).  A row sample of G
    costs len(rows) draws per column, so SA row samples at configs[3] size stay cheap."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((j1 - j0) * len(rows), dtype=np.float64)
    lib().nsko_gaussian_rows(seed, stream, s, _p(rows, _ip), len(rows), j0, j1, _p(out, _dp),
                             nthreads or os.cpu_count())
    return out.reshape(j1 - j0, len(rows)).T


class OracleOperator:
    """Mirror of SketchOperator's draw state (sketch.hpp:40-81) for the oracle."""

    def __init__(self, kind, s, m, seed):
        if kind not in KINDS:
            raise ValueError(f"unknown sketch kind: {kind}")
        if s < 1 or m < 1:
            raise ValueError("sketch draw: s and m must be positive")
        if kind in ("srft", "srdct", "srht") and s > m:
            raise ValueError("sketch draw: subsampled transforms need s <= m")
        if kind == "srht" and (m & (m - 1)) != 0:
            raise ValueError("sketch draw: srht needs m to be a power of two")
        self.kind, self.s, self.m, self.seed = kind, s, m, seed
        self.signs = self.idx = self.bucket = None
        if kind in ("srft", "srdct", "srht"):
            self.signs = signs(seed, m)
            self.idx = sample_indices(seed, m, s)
        elif kind == "countsketch":
            self.bucket, self.signs = countsketch_draw(seed, m, s)

    def dense(self):
        """Explicit s x m matrix (small sizes only), as SketchOperator::dense (sketch.cpp:162-172)."""
        eye = np.eye(self.m)
        return apply(self, eye)


def draw(kind, s, m, seed):
    return OracleOperator(kind, s, m, seed)


# ----------------------------------------------------------------------------- apply

def apply(op: OracleOperator, A, col_range=None):
    """SA = S A for every kind (sketch.cpp:184-232)."""
    A = np.asarray(A)
    if A.ndim == 1:
        A = A[:, None]
    if A.shape[0] != op.m:
        raise ValueError(f"sketch apply: matrix has {A.shape[0]} rows, operator expects {op.m}")
    s, m = op.s, op.m
    if op.kind == "gaussian":
        inv = 1.0 / math.sqrt(s)
        out = np.zeros((s, A.shape[1]), dtype=A.dtype)
        blk = max(1, min(m, (1 << 26) // max(s, 1)))
        for j0 in range(0, m, blk):  # streamed: G is regenerated by column blocks
            j1 = min(m, j0 + blk)
            G = gaussian_block(op.seed, s, j0, j1)
            if np.iscomplexobj(A):  # real_times_complex (sketch.cpp:18-25)
                out += G @ A[j0:j1].real + 1j * (G @ A[j0:j1].imag)
            else:
                out += G @ A[j0:j1]
        return inv * out
    if op.kind == "srft":
        top = op.signs[:, None] * A.astype(np.complex128)
        top = np.fft.ifft(top, axis=0, norm="ortho")
        return math.sqrt(m / s) * top[op.idx]
    if op.kind == "srdct":
        if np.iscomplexobj(A):
            raise ValueError("srdct sketch is defined for real matrices only")
        import scipy.fft
        top = scipy.fft.dct(op.signs[:, None] * A, type=3, norm="ortho", axis=0)
        return math.sqrt(m / s) * top[op.idx]
    if op.kind == "srht":
        if np.iscomplexobj(A):
            raise ValueError("srht sketch is defined for real matrices only")
        A = np.asfortranarray(A, dtype=np.float64)
        n = A.shape[1]
        c0, c1 = col_range or (0, n)
        SA = np.zeros((s, n), dtype=np.float64, order="F")
        lib().nsko_srht_apply(_p(op.signs, _dp), _p(op.idx, _ip), s, m, n, _p(A, _dp), m,
                              _p(SA, _dp), s, c0, c1, os.cpu_count())
        return SA
    if op.kind == "countsketch":
        if np.iscomplexobj(A):
            raise ValueError("countsketch is defined for real matrices only")
        A = np.asfortranarray(A, dtype=np.float64)
        n = A.shape[1]
        SA = np.zeros((s, n), dtype=np.float64, order="F")
        # rows added in increasing order within each column (threads split the columns)
        lib().nsko_countsketch_apply_tables(_p(op.bucket, _i32p), _p(op.signs, _dp), s, m, n, _p(A, _dp), m,
                                            _p(SA, _dp), s, os.cpu_count())
        return SA
    raise ValueError(op.kind)


def srtt_shard_partial(op: OracleOperator, A_local, g, P):
    """Partial sketch of cyclic shard g of P (global rows g, g+P, ...; P | m) by decimation in time
    (SURVEY.md 8e): one length-N = m/P inverse DFT of the local rows, the shard twiddle, the gather.
      srft : (1/sqrt s) w_m^{a g} W[a mod N],                    W = DFT_N(d x)
      srdct: sqrt(m/s) Re(w_{4m}^{(2a+1) g} Z_a),                W = DFT_N(c d x w_{4N}^l),
             Z_a = W[b/2] (b even) or conj(W[(-(b-1)/2 - 1) mod N]) (b odd), b = ((2a+1) mod 4N - 1)/2
    (w_K = e^{+2 pi i/K}); summed over g it equals apply(op, A) (sketch.cpp:206-229)."""
    m, s = op.m, op.s
    if m % P:
        raise ValueError("cyclic shards need P | m")
    N = m // P
    A_local = np.asarray(A_local)
    if A_local.ndim == 1:
        A_local = A_local[:, None]
    rows = g + P * np.arange(N)
    d = op.signs[rows][:, None]
    a = op.idx.astype(np.int64)
    if op.kind == "srft":
        W = np.fft.ifft(d * A_local.astype(np.complex128), axis=0) * N
        post = np.exp(2j * np.pi * ((a * g) % m) / m)
        return post[:, None] * W[a % N] / math.sqrt(s)
    if op.kind != "srdct":
        raise ValueError("srtt_shard_partial: srft / srdct only")
    cj = np.where(rows == 0, math.sqrt(1.0 / m), math.sqrt(2.0 / m))[:, None]
    lw = np.exp(2j * np.pi * np.arange(N) / (4 * N))[:, None]
    W = np.fft.ifft(d * cj * A_local * lw, axis=0) * N
    q = (2 * a + 1) % (4 * N)
    b = (q - 1) // 2
    odd = b % 2 == 1
    f = np.where(odd, (-(b - 1) // 2 - 1) % N, b // 2)
    Z = W[f]
    Z[odd] = np.conj(Z[odd])
    post = np.exp(2j * np.pi * (((2 * a + 1) * g) % (4 * m)) / (4 * m))
    return math.sqrt(m / s) * np.real(post[:, None] * Z)


# ----------------------------------------------------------------------------- solve

def svd(a):
    """Thin SVD, S non-increasing (kernels.cpp:14-22, 54-70); V returned (not V^*)."""
    if a.size == 0:
        raise ValueError("svd: matrix is empty")
    u, sv, vh = np.linalg.svd(a, full_matrices=False)
    return u, sv, vh.conj().T


def from_sketch_svd(sa, k):
    n = sa.shape[1]
    if k < 0 or k >= n:
        raise ValueError(f"nullspace: k must satisfy 0 <= k < n, got k = {k}, n = {n}")
    _, sv, v = svd(sa)
    return v[:, n - k:], sv


def solve_k(A, k, op):
    """W = trailing k right singular vectors of SA; all n sketched sigmas (nullspace.cpp:23-32)."""
    if A.shape[0] != op.m:
        raise ValueError("nullspace: matrix rows do not match the sketch operator")
    if op.s < A.shape[1]:
        raise ValueError(f"nullspace: sketch size s = {op.s} is smaller than n = {A.shape[1]}")
    return from_sketch_svd(apply(op, A), k)


def solve_tol(A, eps, op):
    """k = number of sketched singular values below eps (nullspace.cpp:34-53)."""
    if not (eps >= 0.0):
        raise ValueError("nullspace: eps must be non-negative")
    if A.shape[0] != op.m:
        raise ValueError("nullspace: matrix rows do not match the sketch operator")
    if op.s < A.shape[1]:
        raise ValueError("nullspace: sketch size is smaller than n")
    sa = apply(op, A)
    _, sv, v = svd(sa)
    n = sa.shape[1]
    k = 0
    while k < n and sv[n - 1 - k] < eps:
        k += 1
    if k == n:
        raise ValueError("nullspace: eps selects every singular value")
    return v[:, n - k:], sv, k


def residual_certificate(A, W):
    """||A W||_F (nullspace.cpp:55-62)."""
    if A.shape[1] != W.shape[0]:
        raise ValueError("residual_certificate: dimension mismatch")
    return float(np.linalg.norm(A @ W))


# ----------------------------------------------------------------------------- angles

def complement_sines(big, small):
    """Singular values of small - big (big^* small), descending (kernels.cpp:121-128)."""
    cross = big.conj().T @ small
    resid = small - big @ cross
    return np.linalg.svd(resid, compute_uv=False)


def sin_theta(U, V):
    """sin of the largest canonical angle, spectral (kernels.cpp:153-167)."""
    if U.shape[1] == 0 or V.shape[1] == 0:
        return 0.0
    big, small = (U, V) if U.shape[1] >= V.shape[1] else (V, U)
    return float(min(1.0, complement_sines(big, small)[0]))


def canonical_angles(U, V):
    """Canonical angles ascending (kernels.cpp:132-151)."""
    big, small = (U, V) if U.shape[1] >= V.shape[1] else (V, U)
    k = small.shape[1]
    if k == 0:
        return np.zeros(0)
    cos = np.linalg.svd(big.conj().T @ small, compute_uv=False)
    sin = complement_sines(big, small)
    out = np.empty(k)
    for i in range(k):
        c = min(1.0, max(0.0, cos[i]))
        s_ = min(1.0, max(0.0, sin[k - 1 - i]))
        out[i] = math.asin(s_) if c >= math.sqrt(0.5) else math.acos(c)
    return out


# ----------------------------------------------------------------------------- inputs

def thin_qr(a):
    """Householder thin QR with diag(R) made non-negative (kernels.cpp:32-50)."""
    q, r = np.linalg.qr(a, mode="reduced")
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d, (r.T * d).T


def _cholqr2(a):
    """Q of a well-conditioned tall a by two CholeskyQR passes, diag(R) > 0: the same Q as the
    Householder QR with non-negative diag(R) to O(u) for cond(a) ~ 1 (Gaussian frames)."""
    q = a
    for _ in range(2):
        r = np.linalg.cholesky(q.T @ q).T
        q = q @ np.linalg.inv(r)
    return q


def make_test_matrix(m, n, spectrum, seed, left="haar", qr="householder"):
    """U diag(spectrum) V^T (kernels.cpp:169-203): U = Q of stream-1 Gaussians
    (column-major, m x n), V = Q of stream-2 Gaussians (n x n).  qr="cholqr2" forms U by
    CholeskyQR2 instead of Householder (same Q to rounding; 10x faster at m = 2^20)."""
    spectrum = np.asarray(spectrum, dtype=np.float64)
    if m < n:
        raise ValueError("make_test_matrix: need m >= n")
    if left == "coherent":
        u = np.zeros((m, n))
        u[:n, :n] = np.eye(n)
    else:
        # g[i, c] = Gaussian #(c*m + i) of stream 1 (column-major fill), drawn by threads
        g = gaussian_block(seed, m, 0, n, stream=1)
        u = _cholqr2(g) if qr == "cholqr2" else thin_qr(g)[0]
    gv = gaussians(seed, 2, 0, n * n).reshape(n, n).T
    v = thin_qr(gv)[0]
    return np.asfortranarray((u * spectrum) @ v.T)


def random_real(m, n, seed):
    """Test fixture of the reference (tests/test_support.hpp:18-24): stream 77."""
    return np.asfortranarray(gaussians(seed, 77, 0, m * n).reshape(n, m).T)


def random_complex(m, n, seed):
    """Test fixture of the reference (tests/test_support.hpp:26-33): stream 78, (re, im) pairs."""
    g = gaussians(seed, 78, 0, 2 * m * n).reshape(n, m, 2)
    return np.asfortranarray((g[..., 0] + 1j * g[..., 1]).T)


# ----------------------------------------------------------------------------- incremental state
# sketch.cpp:130-160 (sketch_vector), 174-182 (zero_row), 234-301 (updates).  The
# oracle operator grows the same state the device operator keeps: appended
# Gaussian columns (stream (seed, 1)) and the sorted zeroed rows.

def _m_eff(op):
    return op.m + getattr(op, "appended", 0)


def _zeroed(op):
    if not hasattr(op, "zeroed"):
        op.zeroed = []
    return op.zeroed


def sketch_vector(op, j):
    """Column j of S, scaling included (sketch.cpp:130-160); zeroed gaussian/appended columns are 0."""
    s, m = op.s, op.m
    inv = 1.0 / math.sqrt(s)
    if j >= m:
        if j in _zeroed(op):
            return np.zeros(s)
        return inv * gaussians(op.seed, 1, (j - m) * s, s)
    if op.kind == "gaussian":
        if j in _zeroed(op):
            return np.zeros(s)
        return inv * gaussian_block(op.seed, s, j, j + 1, nthreads=1)[:, 0]
    if op.kind == "countsketch":
        e = np.zeros(s)
        e[op.bucket[j]] = op.signs[j]
        return e
    d = op.signs[j]
    a = op.idx.astype(object)
    if op.kind == "srft":  # transforms.cpp:66-72, argument reduced mod m
        r = np.array([(int(x) * j) % m for x in a], dtype=np.float64)
        return inv * d * np.exp(2j * np.pi * r / m)
    if op.kind == "srdct":  # transforms.cpp:74-80 with exact reduction of j (2a+1) mod 4m
        r = np.array([(j * (2 * int(x) + 1)) % (4 * m) for x in a], dtype=np.float64)
        cj = math.sqrt(1.0 / m) if j == 0 else math.sqrt(2.0 / m)
        return math.sqrt(m / s) * d * cj * np.cos(np.pi * r / (2 * m))
    par = np.array([bin(int(x) & j).count("1") & 1 for x in a])
    return inv * d * np.where(par == 1, -1.0, 1.0)  # srht


def dense_state(op):
    """s x m_effective matrix currently applied (SketchOperator::dense, sketch.cpp:162-172)."""
    cols = [sketch_vector(op, j) for j in range(_m_eff(op))]
    return np.stack(cols, axis=1)


def apply_state(op, A):
    """apply() with appended rows and zeroed rows (sketch.cpp:184-232)."""
    A = np.asarray(A)
    if A.ndim == 1:
        A = A[:, None]
    if A.shape[0] != _m_eff(op):
        raise ValueError("sketch apply: row count mismatch")
    top = A[:op.m].copy()
    if op.kind == "gaussian":  # zeroed columns of G
        for z in _zeroed(op):
            if z < op.m:
                top[z] = 0
    SA = apply(op, top)
    p = _m_eff(op) - op.m
    if p:
        G = np.stack([gaussians(op.seed, 1, c * op.s, op.s) for c in range(p)], axis=1)
        for z in _zeroed(op):
            if z >= op.m:
                G[:, z - op.m] = 0
        bottom = (G @ A[op.m:]) / math.sqrt(op.s)
        SA = SA + bottom
    return SA


def update_row(op, SA, a_row):
    """SA + g a_row / sqrt(s), g = next Gaussian column of stream (seed, 1) (sketch.cpp:268-280)."""
    p = _m_eff(op) - op.m
    g = gaussians(op.seed, 1, p * op.s, op.s)
    op.appended = getattr(op, "appended", 0) + 1
    return SA + np.outer(g, np.ravel(a_row)) / math.sqrt(op.s)


def downdate_row(op, SA, j, a_row):
    """SA - (S e_j) a_row, then zero row j (sketch.cpp:283-301)."""
    if j < 0 or j >= _m_eff(op):
        raise IndexError("downdate_row: row index out of range")
    if j in _zeroed(op):
        raise ValueError("downdate_row: row already removed")
    e = sketch_vector(op, j)
    out = SA - np.outer(e, np.ravel(a_row))
    z = _zeroed(op)
    z.append(j)
    z.sort()
    return out


def update_column(op, SA, a_col, position):
    """Insert the sketch of a_col with zeroed rows forced to 0 (sketch.cpp:234-257)."""
    col = np.array(a_col, dtype=np.result_type(a_col, np.float64)).reshape(-1, 1)
    for z in _zeroed(op):
        col[z] = 0
    sk = apply_state(op, col)
    return np.concatenate([SA[:, :position], sk, SA[:, position:]], axis=1)


def tls_solve_sketched(A, B, op, cond_limit=1e12, allow_marginal=False):
    """Sketched TLS (tls.cpp:97-113, extract_x 26-43, assemble 45-60); returns (X, Vk, sigma, residual, cond)."""
    A = np.asarray(A)
    B = np.asarray(B).reshape(A.shape[0], -1)
    m, n = A.shape
    k = B.shape[1]
    if k < 1 or n < k or m < n + k:
        raise ValueError("tls: bad shape")
    sk = apply_state(op, np.concatenate([A, B], axis=1))
    return tls_from_sketch(sk, n, k, cond_limit, allow_marginal)


def tls_from_sketch(sk, n, k, cond_limit=1e12, allow_marginal=False):
    """The part of tls_solve_sketched after the apply (tls.cpp:110-113, extract_x 26-43):
    SVD of the s x (n+k) sketch, existence check, X = -V1 V2^{-1}."""
    _, sv, v = svd(sk)
    sa = np.linalg.svd(sk[:, :n], compute_uv=False)
    if not (sa[n - 1] > sv[n]) and not allow_marginal:
        raise RuntimeError("tls: solution existence check failed")
    vk = v[:, n:n + k]
    v1, v2 = vk[:n], vk[n:]
    s2 = np.linalg.svd(v2, compute_uv=False)
    cond = np.inf if s2[-1] == 0 else s2[0] / s2[-1]
    if not (cond <= cond_limit):
        raise RuntimeError("tls: V_k2 ill conditioned")
    X = np.linalg.solve(v2.T, -v1.T).T
    return X, vk, sv, math.sqrt(np.sum(sv[n:] ** 2)), cond


def tls_solve_exact(A, B, cond_limit=1e12, allow_marginal=False):
    """Exact TLS (tls.cpp:83-95): Householder thin QR of [A|B] (LAPACK), SVD of R,
    sigma_n(A) from the leading n columns of R; returns (X, Vk, sigma, residual, cond)."""
    A = np.asarray(A)
    B = np.asarray(B).reshape(A.shape[0], -1)
    m, n = A.shape
    k = B.shape[1]
    if k < 1 or n < k or m < n + k:
        raise ValueError("tls: bad shape")
    R = np.linalg.qr(np.concatenate([A, B], axis=1), mode="r")
    _, sv, v = svd(R)
    sa = np.linalg.svd(R[:, :n], compute_uv=False)
    if not (sa[n - 1] > sv[n]) and not allow_marginal:
        raise RuntimeError("tls: solution existence check failed")
    vk = v[:, n:n + k]
    v1, v2 = vk[:n], vk[n:]
    s2 = np.linalg.svd(v2, compute_uv=False)
    cond = np.inf if s2[-1] == 0 else s2[0] / s2[-1]
    if not (cond <= cond_limit):
        raise RuntimeError("tls: V_k2 ill conditioned")
    X = np.linalg.solve(v2.T, -v1.T).T
    return X, vk, sv, math.sqrt(np.sum(sv[n:] ** 2)), cond


def doubles(seed, stream, first, count):
    """next_double #first.. of a stream (rng.hpp:36-39): (u64 >> 11) * 2^-53, u64 = words (2i+1 : 2i)."""
    w = words(seed, stream, 2 * first, 2 * count).astype(np.uint64).reshape(count, 2)
    u = (w[:, 1] << np.uint64(32)) | w[:, 0]
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def loewner_config5(m=100000, n=150, seed=7):
    """BASELINE configs[4]: z on the unit circle by the reference sampler protocol
    (theta = 2 pi next_double of stream 11, bench.cpp:390-398), f(z) = 1/(1.1 - z) + e^z,
    support = floor(j m / n), Loewner (F_i - f_j)/(Z_i - z_j) over the active rows
    (aaa.cpp:152-177).  Returns the (m - n) x n complex matrix."""
    theta = 2.0 * math.pi * doubles(seed, 11, 0, m)
    z = np.cos(theta) + 1j * np.sin(theta)
    f = 1.0 / (1.1 - z) + np.exp(z)
    support = (np.arange(n) * m) // n
    active = np.setdiff1d(np.arange(m), support)
    L = (f[active, None] - f[None, support]) / (z[active, None] - z[None, support])
    return np.asfortranarray(L)
