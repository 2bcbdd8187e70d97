"""Python mirror of the reference's sketch / nullspace API over the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/nullsketch/sketch.hpp and nullspace.hpp):

    S  = SketchOperator.draw(kind, s, m, seed)          sketch.hpp:42
    SA = apply(S, A)                                     sketch.hpp:89
    r  = solve_k(A, k, S)                                nullspace.hpp:24
    r  = solve_tol(A, eps, S)                            nullspace.hpp:30
    f  = residual_certificate(A, W)                      nullspace.hpp:33
    S.descriptor() / SketchOperator.from_descriptor()   sketch.hpp:47-48

Matrices are column-major (matrix.hpp:13-18).  ``A`` may be

* a CUDA ``torch.Tensor`` (float64 or complex128) of shape (m, n); it is
  used in place when column-major (stride(0) == 1) and copied to column-major
  otherwise.  Results come back as CUDA tensors, stream-ordered on torch's
  current stream.
* a NumPy array: the host entry points of the C ABI copy it in, run on the
  current device and copy the results back (the reference's value semantics).

Every call runs the CUDA kernels of libnullsketch_b200.so; there is no
fallback.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (KIND_CODES, KIND_NAMES, NSK_COMPLEX, NSK_REAL, SvdConvergenceError, TlsConditionError,
                   TlsExistenceError, check)

__all__ = ["SketchOperator", "SketchedMatrix", "NullspaceResult", "apply", "apply_shard", "solve_k",
           "solve_tol", "residual_certificate", "svd_trailing", "default_sketch_size", "update_column",
           "downdate_column", "update_row", "downdate_row", "tls_solve_sketched", "tls_solve_exact",
           "tls_error_metrics", "TlsErrorMetrics", "TlsSolution",
           "SvdConvergenceError", "TlsExistenceError", "TlsConditionError", "KINDS"]

KINDS = tuple(KIND_CODES)


def default_sketch_size(kind: str, n: int) -> int:
    """2n for the subsampled transforms, 4n for gaussian (sketch.cpp:99-101); n^2 for countsketch."""
    if kind == "gaussian":
        return 4 * n
    if kind == "countsketch":
        return n * n
    return 2 * n


def _torch():
    import torch
    return torch


def _is_torch(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _stream_ptr():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _colmajor(t):
    """(tensor, ld) with stride(0) == 1; copies if needed."""
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    m, n = t.shape
    if t.stride(0) == 1 and (n <= 1 or t.stride(1) >= max(m, 1)):
        return t, max(t.stride(1) if n > 1 else m, 1)
    f = t.t().contiguous().t()
    return f, max(m, 1)


def _empty_colmajor(rows, cols, dtype, device):
    torch = _torch()
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def _scalar_of(x):
    if _is_torch(x):
        torch = _torch()
        if x.dtype == torch.float64:
            return NSK_REAL
        if x.dtype == torch.complex128:
            return NSK_COMPLEX
        raise ValueError(f"matrix dtype must be float64 or complex128, got {x.dtype}")
    if np.iscomplexobj(x):
        return NSK_COMPLEX
    return NSK_REAL


class SketchOperator:
    """Opaque device-side sketch operator (the descriptor; G is never stored)."""

    def __init__(self, handle):
        self._h = ctypes.c_void_p(handle)
        kind, s, m = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        seed, oid = ctypes.c_uint64(), ctypes.c_uint64()
        check(_lib.load().nsk_op_info(self._h, ctypes.byref(kind), ctypes.byref(s), ctypes.byref(m),
                                      ctypes.byref(seed), ctypes.byref(oid)))
        self._kind, self._s, self._m = KIND_NAMES[kind.value], s.value, m.value
        self._seed, self._id = seed.value, oid.value

    @staticmethod
    def draw(kind: str, s: int, m: int, seed: int) -> "SketchOperator":
        if kind not in KIND_CODES:
            raise ValueError(f"unknown sketch kind: {kind}")
        h = ctypes.c_void_p()
        check(_lib.load().nsk_op_draw(KIND_CODES[kind], int(s), int(m), int(seed) & (2**64 - 1),
                                      ctypes.byref(h)))
        return SketchOperator(h.value)

    @staticmethod
    def from_descriptor(text: str) -> "SketchOperator":
        h = ctypes.c_void_p()
        check(_lib.load().nsk_op_from_descriptor(text.encode(), ctypes.byref(h)))
        return SketchOperator(h.value)

    def descriptor(self) -> str:
        n = ctypes.c_size_t()
        _lib.load().nsk_op_descriptor(self._h, None, 0, ctypes.byref(n))  # size query
        buf = ctypes.create_string_buffer(n.value + 1)
        check(_lib.load().nsk_op_descriptor(self._h, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def sample_indices(self) -> np.ndarray:
        out = np.empty(self._s, dtype=np.int64)
        check(_lib.load().nsk_op_sample_indices(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out

    kind = property(lambda self: self._kind)
    s = property(lambda self: self._s)
    m = property(lambda self: self._m)
    seed = property(lambda self: self._seed)
    id = property(lambda self: self._id)

    def _state(self):
        me, ap, nz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(_lib.load().nsk_op_state(self._h, ctypes.byref(me), ctypes.byref(ap), ctypes.byref(nz), None, 0))
        rows = np.empty(nz.value, dtype=np.int64)
        if nz.value:
            check(_lib.load().nsk_op_state(self._h, None, None, None,
                                           rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), nz.value))
        return me.value, ap.value, [int(r) for r in rows]

    m_effective = property(lambda self: self._state()[0])
    appended_count = property(lambda self: self._state()[1])
    zeroed_rows = property(lambda self: self._state()[2])
    live_rows = property(lambda self: self._state()[0] - len(self._state()[2]))

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().nsk_op_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = ctypes.c_void_p()

    def __repr__(self):
        return f"SketchOperator(kind={self._kind!r}, s={self._s}, m={self._m}, seed={self._seed})"


@dataclasses.dataclass
class SketchedMatrix:
    data: object
    operator_id: int


@dataclasses.dataclass
class NullspaceResult:
    W: object                          # n x k, orthonormal columns
    sketched_singular_values: object   # all n values, non-increasing
    residual_fro: Optional[float] = None
    k: int = 0


def _out_dtype_is_complex(S: SketchOperator, scalar):
    return S.kind == "srft" or scalar == NSK_COMPLEX


def apply(S: SketchOperator, A) -> SketchedMatrix:
    """SA = S A (sketch.cpp:184-232)."""
    L = _lib.load()
    scalar = _scalar_of(A)
    cplx_out = _out_dtype_is_complex(S, scalar)
    if _is_torch(A):
        torch = _torch()
        if not A.is_cuda:
            raise ValueError("torch input must live on a CUDA device")
        A, lda = _colmajor(A)
        m, n = A.shape
        SA = _empty_colmajor(S.s, n, torch.complex128 if cplx_out else torch.float64, A.device)
        check(L.nsk_apply(S.handle, scalar, m, n, ctypes.c_void_p(A.data_ptr()), lda,
                          ctypes.c_void_p(SA.data_ptr()), S.s, _stream_ptr()))
        return SketchedMatrix(SA, S.id)
    A = np.asfortranarray(A, dtype=np.complex128 if scalar == NSK_COMPLEX else np.float64)
    if A.ndim == 1:
        A = A.reshape(-1, 1, order="F")
    m, n = A.shape
    SA = np.empty((S.s, n), dtype=np.complex128 if cplx_out else np.float64, order="F")
    check(L.nsk_apply_host(S.handle, scalar, m, n, A.ctypes.data_as(ctypes.c_void_p), max(m, 1),
                           SA.ctypes.data_as(ctypes.c_void_p), S.s))
    return SketchedMatrix(SA, S.id)


def apply_shard(S: SketchOperator, A_local, row0: int, rstep: int = 1):
    """Partial sketch of a row shard: local row j is global row row0 + rstep*j.

    Summing the partials of a row partition gives apply(S, A) (device tensors only)."""
    torch = _torch()
    L = _lib.load()
    scalar = _scalar_of(A_local)
    cplx_out = _out_dtype_is_complex(S, scalar)
    A_local, lda = _colmajor(A_local)
    mloc, n = A_local.shape
    SA = _empty_colmajor(S.s, n, torch.complex128 if cplx_out else torch.float64, A_local.device)
    check(L.nsk_apply_shard(S.handle, scalar, int(row0), int(rstep), mloc, n, ctypes.c_void_p(A_local.data_ptr()),
                            lda, ctypes.c_void_p(SA.data_ptr()), S.s, _stream_ptr()))
    return SA


def svd_trailing(SA, k: int):
    """(W, sigma): trailing k right singular vectors of a device sketch, all sigmas."""
    torch = _torch()
    L = _lib.load()
    scalar = _scalar_of(SA)
    SA, ld = _colmajor(SA)
    s, n = SA.shape
    W = _empty_colmajor(n, max(k, 0), SA.dtype, SA.device)
    sig = torch.empty(n, dtype=torch.float64, device=SA.device)
    check(L.nsk_svd_trailing(scalar, s, n, ctypes.c_void_p(SA.data_ptr()), ld, int(k),
                             ctypes.c_void_p(W.data_ptr()), max(n, 1), ctypes.c_void_p(sig.data_ptr()),
                             _stream_ptr()))
    return W, sig


def solve_k(A, k: int, S: SketchOperator) -> NullspaceResult:
    """Trailing k right singular vectors of S A (nullspace.cpp:23-32)."""
    L = _lib.load()
    scalar = _scalar_of(A)
    cplx_out = _out_dtype_is_complex(S, scalar)
    if _is_torch(A):
        torch = _torch()
        A, lda = _colmajor(A)
        m, n = A.shape
        W = _empty_colmajor(n, max(k, 0), torch.complex128 if cplx_out else torch.float64, A.device)
        sig = torch.empty(n, dtype=torch.float64, device=A.device)
        check(L.nsk_solve_k(S.handle, scalar, m, n, ctypes.c_void_p(A.data_ptr()), lda, int(k),
                            ctypes.c_void_p(W.data_ptr()), max(n, 1), ctypes.c_void_p(sig.data_ptr()),
                            _stream_ptr()))
        return NullspaceResult(W, sig, None, int(k))
    A = np.asfortranarray(A, dtype=np.complex128 if scalar == NSK_COMPLEX else np.float64)
    m, n = A.shape
    W = np.empty((n, max(k, 0)), dtype=np.complex128 if cplx_out else np.float64, order="F")
    sig = np.empty(n, dtype=np.float64)
    check(L.nsk_solve_k_host(S.handle, scalar, m, n, A.ctypes.data_as(ctypes.c_void_p), max(m, 1), int(k),
                             W.ctypes.data_as(ctypes.c_void_p), max(n, 1), sig.ctypes.data_as(ctypes.c_void_p)))
    return NullspaceResult(W, sig, None, int(k))


def solve_tol(A, eps: float, S: SketchOperator) -> NullspaceResult:
    """k = #sketched singular values below eps (nullspace.cpp:34-53)."""
    L = _lib.load()
    scalar = _scalar_of(A)
    cplx_out = _out_dtype_is_complex(S, scalar)
    kout = ctypes.c_int64()
    if _is_torch(A):
        torch = _torch()
        A, lda = _colmajor(A)
        m, n = A.shape
        W = _empty_colmajor(n, max(n - 1, 1), torch.complex128 if cplx_out else torch.float64, A.device)
        sig = torch.empty(n, dtype=torch.float64, device=A.device)
        check(L.nsk_solve_tol(S.handle, scalar, m, n, ctypes.c_void_p(A.data_ptr()), lda, float(eps),
                              ctypes.byref(kout), ctypes.c_void_p(W.data_ptr()), max(n, 1),
                              ctypes.c_void_p(sig.data_ptr()), _stream_ptr()))
        return NullspaceResult(W[:, :kout.value], sig, None, kout.value)
    A = np.asfortranarray(A, dtype=np.complex128 if scalar == NSK_COMPLEX else np.float64)
    m, n = A.shape
    W = np.empty((n, max(n - 1, 1)), dtype=np.complex128 if cplx_out else np.float64, order="F")
    sig = np.empty(n, dtype=np.float64)
    check(L.nsk_solve_tol_host(S.handle, scalar, m, n, A.ctypes.data_as(ctypes.c_void_p), max(m, 1), float(eps),
                               ctypes.byref(kout), W.ctypes.data_as(ctypes.c_void_p), max(n, 1),
                               sig.ctypes.data_as(ctypes.c_void_p)))
    return NullspaceResult(W[:, :kout.value], sig, None, kout.value)


def residual_certificate(A, W) -> float:
    """||A W||_F in one pass over A (nullspace.cpp:55-62).  Device tensors."""
    torch = _torch()
    L = _lib.load()
    if not _is_torch(A):
        A = torch.from_numpy(np.asfortranarray(A)).cuda()
    if not _is_torch(W):
        W = torch.from_numpy(np.asfortranarray(W)).cuda()
    if A.shape[1] != W.shape[0]:
        raise ValueError(f"residual_certificate: basis lives in dimension {W.shape[0]}, "
                         f"matrix has {A.shape[1]} columns")
    scalar = NSK_COMPLEX if (A.is_complex() or W.is_complex()) else NSK_REAL
    if scalar == NSK_COMPLEX:
        A, W = A.to(torch.complex128), W.to(torch.complex128)
    A, lda = _colmajor(A)
    W, ldw = _colmajor(W)
    out = ctypes.c_double()
    check(L.nsk_residual_fro(scalar, A.shape[0], A.shape[1], ctypes.c_void_p(A.data_ptr()), lda, W.shape[1],
                             ctypes.c_void_p(W.data_ptr()), ldw, ctypes.byref(out), _stream_ptr()))
    return out.value


# ----------------------------------------------------------------------------- incremental maintenance
# sketch.hpp:90-109.  SketchedMatrix.data is a CUDA tensor; host arrays are moved to the device.

def _as_device(x, like=None):
    torch = _torch()
    if _is_torch(x):
        return x
    dev = like.device if like is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(np.asfortranarray(x)).to(dev)


def _require_same_operator(sa: SketchedMatrix, S: SketchOperator):
    if sa.operator_id != S.id:  # sketch.cpp:75-79
        raise ValueError("sketched matrix does not belong to this operator")


def _promoted(data, cplx):
    torch = _torch()
    if cplx and not data.is_complex():
        return data.to(torch.complex128).t().contiguous().t()
    return data.clone() if data.stride(0) == 1 else data.t().contiguous().t()


def update_column(sa: SketchedMatrix, S: SketchOperator, a_col, position: int) -> SketchedMatrix:
    """Insert the sketch of a_col (zeroed rows forced to 0) at `position` (sketch.cpp:234-257)."""
    torch = _torch()
    _require_same_operator(sa, S)
    a_col = _as_device(a_col, sa.data)
    if a_col.dim() == 1:
        a_col = a_col.reshape(-1, 1)
    if a_col.shape != (S.m_effective, 1):
        raise ValueError(f"update_column: column must be {S.m_effective} x 1")
    n = sa.data.shape[1]
    if position < 0 or position > n:
        raise IndexError("update_column: position out of range")
    scalar = _scalar_of(a_col)
    cplx_out = _out_dtype_is_complex(S, scalar)
    col = _empty_colmajor(S.s, 1, torch.complex128 if cplx_out else torch.float64, a_col.device)
    a_col = a_col.contiguous()
    check(_lib.load().nsk_update_column(S.handle, scalar, S.m_effective, ctypes.c_void_p(a_col.data_ptr()),
                                        ctypes.c_void_p(col.data_ptr()), _stream_ptr()))
    data = sa.data
    if col.is_complex() and not data.is_complex():
        data = data.to(torch.complex128)
    elif data.is_complex() and not col.is_complex():
        col = col.to(torch.complex128)
    out = torch.cat([data[:, :position], col, data[:, position:]], dim=1)
    return SketchedMatrix(out.t().contiguous().t(), sa.operator_id)


def downdate_column(sa: SketchedMatrix, position: int) -> SketchedMatrix:
    """Remove a column: an exact splice, no arithmetic (sketch.cpp:259-266)."""
    torch = _torch()
    n = sa.data.shape[1]
    if position < 0 or position >= n:
        raise IndexError("downdate_column: position out of range")
    out = torch.cat([sa.data[:, :position], sa.data[:, position + 1:]], dim=1)
    return SketchedMatrix(out.t().contiguous().t(), sa.operator_id)


def _row_arg(S, a_row, n, like):
    a_row = _as_device(a_row, like)
    if a_row.dim() == 1:
        a_row = a_row.reshape(1, -1)
    if a_row.shape != (1, n):
        raise ValueError(f"expected a 1 x {n} row, got {a_row.shape[0]} x {a_row.shape[1]}")
    return a_row.contiguous().reshape(-1)


def update_row(sa: SketchedMatrix, S: SketchOperator, a_row) -> SketchedMatrix:
    """Append row a_row: SA + g a_row / sqrt(s), g the next Gaussian column of stream (seed, 1) (sketch.cpp:268-280)."""
    _require_same_operator(sa, S)
    n = sa.data.shape[1]
    row = _row_arg(S, a_row, n, sa.data)
    rs = _scalar_of(row)
    if S.kind == "srdct" and rs == NSK_COMPLEX:
        raise ValueError("update_row: srdct sketch carries real data only")
    data = _promoted(sa.data, rs == NSK_COMPLEX)
    check(_lib.load().nsk_update_row(S.handle, _scalar_of(data), n, rs, ctypes.c_void_p(row.data_ptr()),
                                     ctypes.c_void_p(data.data_ptr()), data.stride(1) if n > 1 else S.s,
                                     _stream_ptr()))
    return SketchedMatrix(data, sa.operator_id)


def downdate_row(sa: SketchedMatrix, S: SketchOperator, j: int, a_row_j) -> SketchedMatrix:
    """Remove row j with content a_row_j: SA - (S e_j) a_row_j (sketch.cpp:283-301)."""
    _require_same_operator(sa, S)
    n = sa.data.shape[1]
    row = _row_arg(S, a_row_j, n, sa.data)
    rs = _scalar_of(row)
    cplx = rs == NSK_COMPLEX or (S.kind == "srft" and j < S.m)
    data = _promoted(sa.data, cplx)
    check(_lib.load().nsk_downdate_row(S.handle, int(j), _scalar_of(data), n, rs, ctypes.c_void_p(row.data_ptr()),
                                       ctypes.c_void_p(data.data_ptr()), data.stride(1) if n > 1 else S.s,
                                       _stream_ptr()))
    return SketchedMatrix(data, sa.operator_id)


# ----------------------------------------------------------------------------- sketched TLS

@dataclasses.dataclass
class TlsSolution:
    X: object                      # n x k, X = -V_k1 V_k2^{-1}
    Vk: object                     # (n+k) x k trailing subspace of [A|B]
    tls_residual: float            # sqrt(sum of the k trailing sigma^2)
    cond_Vk2: float
    augmented_singular_values: object
    residual_certificate: Optional[float] = None


def _tls_inputs(A, B):
    torch = _torch()
    A = _as_device(A)
    B = _as_device(B, A)
    if B.dim() == 1:
        B = B.reshape(-1, 1)
    if B.shape[0] != A.shape[0]:
        raise ValueError("tls: A and B row counts differ")
    scalar = NSK_COMPLEX if (A.is_complex() or B.is_complex()) else NSK_REAL
    if scalar == NSK_COMPLEX:
        A, B = A.to(torch.complex128), B.to(torch.complex128)
    A, lda = _colmajor(A)
    B, ldb = _colmajor(B)
    return A, lda, B, ldb, scalar


def _tls_certify(sol, A, B, n, k):
    """||[A|B] Vk||_F = ||A V_k1 + B V_k2||_F (tls.cpp:55-58), opt-in check."""
    torch = _torch()
    pd = sol.Vk.dtype
    prod = A.to(pd) @ sol.Vk[:n, :k] + B.to(pd) @ sol.Vk[n:, :k]
    sol.residual_certificate = float(torch.linalg.norm(prod).item())


def tls_solve_exact(A, B, cond_limit: float = 1e12, allow_marginal: bool = False,
                    certificate: bool = False) -> TlsSolution:
    """Exact total least squares (tls.cpp:83-95): thin QR of [A|B] on the device
    (shifted CholeskyQR3), SVD of the (n+k)^2 triangle, X = -V_k1 V_k2^{-1}."""
    torch = _torch()
    L = _lib.load()
    A, lda, B, ldb, scalar = _tls_inputs(A, B)
    m, n = A.shape
    k = B.shape[1]
    dt = torch.complex128 if scalar == NSK_COMPLEX else torch.float64
    X = _empty_colmajor(n, max(k, 1), dt, A.device)
    Vk = _empty_colmajor(n + k, max(k, 1), dt, A.device)
    sig = torch.empty(n + k, dtype=torch.float64, device=A.device)
    info = np.zeros(4)
    check(L.nsk_tls_solve_exact(scalar, m, n, k, ctypes.c_void_p(A.data_ptr()), lda, ctypes.c_void_p(B.data_ptr()),
                                ldb, float(cond_limit), int(bool(allow_marginal)), ctypes.c_void_p(X.data_ptr()),
                                max(n, 1), ctypes.c_void_p(Vk.data_ptr()), n + k, ctypes.c_void_p(sig.data_ptr()),
                                info.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream_ptr()))
    sol = TlsSolution(X[:, :k], Vk[:, :k], float(info[0]), float(info[1]), sig)
    if certificate:
        _tls_certify(sol, A, B, n, k)
    return sol


@dataclasses.dataclass
class TlsErrorMetrics:
    rel_err: float  # ||X - Xs||_2 / ||X||_2
    sin_X: float    # spectral sin between the column spans of X and Xs
    sin_Vk: float   # spectral sin between the trailing subspaces


def _sin_theta_spectral(U, V):
    """Largest complement sine between two column spans (kernels.cpp:121-167, 153-167)."""
    big, small = (U, V) if U.shape[1] >= V.shape[1] else (V, U)
    if big.shape[1] == 0 or small.shape[1] == 0:
        return 0.0
    r = small - big @ (big.conj().T @ small)
    return min(1.0, float(np.linalg.svd(r, compute_uv=False)[0]))


def tls_error_metrics(exact: TlsSolution, sk: TlsSolution) -> TlsErrorMetrics:
    """Errors of a sketched solution against the exact one (tls.cpp:115-131)."""
    def host(x):
        return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
    X, Xs = host(exact.X), host(sk.X)
    if X.shape != Xs.shape:
        raise ValueError("tls_error_metrics: X shapes differ")
    x_norm = float(np.linalg.svd(X, compute_uv=False)[0])
    if x_norm == 0.0:
        raise ValueError("tls_error_metrics: exact X is zero; rel_err undefined")
    rel = float(np.linalg.svd(X.astype(np.complex128) - Xs.astype(np.complex128), compute_uv=False)[0]) / x_norm
    qe, _ = np.linalg.qr(X)
    qs, _ = np.linalg.qr(Xs)
    return TlsErrorMetrics(rel, _sin_theta_spectral(qe, qs), _sin_theta_spectral(host(exact.Vk), host(sk.Vk)))


def tls_solve_sketched(A, B, S: SketchOperator, cond_limit: float = 1e12, allow_marginal: bool = False,
                       certificate: bool = False) -> TlsSolution:
    """Sketched total least squares (tls.cpp:97-113): trailing subspace of S [A|B], X = -V_k1 V_k2^{-1}."""
    torch = _torch()
    L = _lib.load()
    A, lda, B, ldb, scalar = _tls_inputs(A, B)
    m, n = A.shape
    k = B.shape[1]
    cplx_out = _out_dtype_is_complex(S, scalar)
    dt = torch.complex128 if cplx_out else torch.float64
    X = _empty_colmajor(n, max(k, 1), dt, A.device)
    Vk = _empty_colmajor(n + k, max(k, 1), dt, A.device)
    sig = torch.empty(n + k, dtype=torch.float64, device=A.device)
    info = np.zeros(4)
    check(L.nsk_tls_solve_sketched(S.handle, scalar, m, n, k, ctypes.c_void_p(A.data_ptr()), lda,
                                   ctypes.c_void_p(B.data_ptr()), ldb, float(cond_limit), int(bool(allow_marginal)),
                                   ctypes.c_void_p(X.data_ptr()), max(n, 1), ctypes.c_void_p(Vk.data_ptr()), n + k,
                                   ctypes.c_void_p(sig.data_ptr()), info.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   _stream_ptr()))
    sol = TlsSolution(X[:, :k], Vk[:, :k], float(info[0]), float(info[1]), sig)
    if certificate:
        _tls_certify(sol, A, B, n, k)
    return sol
