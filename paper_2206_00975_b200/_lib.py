"""ctypes binding of libnullsketch_b200.so (the C ABI in include/nullsketch_b200.h).

The library is the product: there is no CPU or PyTorch fallback.  Loading
fails loudly (ImportError) when the shared object is missing, and every
status code other than NSK_OK is raised as the Python analogue of the
reference's C++ exception (std::invalid_argument -> ValueError,
std::out_of_range -> IndexError, SvdConvergenceError -> SvdConvergenceError).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnullsketch_b200.so")

NSK_OK, NSK_EINVAL, NSK_ERANGE, NSK_ENOCONV, NSK_ECUDA, NSK_ENOMEM, NSK_ETLS_EXISTENCE, NSK_ETLS_CONDITION = range(8)
NSK_REAL, NSK_COMPLEX = 0, 1
KIND_CODES = {"gaussian": 0, "srft": 1, "srdct": 2, "srht": 3, "countsketch": 4}
KIND_NAMES = {v: k for k, v in KIND_CODES.items()}

# Symbols declared in include/nullsketch_b200.h (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "nsk_last_error", "nsk_version", "nsk_op_draw", "nsk_op_destroy", "nsk_op_info",
    "nsk_op_sample_indices", "nsk_op_descriptor", "nsk_op_from_descriptor", "nsk_apply",
    "nsk_apply_shard", "nsk_svd_trailing", "nsk_solve_k", "nsk_solve_tol", "nsk_residual_fro",
    "nsk_apply_host", "nsk_solve_k_host", "nsk_solve_tol_host", "nsk_residual_fro_host", "nsk_kernel_launches",
    "nsk_timing_enable", "nsk_timing_collect", "nsk_timing_kernel", "nsk_op_state", "nsk_update_row", "nsk_downdate_row",
    "nsk_update_column", "nsk_tls_solve_sketched", "nsk_tls_solve_sketched_host", "nsk_tls_solve_exact", "nsk_tls_solve_exact_host", "nsk_update_row_host",
    "nsk_downdate_row_host", "nsk_update_column_host", "nsk_nccl_unique_id", "nsk_nccl_comm_init",
    "nsk_nccl_comm_destroy", "nsk_apply_allreduce", "nsk_solve_k_sharded", "nsk_release_scratch",
    "nsk_solve_k_sharded_host",
)


class SvdConvergenceError(RuntimeError):
    """Raised when the on-device SVD does not converge (kernels.hpp:18-20)."""


class TlsExistenceError(RuntimeError):
    """sigma_n(A) is not above sigma_{n+1}([A|B]) (tls.hpp:37-48)."""


class TlsConditionError(RuntimeError):
    """V_k2 is ill conditioned (tls.hpp:50-57)."""


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2206_00975_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, u64, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)
    i64p = ctypes.POINTER(ctypes.c_int64)
    c_int = ctypes.c_int
    L.nsk_last_error.restype = ctypes.c_char_p
    L.nsk_version.restype = ctypes.c_char_p
    L.nsk_op_draw.argtypes = [c_int, i64, i64, u64, ctypes.POINTER(vp)]
    L.nsk_op_destroy.argtypes = [vp]
    L.nsk_op_destroy.restype = None
    L.nsk_op_info.argtypes = [vp, ctypes.POINTER(c_int), i64p, i64p, ctypes.POINTER(u64), ctypes.POINTER(u64)]
    L.nsk_op_sample_indices.argtypes = [vp, i64p]
    L.nsk_op_descriptor.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    L.nsk_op_from_descriptor.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.nsk_apply.argtypes = [vp, c_int, i64, i64, vp, i64, vp, i64, vp]
    L.nsk_apply_shard.argtypes = [vp, c_int, i64, i64, i64, i64, vp, i64, vp, i64, vp]
    L.nsk_svd_trailing.argtypes = [c_int, i64, i64, vp, i64, i64, vp, i64, vp, vp]
    L.nsk_solve_k.argtypes = [vp, c_int, i64, i64, vp, i64, i64, vp, i64, vp, vp]
    L.nsk_solve_tol.argtypes = [vp, c_int, i64, i64, vp, i64, ctypes.c_double, i64p, vp, i64, vp, vp]
    L.nsk_residual_fro.argtypes = [c_int, i64, i64, vp, i64, i64, vp, i64, dp, vp]
    L.nsk_apply_host.argtypes = [vp, c_int, i64, i64, vp, i64, vp, i64]
    L.nsk_solve_k_host.argtypes = [vp, c_int, i64, i64, vp, i64, i64, vp, i64, vp]
    L.nsk_solve_tol_host.argtypes = [vp, c_int, i64, i64, vp, i64, ctypes.c_double, i64p, vp, i64, vp]
    L.nsk_residual_fro_host.argtypes = [c_int, i64, i64, vp, i64, i64, vp, i64, dp]
    L.nsk_op_state.argtypes = [vp, i64p, i64p, i64p, i64p, i64]
    L.nsk_update_row.argtypes = [vp, c_int, i64, c_int, vp, vp, i64, vp]
    L.nsk_downdate_row.argtypes = [vp, i64, c_int, i64, c_int, vp, vp, i64, vp]
    L.nsk_update_column.argtypes = [vp, c_int, i64, vp, vp, vp]
    L.nsk_update_row_host.argtypes = [vp, c_int, i64, c_int, vp, vp, i64]
    L.nsk_downdate_row_host.argtypes = [vp, i64, c_int, i64, c_int, vp, vp, i64]
    L.nsk_update_column_host.argtypes = [vp, c_int, i64, vp, vp]
    L.nsk_tls_solve_sketched.argtypes = [vp, c_int, i64, i64, i64, vp, i64, vp, i64, ctypes.c_double, c_int, vp, i64,
                                         vp, i64, vp, dp, vp]
    L.nsk_tls_solve_sketched_host.argtypes = [vp, c_int, i64, i64, i64, vp, i64, vp, i64, ctypes.c_double, c_int, vp,
                                              i64, vp, i64, vp, dp]
    L.nsk_tls_solve_exact.argtypes = [c_int, i64, i64, i64, vp, i64, vp, i64, ctypes.c_double, c_int, vp, i64, vp,
                                      i64, vp, dp, vp]
    L.nsk_tls_solve_exact_host.argtypes = [c_int, i64, i64, i64, vp, i64, vp, i64, ctypes.c_double, c_int, vp, i64,
                                           vp, i64, vp, dp]
    L.nsk_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.nsk_nccl_comm_init.argtypes = [c_int, ctypes.c_char_p, c_int, ctypes.POINTER(vp)]
    L.nsk_nccl_comm_destroy.argtypes = [vp]
    L.nsk_apply_allreduce.argtypes = [vp, c_int, i64, i64, i64, i64, vp, i64, vp, i64, vp, vp]
    L.nsk_solve_k_sharded.argtypes = [vp, c_int, i64, i64, i64, i64, vp, i64, i64, vp, i64, vp, vp, vp]
    L.nsk_solve_k_sharded_host.argtypes = [vp, c_int, i64, i64, i64, i64, vp, i64, i64, vp, i64, vp, vp]
    L.nsk_kernel_launches.restype = i64
    L.nsk_timing_enable.argtypes = [c_int]
    L.nsk_timing_enable.restype = None
    L.nsk_timing_kernel.restype = ctypes.c_char_p
    L.nsk_timing_collect.argtypes = [dp, i64p]
    for name in EXPORTS:
        getattr(L, name)  # every declared symbol must resolve
    _lib = L
    return L


def check(rc):
    if rc == NSK_OK:
        return
    msg = (load().nsk_last_error() or b"").decode(errors="replace")
    if rc == NSK_EINVAL:
        raise ValueError(msg)
    if rc == NSK_ERANGE:
        raise IndexError(msg)
    if rc == NSK_ENOCONV:
        raise SvdConvergenceError(msg)
    if rc == NSK_ENOMEM:
        raise MemoryError(msg)
    if rc == NSK_ETLS_EXISTENCE:
        raise TlsExistenceError(msg)
    if rc == NSK_ETLS_CONDITION:
        raise TlsConditionError(msg)
    raise RuntimeError(f"nullsketch CUDA failure: {msg}")
