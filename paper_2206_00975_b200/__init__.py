"""nullsketch-b200: B200-native sketch-and-solve null-space hot path.

Public API mirrors the reference's sketch / nullspace modules
(/root/reference/proj/include/nullsketch/sketch.hpp, nullspace.hpp); the
compute runs in libnullsketch_b200.so (hand-written sm_100a CUDA) through the
C ABI declared in include/nullsketch_b200.h.
"""
from .sketch import (KINDS, NullspaceResult, SketchedMatrix, SketchOperator, SvdConvergenceError, TlsConditionError,
                     TlsExistenceError, TlsSolution, apply, apply_shard, default_sketch_size, downdate_column,
                     downdate_row, residual_certificate, solve_k, solve_tol, svd_trailing, tls_solve_sketched,
                     tls_solve_exact, tls_error_metrics, TlsErrorMetrics, update_column, update_row)

__all__ = ["KINDS", "NullspaceResult", "SketchedMatrix", "SketchOperator", "SvdConvergenceError", "TlsConditionError",
           "TlsExistenceError", "TlsSolution", "apply", "apply_shard", "default_sketch_size", "downdate_column",
           "downdate_row", "residual_certificate", "solve_k", "solve_tol", "svd_trailing", "tls_solve_sketched",
           "tls_solve_exact", "tls_error_metrics", "TlsErrorMetrics", "update_column", "update_row"]
