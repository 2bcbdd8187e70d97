"""Row-sharded multi-GPU sketching: one process per GPU, NCCL over NVLink.

SA = sum_g S[:, rows_g] A_g, so each rank sketches the rows it holds with
nsk_apply_shard (the operator regenerates S for the *global* row indices;
nothing is communicated before the reduce) and one all-reduce (sum) of the
s x n partials -- 2 MiB at BASELINE configs[1] -- produces SA on every rank.
The SVD of the small SA then runs on the root rank (or every rank).

Row maps:
  gaussian, countsketch, srht   contiguous shards (srht: multiples of 2048
                                rows so the Hadamard split stays block-aligned;
                                countsketch: multiples of 12288 rows, or 512 for short matrices;
                                each rank builds CountSketch tables for its own rows only)
  srft, srdct                   cyclic shards: rank g holds rows g, g+P, ...
                                (decimation in time: one local length-m/P
                                transform, a twiddle and the sampled gather)

Two reduce paths: sharded_apply / sharded_solve_k all-reduce with
torch.distributed (any backend; the gloo tests use it), and NcclComm +
sharded_apply_nccl / sharded_solve_k_nccl go through the library's C ABI
(nsk_apply_allreduce / nsk_solve_k_sharded), which own the NCCL all-reduce
themselves -- the path a C++ caller of the reference API uses.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional


@dataclasses.dataclass(frozen=True)
class RowShard:
    row0: int
    rstep: int
    mloc: int

    def global_rows(self):
        return range(self.row0, self.row0 + self.rstep * self.mloc, self.rstep) if self.mloc else range(0)


def _align_for(kind: str) -> int:
    return {"srht": 2048, "countsketch": 512}.get(kind, 1)


def row_partition(m: int, world: int, kind: str) -> List[RowShard]:
    """Per-rank row shards covering 0..m-1 exactly once."""
    if world < 1:
        raise ValueError("world size must be positive")
    if kind in ("srft", "srdct"):
        return [RowShard(g, world, (m - g + world - 1) // world if g < m else 0) for g in range(world)]
    align = _align_for(kind)
    if kind == "countsketch":
        # 12288 = lcm of the owner kernel's 3072/4096-row schedule tiles: every
        # shard starts on a tile; short matrices keep the kernels' 512-row rule.
        align = 12288 if m >= 12288 * world else 512
    elif m < align * world:
        align = 1
    units = (m + align - 1) // align
    shards = []
    for g in range(world):
        u0 = units * g // world
        u1 = units * (g + 1) // world
        r0 = min(m, u0 * align)
        r1 = min(m, u1 * align)
        shards.append(RowShard(r0, 1, r1 - r0))
    return shards


def local_rows(A_full, shard: RowShard):
    """The rows of a full matrix a rank would hold (tests and examples)."""
    return A_full[shard.row0: shard.row0 + shard.rstep * shard.mloc: shard.rstep]


def sharded_apply(S, A_local, shard: RowShard, group=None,
                  partial_fn: Optional[Callable] = None):
    """SA on every rank: local partial sketch + all-reduce(sum).

    partial_fn(S, A_local, row0, rstep) defaults to the CUDA path
    (paper_2206_00975_b200.apply_shard); tests inject a CPU oracle."""
    import torch.distributed as dist
    if partial_fn is None:
        from .sketch import apply_shard
        partial_fn = apply_shard
    part = partial_fn(S, A_local, shard.row0, shard.rstep)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part


def sharded_solve_k(S, A_local, k: int, shard: RowShard, group=None, root: int = 0,
                    partial_fn: Optional[Callable] = None, svd_fn: Optional[Callable] = None):
    """solve_k over row shards: (W, sigma) on every rank (broadcast from root)."""
    import torch
    import torch.distributed as dist
    SA = sharded_apply(S, A_local, shard, group, partial_fn)
    if svd_fn is None:
        from .sketch import svd_trailing
        svd_fn = svd_trailing
    n = SA.shape[1]
    multi = dist.is_initialized() and dist.get_world_size(group) > 1
    if not multi or dist.get_rank(group) == root:
        W, sig = svd_fn(SA, k)
        W = W.contiguous()
    else:
        W = torch.empty((n, k), dtype=SA.dtype, device=SA.device)
        sig = torch.empty(n, dtype=torch.float64, device=SA.device)
    if multi:
        dist.broadcast(W, src=root, group=group)
        dist.broadcast(sig, src=root, group=group)
    return W, sig


class NcclComm:
    """An NCCL communicator owned by the library (nsk_nccl_comm_init); the unique id is
    distributed over torch.distributed (any backend).  world/rank default to the process group's."""

    def __init__(self, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib
        L = _lib.load()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(L.nsk_nccl_unique_id(uid))
        if self.world > 1:
            box = [uid.raw]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        h = ctypes.c_void_p()
        _lib.check(L.nsk_nccl_comm_init(self.world, uid, self.rank, ctypes.byref(h)))
        self.handle = h

    def close(self):
        from . import _lib
        if self.handle is not None and self.handle.value:
            _lib.check(_lib.load().nsk_nccl_comm_destroy(self.handle))
        self.handle = None


def sharded_apply_nccl(S, A_local, shard: RowShard, comm: NcclComm):
    """SA on every rank through the C ABI: nsk_apply_allreduce (partial + ncclAllReduce)."""
    import ctypes

    import torch

    from . import _lib
    from .sketch import _colmajor, _empty_colmajor, _out_dtype_is_complex, _scalar_of, _stream_ptr
    L = _lib.load()
    scalar = _scalar_of(A_local)
    A_local, lda = _colmajor(A_local)
    mloc, n = A_local.shape
    dt = torch.complex128 if _out_dtype_is_complex(S, scalar) else torch.float64
    SA = _empty_colmajor(S.s, n, dt, A_local.device)
    _lib.check(L.nsk_apply_allreduce(S.handle, scalar, shard.row0, shard.rstep, mloc, n,
                                     ctypes.c_void_p(A_local.data_ptr()), lda, ctypes.c_void_p(SA.data_ptr()), S.s,
                                     comm.handle, _stream_ptr()))
    return SA


def sharded_solve_k_nccl(S, A_local, k: int, shard: RowShard, comm: NcclComm):
    """(W, sigma) on every rank through the C ABI: nsk_solve_k_sharded."""
    import ctypes

    import torch

    from . import _lib
    from .sketch import _colmajor, _empty_colmajor, _out_dtype_is_complex, _scalar_of, _stream_ptr
    L = _lib.load()
    scalar = _scalar_of(A_local)
    A_local, lda = _colmajor(A_local)
    mloc, n = A_local.shape
    dt = torch.complex128 if _out_dtype_is_complex(S, scalar) else torch.float64
    W = _empty_colmajor(n, max(k, 0), dt, A_local.device)
    sig = torch.empty(n, dtype=torch.float64, device=A_local.device)
    _lib.check(L.nsk_solve_k_sharded(S.handle, scalar, shard.row0, shard.rstep, mloc, n,
                                     ctypes.c_void_p(A_local.data_ptr()), lda, int(k), ctypes.c_void_p(W.data_ptr()),
                                     max(n, 1), ctypes.c_void_p(sig.data_ptr()), comm.handle, _stream_ptr()))
    return W, sig


def sharded_solve_k_host_nccl(S, A_host, k: int, shard: RowShard, comm: NcclComm):
    """(W, sigma) on every rank from the rank's shard in HOST memory: nsk_solve_k_sharded_host (a
    contiguous shard streams in row chunks that are sketched as they land; then ncclAllReduce and
    the SVD on every rank).  numpy in, numpy out."""
    import ctypes

    import numpy as np

    from . import _lib
    from .sketch import NSK_COMPLEX, NSK_REAL
    L = _lib.load()
    cplx = np.iscomplexobj(A_host)
    A = np.asfortranarray(A_host, dtype=np.complex128 if cplx else np.float64)
    mloc, n = A.shape
    cplx_out = cplx or S.kind == "srft"
    W = np.empty((n, max(k, 0)), dtype=np.complex128 if cplx_out else np.float64, order="F")
    sig = np.empty(n)
    _lib.check(L.nsk_solve_k_sharded_host(S.handle, NSK_COMPLEX if cplx else NSK_REAL, shard.row0, shard.rstep, mloc,
                                          n, A.ctypes.data_as(ctypes.c_void_p), max(mloc, 1), int(k),
                                          W.ctypes.data_as(ctypes.c_void_p), max(n, 1),
                                          sig.ctypes.data_as(ctypes.c_void_p), comm.handle))
    return W, sig
