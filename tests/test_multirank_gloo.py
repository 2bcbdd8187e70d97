"""World-size-2 gloo tests of the row-sharded path (CPU only).

The partial sketch of each rank is computed by the oracle on the rank's
rows (placed at their global positions), the ranks all-reduce through
torch.distributed exactly as the NCCL path does, and the sum must equal the
oracle's single-process apply.  This covers row_partition (contiguous and
cyclic maps), sharded_apply and sharded_solve_k's broadcast.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_00975_b200.distributed import local_rows, row_partition, sharded_apply, sharded_solve_k


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_partial(kind, s, m, seed, n):
    from oracle import sketch_oracle as O
    op = O.draw(kind, s, m, seed)

    def fn(S, A_local, row0, rstep):
        full = np.zeros((m, n))
        full[row0: row0 + rstep * A_local.shape[0]: rstep] = A_local.numpy()
        return torch.from_numpy(np.ascontiguousarray(O.apply(op, full)))
    return fn


def _worker(rank, world, port, kind, s, m, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sketch_oracle as O
        A = O.random_real(m, n, 3)
        shard = row_partition(m, world, kind)[rank]
        A_loc = torch.from_numpy(np.ascontiguousarray(local_rows(A, shard)))
        fn = _oracle_partial(kind, s, m, seed, n)
        SA = sharded_apply(None, A_loc, shard, partial_fn=fn)

        def svd_fn(SA_, k):
            _, sv, vh = np.linalg.svd(SA_.numpy(), full_matrices=False)
            return torch.from_numpy(vh.T[:, n - k:].copy()), torch.from_numpy(sv.copy())
        W, sig = sharded_solve_k(None, A_loc, 2, shard, partial_fn=fn, svd_fn=svd_fn)
        q.put((rank, SA.numpy(), W.numpy(), sig.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,m", [("gaussian", 3001), ("srht", 4096), ("countsketch", 5000), ("srdct", 999),
                                    ("srft", 1000)])
def test_two_rank_sharded_apply_matches_single(kind, m):
    from oracle import sketch_oracle as O
    O.build()
    world, s, n, seed = 2, 48, 6, 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, s, m, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = O.random_real(m, n, 3)
    ref = O.apply(O.draw(kind, s, m, seed), A)
    for rank, SA, W, sig in out:
        assert np.linalg.norm(SA - ref) <= 1e-12 * np.linalg.norm(ref)
    # every rank holds the root's W and sigma
    assert np.array_equal(out[0][2], out[1][2]) and np.array_equal(out[0][3], out[1][3])


@pytest.mark.parametrize("kind", ["gaussian", "srht", "countsketch", "srdct", "srft"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_row_partition_covers_rows_once(kind, world):
    for m in (1, 7, 1024, 4096, 10**5 + 3, 1 << 20):
        if kind == "srht" and m & (m - 1):
            continue
        shards = row_partition(m, world, kind)
        rows = np.concatenate([np.fromiter(sh.global_rows(), dtype=np.int64, count=sh.mloc) for sh in shards])
        assert np.array_equal(np.sort(rows), np.arange(m))
        if kind == "srht" and m >= 2048 * world:
            assert all(sh.row0 % 2048 == 0 and sh.mloc % 2048 == 0 for sh in shards)
        if kind == "countsketch" and m >= 512 * world:
            assert all(sh.row0 % 512 == 0 for sh in shards)


def _dit_worker(rank, world, port, kind, s, m, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sketch_oracle as O
        A = O.random_real(m, n, 3)
        shard = row_partition(m, world, kind)[rank]
        assert (shard.row0, shard.rstep) == (rank, world)  # cyclic map
        op = O.draw(kind, s, m, seed)

        def fn(S, A_local, row0, rstep):  # the decimation-in-time local transform, not a zero-filled apply
            part = O.srtt_shard_partial(op, A_local.numpy(), row0, rstep)
            return torch.from_numpy(np.ascontiguousarray(part))
        A_loc = torch.from_numpy(np.ascontiguousarray(local_rows(A, shard)))
        SA = sharded_apply(None, A_loc, shard, partial_fn=fn)
        q.put((rank, SA.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,m,world", [("srft", 1000, 2), ("srdct", 1000, 2), ("srft", 4096, 4), ("srdct", 840, 4)])
def test_cyclic_shards_decimation_in_time(kind, m, world):
    """srft / srdct across ranks: each rank's partial is its local length-m/P transform, twiddled
    and gathered (oracle.srtt_shard_partial, the algorithm srtt_general.cu / srtt_fast.cu run on the
    GPU); the gloo all-reduce of the partials equals the single-process apply."""
    from oracle import sketch_oracle as O
    O.build()
    s, n, seed = 40, 5, 23
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dit_worker, args=(r, world, port, kind, s, m, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.apply(O.draw(kind, s, m, seed), O.random_real(m, n, 3))
    for rank, SA in out:
        assert np.linalg.norm(SA - ref) <= 1e-12 * np.linalg.norm(ref)
