"""N > 1 path on CPU: world_size-2 gloo ranks exercise the by-matrix partition and
the gather (paper_1602_07527_b200/shard.py) with the CPU oracle standing in for the
per-rank kernel (SURVEY §4 "fake backends").  The CUDA kernels themselves are
covered by the -m gpu tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1602_07527_b200.shard import chol_fwd_sharded, chol_rev_sharded, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_rev(L, Lb):
    import oracle
    out = np.stack([oracle.chol_rev(L[b].numpy(), Lb[b].numpy()) for b in range(L.shape[0])])
    return torch.from_numpy(out)


def _oracle_fwd(L, Sd):
    import oracle
    out = np.stack([oracle.chol_fwd(L[b].numpy(), Sd[b].numpy()) for b in range(L.shape[0])])
    return torch.from_numpy(out)


def _worker(rank, world, port, n, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synthetic
        lo, hi = shard_range(total, world, rank)
        L, Lb, Sd = synthetic.draw_batch(n, hi - lo, seed=0, sdot=True, start=lo)
        Lt, Lbt, Sdt = (torch.from_numpy(a) for a in (L, Lb, np.tril(Sd)))
        rev = chol_rev_sharded(Lt, Lbt, total, compute=lambda a, b: _oracle_rev(a, b))
        fwd = chol_fwd_sharded(Lt, Sdt, total, compute=lambda a, b: _oracle_fwd(a, b))
        if rank == 0:
            q.put((rev.contiguous().numpy(), fwd.contiguous().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 7])
def test_two_rank_shard_and_gather_matches_single_process(total):
    import oracle
    import synthetic
    n, world = 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    rev, fwd = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    L, Lb, Sd = synthetic.draw_batch(n, total, seed=0, sdot=True)
    for b in range(total):
        assert np.array_equal(rev[b], oracle.chol_rev(L[b], Lb[b]))
        assert np.array_equal(fwd[b], oracle.chol_fwd(L[b], np.tril(Sd[b])))


def test_shard_range_partitions():
    for total in (0, 1, 7, 8, 65536, 65537):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
