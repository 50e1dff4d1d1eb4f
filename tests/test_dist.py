"""Distributed single-matrix reverse sweep (paper_1602_07527_b200/dist.py).
CPU: the schedule with the numpy step engine (tests/dist_steps.py) for several simulated rank counts,
and world_size-2 gloo ranks exchanging the panel broadcasts; both against the oracle.  The CUDA steps
(cd_dist_rev_panel / _update) are checked by the -m gpu tests at the end."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthetic
from dist_steps import NumpySteps
from paper_1602_07527_b200 import dist as cdd


def _rel(out, ref):
    return np.abs(np.tril(out) - np.tril(ref)).max() / np.linalg.norm(np.tril(ref))


def test_partition_and_ownership():
    for n, nb in [(300, 128), (256, 128), (37, 8), (5, 8)]:
        blocks = cdd.reverse_blocks(n, nb)
        assert blocks[0][0] == 0 and sum(w for _, w in blocks) == n
        assert all(w == nb for _, w in blocks[1:]) and 0 < blocks[0][1] <= nb  # short block top left
        for world in (1, 2, 3):
            owned = [cdd.owned_blocks(n, nb, r, world) for r in range(world)]
            Ks = sorted(K for o in owned for (K, _, _, _) in o)
            assert Ks == list(range(len(blocks)))
            M = torch.arange(n * n, dtype=torch.float64).reshape(n, n)
            parts = [cdd.local_columns(M, nb, r, world) for r in range(world)]
            assert torch.equal(cdd.assemble(parts, n, nb), M)


@pytest.mark.parametrize("n,nb,world", [(40, 8, 1), (40, 8, 2), (37, 8, 3), (64, 16, 2), (50, 16, 4)])
def test_loopback_schedule_matches_oracle(n, nb, world):
    L, Lb, _ = synthetic.draw(n, 900 + n)
    Lb_poison = Lb + np.triu(np.full((n, n), np.nan), 1)  # the upper triangle must never be read
    out = cdd.chol_rev_loopback(torch.from_numpy(L), torch.from_numpy(Lb_poison), nb, world, steps=NumpySteps())
    assert _rel(out.numpy(), oracle.chol_rev(L, Lb)) < 1e-12


@pytest.mark.parametrize("n,nb,world", [(40, 8, 1), (40, 8, 2), (37, 8, 3), (50, 16, 4)])
def test_loopback_fwd_schedule_matches_oracle(n, nb, world):
    L, _, Sd = synthetic.draw(n, 950 + n, lbar=False, sdot=True)
    S_poison = np.tril(Sd) + np.triu(np.full((n, n), np.nan), 1)
    out = cdd.chol_fwd_loopback(torch.from_numpy(L), torch.from_numpy(S_poison), nb, world, steps=NumpySteps())
    ref = oracle.chol_fwd(L, Sd)
    assert _rel(out.numpy(), ref) < 1e-12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, nb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, Lb, _ = synthetic.draw(n, 77)
        Lloc = cdd.local_columns(torch.from_numpy(L), nb, rank, world)
        Aloc = cdd.local_columns(torch.from_numpy(Lb), nb, rank, world)
        cdd.chol_rev_distributed(Lloc, Aloc, n, nb, steps=NumpySteps())
        gathered = [None] * world
        dist.all_gather_object(gathered, Aloc)
        _, _, Sd = synthetic.draw(n, 78, lbar=False, sdot=True)
        Sloc = cdd.local_columns(torch.from_numpy(np.tril(Sd)), nb, rank, world)
        cdd.chol_fwd_distributed(Lloc, Sloc, n, nb, steps=NumpySteps())
        gathered_f = [None] * world
        dist.all_gather_object(gathered_f, Sloc)
        if rank == 0:
            q.put((cdd.assemble(gathered, n, nb).numpy(), cdd.assemble(gathered_f, n, nb).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nb", [(45, 8), (48, 16)])
def test_two_rank_gloo_matches_oracle(n, nb):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    out, outf = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    L, Lb, _ = synthetic.draw(n, 77)
    assert _rel(out, oracle.chol_rev(L, Lb)) < 1e-12
    _, _, Sd = synthetic.draw(n, 78, lbar=False, sdot=True)
    assert _rel(outf, oracle.chol_fwd(L, Sd)) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,nb,world,dt", [(300, 128, 2, torch.float64), (300, 128, 3, torch.float64),
                                           (1000, 64, 3, torch.float64), (1000, 128, 4, torch.float64),
                                           (513, 128, 2, torch.float32), (256, 128, 1, torch.float64),
                                           (40, 16, 2, torch.float64)])
def test_gpu_loopback_matches_oracle(n, nb, world, dt):
    from gpu_helpers import fp32_round
    L, Lb, _ = synthetic.draw(n, 1300 + n)
    if dt == torch.float32:
        L, Lb = fp32_round(L, Lb)
    Lb_poison = Lb + np.triu(np.full((n, n), np.nan), 1)
    out = cdd.chol_rev_loopback(torch.from_numpy(L).to(dt).cuda(), torch.from_numpy(Lb_poison).to(dt).cuda(), nb,
                                world)
    torch.cuda.synchronize()
    assert _rel(out.double().cpu().numpy(), oracle.chol_rev(L, Lb)) < (1e-10 if dt == torch.float64 else 1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("n,nb,world,dt", [(300, 128, 2, torch.float64), (1000, 64, 3, torch.float64),
                                           (1000, 128, 4, torch.float64), (513, 128, 2, torch.float32),
                                           (256, 128, 1, torch.float64), (40, 16, 2, torch.float64)])
def test_gpu_fwd_loopback_matches_oracle(n, nb, world, dt):
    from gpu_helpers import fp32_round
    L, _, Sd = synthetic.draw(n, 1700 + n, lbar=False, sdot=True)
    if dt == torch.float32:
        L, Sd = fp32_round(L, Sd)
    S_poison = np.tril(Sd) + np.triu(np.full((n, n), np.nan), 1)
    out = cdd.chol_fwd_loopback(torch.from_numpy(L).to(dt).cuda(), torch.from_numpy(S_poison).to(dt).cuda(), nb,
                                world)
    torch.cuda.synchronize()
    assert _rel(out.double().cpu().numpy(), oracle.chol_fwd(L, Sd)) < (1e-10 if dt == torch.float64 else 1e-4)


@pytest.mark.gpu
def test_gpu_nccl_single_rank_group():
    # the torch.distributed path itself (NCCL broadcasts of X) on a one-rank group
    n, nb = 700, 128
    L, Lb, _ = synthetic.draw(n, 4242)
    store = dist.HashStore()
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        Lloc = cdd.local_columns(torch.from_numpy(L).cuda(), nb, 0, 1)
        Aloc = cdd.local_columns(torch.from_numpy(Lb).cuda(), nb, 0, 1)
        cdd.chol_rev_distributed(Lloc, Aloc, n, nb)
        out = cdd.assemble([Aloc], n, nb)
        _, _, Sd = synthetic.draw(n, 4243, lbar=False, sdot=True)
        Sloc = cdd.local_columns(torch.from_numpy(np.tril(Sd)).cuda(), nb, 0, 1)
        cdd.chol_fwd_distributed(Lloc, Sloc, n, nb)
        outf = cdd.assemble([Sloc], n, nb)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    assert _rel(out.cpu().numpy(), oracle.chol_rev(L, Lb)) < 1e-10
    assert _rel(outf.cpu().numpy(), oracle.chol_fwd(L, Sd)) < 1e-10
