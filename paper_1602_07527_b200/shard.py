"""Batched workloads across ranks (one process per GPU): shard by matrix, no
data-path collective, one gather at the end.

Matrices are independent units, so rank r of P owns the contiguous range
``shard_range(total, P, r)``, generates / holds only that shard, runs the batched
kernel locally, and -- if the caller wants the whole result on every rank -- the
outputs are collected with one all-gather (NCCL ``all_gather_into_tensor`` over
NVLink when the shards are equal-sized, a padded all-gather otherwise).  Single
large matrices do not shard (the panel chain of the blocked sweep is sequential):
they run as independent replicas.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) range of matrix indices owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_batches(local: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather per-rank shards of shape (B_r, N, N) into (total, N, N) on every rank
    (rank order = matrix order).  Column-major per-matrix memory is preserved."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = local.shape[-1]
    sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank} holds {local.shape[0]} matrices, expected {sizes[rank]}")
    src = local.transpose(-1, -2).contiguous()  # bytes of the column-major layout
    m = max(sizes)
    if all(s == m for s in sizes):
        out = torch.empty((total, n, n), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, src, group=group)
    else:
        pad = torch.zeros((m, n, n), dtype=local.dtype, device=local.device)
        pad[: src.shape[0]] = src
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        out = torch.cat([bufs[r][: sizes[r]] for r in range(world)], dim=0)
    return out.transpose(-1, -2)


def chol_rev_sharded(L_local: torch.Tensor, Lbar_local: torch.Tensor, total: int, *, group=None,
                     gather: bool = True, compute=None, **kw):
    """Reverse mode on this rank's shard; optionally gather the whole batch.

    ``compute(L, Lbar, **kw)`` defaults to the CUDA kernels (``chol_rev``); tests pass
    a CPU stand-in to exercise the partition / gather logic on gloo ranks."""
    if compute is None:
        from . import chol_rev as compute
    out = compute(L_local, Lbar_local, **kw)
    return gather_batches(out, total, group) if gather else out


def chol_fwd_sharded(L_local: torch.Tensor, Sdot_local: torch.Tensor, total: int, *, group=None,
                     gather: bool = True, compute=None, **kw):
    if compute is None:
        from . import chol_fwd as compute
    out = compute(L_local, Sdot_local, **kw)
    return gather_batches(out, total, group) if gather else out
