"""Distributed single-matrix reverse sweep: the blocked reverse of PAPER.md:689-701
with the columns of L and Abar distributed 1-D block-cyclically over P ranks (include/choldiff.h,
cd_dist_rev_panel / cd_dist_rev_update).

Block K = [j, k) of the reverse partition (the short block at the top left) lives
on rank K mod P.  A rank stores its column blocks side by side -- all n rows -- as a "storage" tensor
of shape (c_loc, n): row t of the tensor is local column t, so the local matrix is column-major with
ld = n.  Per block, right to left:

    owner:  panel   Cbar <- Cbar D^-1; Dbar <- Dbar - tril(Cbar^T C); Dbar <- chol_unblocked_rev(D, Dbar);
                    X = [S; Cbar], S = Dbar + Dbar^T
    all:    X broadcast from the owner (the one exchange per block: (n - j) x w elements)
    all:    update  Bbar <- Bbar - Cbar R;  Rbar <- Rbar - X^T [R; B]  on the rank's columns left
                    of the panel (a prefix of its storage: its blocks are stored in order)

Forward mode on the same distribution and partition, blocks left to right:

    all:    partial Z_r = [Adot L][j:n, cols] [L Adot][j:k, cols]^T over the rank's columns left of
                    the block (its share of [Rdot R^T + R Rdot^T ; Bdot R^T + B Rdot^T])
    all:    sum-reduce of Z onto the owner (the one exchange per block)
    owner:  panel   Ddot -= tril(Z_top); Cdot -= Z_bottom; Ddot <- chol_unblocked_fwd(D, Ddot);
                    Cdot <- (Cdot - C Ddot^T) D^-T

Every arithmetic step runs in libcholdiff's kernels (CudaSteps); this module is the host loop and the
ownership bookkeeping.  `bcast(tensor, src_rank)` is torch.distributed.broadcast for a process group
(chol_rev_distributed) or a no-op when all ranks live in one process (chol_rev_loopback, which runs
the same loop for P simulated ranks on one device -- the single-GPU check of the schedule).
"""
from __future__ import annotations

import ctypes

import torch

from . import CholdiffError, _check, _dt, lib


def reverse_blocks(n: int, nb: int) -> list[tuple[int, int]]:
    """(j, w) of blocks K = 0..nblk-1 of the reverse partition: block 0 holds the n mod nb remainder."""
    r = n % nb
    out = [(0, r)] if r else []
    j = r
    while j < n:
        out.append((j, nb))
        j += nb
    return out


def owned_blocks(n: int, nb: int, rank: int, world: int) -> list[tuple[int, int, int, int]]:
    """(K, j, w, local column offset) of the blocks rank `rank` owns, in storage order."""
    out, co = [], 0
    for K, (j, w) in enumerate(reverse_blocks(n, nb)):
        if K % world == rank:
            out.append((K, j, w, co))
            co += w
    return out


def local_columns(M: torch.Tensor, nb: int, rank: int, world: int) -> torch.Tensor:
    """Storage tensor (c_loc, n) of rank `rank`'s column blocks of the logical (n, n) matrix M."""
    n = M.shape[-1]
    cols = [M[:, j:j + w].t() for (_, j, w, _) in owned_blocks(n, nb, rank, world)]
    if not cols:
        return M.new_empty((0, n))
    return torch.cat(cols, 0).contiguous()


def assemble(parts: list[torch.Tensor], n: int, nb: int) -> torch.Tensor:
    """Logical (n, n) matrix from the storage tensors of all ranks (inverse of local_columns)."""
    world = len(parts)
    out = parts[0].new_zeros((n, n))
    for r in range(world):
        for (_, j, w, co) in owned_blocks(n, nb, r, world):
            out[:, j:j + w] = parts[r][co:co + w].t()
    return out


class CudaSteps:
    """The two steps on libcholdiff (device storage tensors, the current CUDA stream)."""

    def __init__(self, device: torch.device, dtype: torch.dtype, nb: int):
        self.L = lib()
        self.dt = _dt(torch.empty(0, dtype=dtype))
        self.ws_bytes = int(self.L.cd_dist_workspace_size(self.dt, nb))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=device)
        self.device = device

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def panel(self, n, j, w, Lk, Ak, X):
        _check(self.L.cd_dist_rev_panel(self.dt, n, j, w, Lk.data_ptr(), n, Ak.data_ptr(), n, X.data_ptr(), n - j,
                                        self.ws.data_ptr(), self.ws_bytes, self._stream()))

    def update(self, n, j, w, X, q, Lq, Aq):
        if q == 0:
            return
        _check(self.L.cd_dist_rev_update(self.dt, n, j, w, X.data_ptr(), n - j, q, Lq.data_ptr(), n,
                                         Aq.data_ptr(), n, self.ws.data_ptr(), self.ws_bytes, self._stream()))

    def fwd_partial(self, n, j, w, q, Lq, Aq, Z):
        lp = Lq.data_ptr() if q else None
        ap = Aq.data_ptr() if q else None
        _check(self.L.cd_dist_fwd_partial(self.dt, n, j, w, q, lp, n, ap, n, Z.data_ptr(), n - j,
                                          self.ws.data_ptr(), self.ws_bytes, self._stream()))

    def fwd_panel(self, n, j, w, Lk, Ak, Z):
        _check(self.L.cd_dist_fwd_panel(self.dt, n, j, w, Lk.data_ptr(), n, Ak.data_ptr(), n, Z.data_ptr(), n - j,
                                        self.ws.data_ptr(), self.ws_bytes, self._stream()))


def run_schedule(n: int, nb: int, rank: int, world: int, Lloc: torch.Tensor, Aloc: torch.Tensor, steps, bcast,
                 xbuf: torch.Tensor | None = None) -> torch.Tensor:
    """The host loop of one rank: Aloc (storage of tril(Lbar) columns) -> tril(Sigma_bar) columns, in place."""
    mine = {K: (j, w, co) for (K, j, w, co) in owned_blocks(n, nb, rank, world)}
    blocks = reverse_blocks(n, nb)
    X = xbuf if xbuf is not None else Aloc.new_empty(n * nb)
    for K in range(len(blocks) - 1, -1, -1):
        j, w = blocks[K]
        Xk = X[: (n - j) * w]
        owner = K % world
        if owner == rank:
            _, _, co = mine[K]
            steps.panel(n, j, w, Lloc[co:co + w], Aloc[co:co + w], Xk)
        bcast(Xk, owner)
        q = sum(ww for (KK, (_, ww, _)) in mine.items() if KK < K)
        steps.update(n, j, w, Xk, q, Lloc[:q], Aloc[:q])
    return Aloc


def run_schedule_fwd(n: int, nb: int, rank: int, world: int, Lloc: torch.Tensor, Aloc: torch.Tensor, steps,
                     reduce, zbuf: torch.Tensor | None = None) -> torch.Tensor:
    """Forward host loop of one rank: Aloc (storage of tril(Sigma_dot) columns) -> L_dot columns, in place.
    `reduce(tensor, dst_rank)` sums the ranks' tensors onto dst."""
    mine = {K: (j, w, co) for (K, j, w, co) in owned_blocks(n, nb, rank, world)}
    Z = zbuf if zbuf is not None else Aloc.new_empty(n * nb)
    for K, (j, w) in enumerate(reverse_blocks(n, nb)):
        Zk = Z[: (n - j) * w]
        q = sum(ww for (KK, (_, ww, _)) in mine.items() if KK < K)
        steps.fwd_partial(n, j, w, q, Lloc[:q], Aloc[:q], Zk)
        owner = K % world
        reduce(Zk, owner)
        if owner == rank:
            _, _, co = mine[K]
            steps.fwd_panel(n, j, w, Lloc[co:co + w], Aloc[co:co + w], Zk)
    return Aloc


def chol_fwd_distributed(Lloc: torch.Tensor, Aloc: torch.Tensor, n: int, nb: int = 128, group=None,
                         steps=None) -> torch.Tensor:
    """One rank of the distributed forward sweep (Aloc: storage of tril(Sigma_dot) -> L_dot)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if Lloc.shape != Aloc.shape or Lloc.dtype != Aloc.dtype:
        raise ValueError("Lloc and Aloc must be storage tensors of the same shape and dtype")
    if steps is None:
        if not Aloc.is_cuda:
            raise CholdiffError("chol_fwd_distributed runs on CUDA storage tensors (no CPU fallback)")
        steps = CudaSteps(Aloc.device, Aloc.dtype, nb)
    ranks = None if group is None else dist.get_process_group_ranks(group)

    def reduce(t, dst):
        dist.reduce(t, dst if ranks is None else ranks[dst], op=dist.ReduceOp.SUM, group=group)

    return run_schedule_fwd(n, nb, rank, world, Lloc, Aloc, steps, reduce)


def chol_fwd_loopback(L: torch.Tensor, Sdot: torch.Tensor, nb: int, world: int, steps=None) -> torch.Tensor:
    """The distributed forward schedule for `world` simulated ranks in this process: each rank's partial
    is computed into its own buffer and summed in place of the reduction; returns L_dot (n, n)."""
    n = L.shape[-1]
    Ls = [local_columns(L, nb, r, world) for r in range(world)]
    As = [local_columns(Sdot, nb, r, world) for r in range(world)]
    if steps is None:
        if not L.is_cuda:
            raise CholdiffError("chol_fwd_loopback runs on CUDA tensors (no CPU fallback)")
        steps = CudaSteps(L.device, L.dtype, nb)
    mine = [{K: (j, w, co) for (K, j, w, co) in owned_blocks(n, nb, r, world)} for r in range(world)]
    Zs = [L.new_empty(n * nb) for _ in range(world)]
    for K, (j, w) in enumerate(reverse_blocks(n, nb)):
        m = (n - j) * w
        for r in range(world):
            q = sum(ww for (KK, (_, ww, _)) in mine[r].items() if KK < K)
            steps.fwd_partial(n, j, w, q, Ls[r][:q], As[r][:q], Zs[r][:m])
        o = K % world
        for r in range(world):
            if r != o:
                Zs[o][:m] += Zs[r][:m]  # the reduction (a device add; the arithmetic of the method stays in the steps)
        _, _, co = mine[o][K]
        steps.fwd_panel(n, j, w, Ls[o][co:co + w], As[o][co:co + w], Zs[o][:m])
    return assemble(As, n, nb)


def chol_rev_distributed(Lloc: torch.Tensor, Aloc: torch.Tensor, n: int, nb: int = 128, group=None,
                         steps=None) -> torch.Tensor:
    """One rank of the distributed sweep over a torch.distributed process group (NCCL for CUDA
    tensors).  Lloc / Aloc: this rank's storage tensors (local_columns)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if Lloc.shape != Aloc.shape or Lloc.dtype != Aloc.dtype:
        raise ValueError("Lloc and Aloc must be storage tensors of the same shape and dtype")
    if steps is None:
        if not Aloc.is_cuda:
            raise CholdiffError("chol_rev_distributed runs on CUDA storage tensors (no CPU fallback)")
        steps = CudaSteps(Aloc.device, Aloc.dtype, nb)
    ranks = None if group is None else dist.get_process_group_ranks(group)

    def bcast(t, src):
        dist.broadcast(t, src if ranks is None else ranks[src], group=group)

    return run_schedule(n, nb, rank, world, Lloc, Aloc, steps, bcast)


def chol_rev_loopback(L: torch.Tensor, Lbar: torch.Tensor, nb: int, world: int, steps=None) -> torch.Tensor:
    """The distributed schedule for `world` simulated ranks in this process (one device): split the
    logical (n, n) matrices into per-rank storage, run the ranks' steps in lock step with the owner's
    X shared in place of the broadcast, and assemble tril(Sigma_bar)."""
    n = L.shape[-1]
    Ls = [local_columns(L, nb, r, world) for r in range(world)]
    As = [local_columns(Lbar, nb, r, world) for r in range(world)]
    if steps is None:
        if not L.is_cuda:
            raise CholdiffError("chol_rev_loopback runs on CUDA tensors (no CPU fallback)")
        steps = CudaSteps(L.device, L.dtype, nb)
    mine = [{K: (j, w, co) for (K, j, w, co) in owned_blocks(n, nb, r, world)} for r in range(world)]
    blocks = reverse_blocks(n, nb)
    X = L.new_empty(n * nb)
    for K in range(len(blocks) - 1, -1, -1):
        j, w = blocks[K]
        Xk = X[: (n - j) * w]
        o = K % world
        _, _, co = mine[o][K]
        steps.panel(n, j, w, Ls[o][co:co + w], As[o][co:co + w], Xk)
        for r in range(world):
            q = sum(ww for (KK, (_, ww, _)) in mine[r].items() if KK < K)
            steps.update(n, j, w, Xk, q, Ls[r][:q], As[r][:q])
    return assemble(As, n, nb)
