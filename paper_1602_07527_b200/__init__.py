"""paper_1602_07527_b200 -- thin Python binding of libcholdiff.so (include/choldiff.h).

Derivatives of the Cholesky decomposition Sigma = L L^T on B200 (arXiv 1602.07527):

* ``chol_rev(L, Lbar)``  -> tril(Sigma_bar)  (reverse mode)
* ``chol_fwd(L, Sdot)``  -> L_dot            (forward mode)

Arguments are torch CUDA tensors (float64 or float32) holding one (N, N) matrix or
a batch (B, N, N), in *logical* orientation with COLUMN-MAJOR memory per matrix,
i.e. ``t.stride(-2) == 1`` (``colmajor(t)`` makes such a copy).  Only lower
triangles are read.  The computation is in place on the second argument (as in
the paper) unless ``inplace=False``: a column-major second argument is updated
directly; any other layout is processed in a column-major copy whose result is
copied back into the caller's tensor, so the in-place contract holds for every
layout (the returned tensor is always the caller's).

Numerical status (SPEC.md's SingularFactorError; include/choldiff.h d_info) is
asynchronous: ``info=True`` returns the per-matrix status tensor without a
synchronisation; ``check=True`` synchronises and raises
:class:`SingularFactorError` when some L[j, j] is zero or non-finite.  The
default (neither) never synchronises, so the calls can be captured in CUDA
graphs and timed back to back; a singular factor then yields unspecified
(non-finite) outputs.

This module only marshals arguments (pointers, leading dimensions, the current
torch stream and a workspace tensor) into the C ABI; every arithmetic step runs in
the CUDA kernels of the library.  There is no CPU fallback: if the library is
missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _build

__all__ = ["chol_rev", "chol_fwd", "chol_host", "colmajor", "workspace_size", "lib", "library_path",
           "launch_count", "reset_launch_count", "CholdiffError", "OUT_MODES", "ROUTES", "host_bytes",
           "chol_fwd_fused", "chol_rev_fwd", "SingularFactorError"]

CD_F64, CD_F32 = 0, 1
CD_OP_REV, CD_OP_FWD, CD_OP_CHOL_FWD = 0, 1, 2
ROUTES = {"auto": 0, "algorithmic": 1, "symbolic": 2}
OUT_MODES = {"tril": 0, "sym": 1, "grad": 2}

_lib = None
_lock = threading.Lock()


class CholdiffError(RuntimeError):
    pass


class SingularFactorError(CholdiffError, ValueError):
    """A diagonal entry L[j, j] is zero or non-finite (``.info``: per-matrix 1-based index, 0 = ok)."""

    def __init__(self, info):
        self.info = info
        bad = [(b, int(v)) for b, v in enumerate(info) if v]
        super().__init__(f"singular factor: (matrix, 1-based column) {bad[:8]}{' ...' if len(bad) > 8 else ''}")


class _Opts(ctypes.Structure):
    _fields_ = [("nb", ctypes.c_int32), ("route", ctypes.c_int32), ("out_mode", ctypes.c_int32),
                ("flags", ctypes.c_int32)]


def library_path() -> str:
    return _build.LIB


def lib():
    """Load libcholdiff.so (building it first if the sources are newer)."""
    global _lib
    with _lock:
        if _lib is None:
            path = _build.LIB
            if not os.path.exists(path) or _build.stale():
                _build.build()
            L = ctypes.CDLL(path)
            vp, i64, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
            po = ctypes.POINTER(_Opts)
            for name in ("cd_chol_rev", "cd_chol_fwd"):
                f = getattr(L, name)
                f.argtypes = [ctypes.c_int, i64, vp, i64, vp, i64, po, vp, sz, vp, vp]
                f.restype = ctypes.c_int
            for name in ("cd_chol_rev_strided_batched", "cd_chol_fwd_strided_batched"):
                f = getattr(L, name)
                f.argtypes = [ctypes.c_int, i64, vp, i64, i64, vp, i64, i64, i64, po, vp, sz, vp, vp]
                f.restype = ctypes.c_int
            L.cd_chol_fwd_fused.argtypes = [ctypes.c_int, i64, vp, i64, vp, i64, po, vp, sz, vp, vp]
            L.cd_chol_fwd_fused.restype = ctypes.c_int
            L.cd_chol_fwd_fused_strided_batched.argtypes = [ctypes.c_int, i64, vp, i64, i64, vp, i64, i64, i64, po,
                                                             vp, sz, vp, vp]
            L.cd_chol_fwd_fused_strided_batched.restype = ctypes.c_int
            for name in ("cd_chol_rev_batched", "cd_chol_fwd_batched"):
                f = getattr(L, name)
                f.argtypes = [ctypes.c_int, i64, vp, i64, vp, i64, i64, po, vp, sz, vp, vp]
                f.restype = ctypes.c_int
            L.cd_workspace_size.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, po]
            L.cd_workspace_size.restype = sz
            L.cd_workspace_size_host.argtypes = [ctypes.c_int, ctypes.c_int, i64, po]
            L.cd_workspace_size_host.restype = sz
            L.cd_chol_host.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp, po, vp, sz, vp]
            L.cd_chol_host.restype = ctypes.c_int
            L.cd_dist_workspace_size.argtypes = [ctypes.c_int, i64]
            L.cd_dist_workspace_size.restype = sz
            L.cd_dist_rev_panel.argtypes = [ctypes.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, sz, vp]
            L.cd_dist_rev_panel.restype = ctypes.c_int
            L.cd_dist_rev_update.argtypes = [ctypes.c_int, i64, i64, i64, vp, i64, i64, vp, i64, vp, i64, vp, sz, vp]
            L.cd_dist_rev_update.restype = ctypes.c_int
            L.cd_dist_fwd_partial.argtypes = [ctypes.c_int, i64, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, sz, vp]
            L.cd_dist_fwd_partial.restype = ctypes.c_int
            L.cd_dist_fwd_panel.argtypes = [ctypes.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, sz, vp]
            L.cd_dist_fwd_panel.restype = ctypes.c_int
            L.cd_workspace_size_rev_fwd.argtypes = [ctypes.c_int, i64, i64, po]
            L.cd_workspace_size_rev_fwd.restype = sz
            L.cd_chol_rev_fwd_strided_batched.argtypes = [ctypes.c_int, i64, vp, i64, i64, vp, i64, i64, vp, i64,
                                                          i64, i64, po, vp, sz, vp, vp]
            L.cd_chol_rev_fwd_strided_batched.restype = ctypes.c_int
            L.cd_status_string.argtypes = [ctypes.c_int]
            L.cd_status_string.restype = ctypes.c_char_p
            L.cd_last_cuda_error.restype = ctypes.c_char_p
            L.cd_version.restype = ctypes.c_int
            L.cd_launch_count.restype = i64
            L.cd_reset_launch_count.restype = None
            _lib = L
    return _lib


def launch_count() -> int:
    return int(lib().cd_launch_count())


def reset_launch_count() -> None:
    lib().cd_reset_launch_count()


def _check(rc: int):
    if rc != 0:
        L = lib()
        msg = L.cd_status_string(rc).decode()
        if rc == 1:
            msg += ": " + L.cd_last_cuda_error().decode()
        raise CholdiffError(f"libcholdiff status {rc}: {msg}")


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return CD_F64
    if t.dtype == torch.float32:
        return CD_F32
    raise TypeError(f"unsupported dtype {t.dtype} (float64 / float32 only)")


def colmajor(t: torch.Tensor) -> torch.Tensor:
    """Copy of a logical (..., N, N) tensor whose per-matrix memory is column-major."""
    return t.transpose(-1, -2).contiguous().transpose(-1, -2)


def is_colmajor(t: torch.Tensor) -> bool:
    n = t.shape[-1]
    if t.shape[-2] != n:
        return False
    if n <= 1:
        return True
    ok = t.stride(-2) == 1 and t.stride(-1) >= n
    if t.dim() == 3 and t.shape[0] > 1:
        ok = ok and t.stride(0) >= t.stride(-1) * n
    return ok


def _opts(nb, route, out):
    return _Opts(int(nb or 0), ROUTES[route], OUT_MODES[out], 0)


_ws_cache: dict = {}


def _workspace(nbytes: int, device: torch.device) -> torch.Tensor | None:
    if nbytes == 0:
        return None
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def workspace_size(op: str, dtype: torch.dtype, n: int, batch: int = 1, nb=None, route="auto", out="tril") -> int:
    o = _opts(nb, route, out)
    return int(lib().cd_workspace_size(CD_OP_REV if op == "rev" else CD_OP_FWD,
                                       CD_F64 if dtype == torch.float64 else CD_F32, n, batch, ctypes.byref(o)))


def _prep(L: torch.Tensor, A: torch.Tensor, inplace: bool):
    """Returns (L, A, dest): column-major operands, and the caller's tensor to copy the
    result back into when an in-place call had to work on a column-major copy (else None)."""
    if not (L.is_cuda and A.is_cuda):
        raise CholdiffError("chol_rev/chol_fwd take CUDA tensors (use chol_host for host buffers)")
    if L.dtype != A.dtype:
        raise TypeError("L and the sensitivity must have the same dtype")
    if L.shape != A.shape or L.dim() not in (2, 3) or L.shape[-1] != L.shape[-2]:
        raise ValueError(f"expected matching (N,N) or (B,N,N) tensors, got {tuple(L.shape)} / {tuple(A.shape)}")
    if not is_colmajor(L):
        L = colmajor(L)
    dest = None
    if not inplace:
        A = colmajor(A)
    elif not is_colmajor(A):
        dest, A = A, colmajor(A)
    return L, A, dest


def _finish(A: torch.Tensor, dest, info_t, info: bool, check: bool):
    if dest is not None:
        dest.copy_(A)  # in-place contract for non-column-major sensitivities
        A = dest
    if check and info_t is not None:
        host = info_t.cpu()  # synchronises the current stream
        if bool(host.any()):
            raise SingularFactorError(host.tolist())
    return (A, info_t) if info else A


def _run(op: int, L: torch.Tensor, A: torch.Tensor, nb, route, out, info: bool):
    """One C-ABI call; returns (A, info tensor or None)."""
    Lc = lib()
    n = A.shape[-1]
    batch = A.shape[0] if A.dim() == 3 else 1
    if n == 0 or batch == 0:  # no-op (the C ABI returns CD_SUCCESS as well)
        return A, (torch.zeros(batch, dtype=torch.int32, device=A.device) if info else None)
    o = _opts(nb, route, out)
    dt = _dt(A)
    dev = A.device
    with torch.cuda.device(dev):
        nbytes = int(Lc.cd_workspace_size(op, dt, n, batch, ctypes.byref(o)))
        ws = _workspace(nbytes, dev)
        info_t = torch.zeros(batch, dtype=torch.int32, device=dev) if info else None
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        ldl = max(1, L.stride(-1)) if n > 1 else max(1, n)
        lda = max(1, A.stride(-1)) if n > 1 else max(1, n)
        wsp = ctypes.c_void_p(ws.data_ptr()) if ws is not None else None
        ip = ctypes.c_void_p(info_t.data_ptr()) if info_t is not None else None
        single = {CD_OP_REV: Lc.cd_chol_rev, CD_OP_FWD: Lc.cd_chol_fwd, CD_OP_CHOL_FWD: Lc.cd_chol_fwd_fused}
        strided = {CD_OP_REV: Lc.cd_chol_rev_strided_batched, CD_OP_FWD: Lc.cd_chol_fwd_strided_batched,
                   CD_OP_CHOL_FWD: Lc.cd_chol_fwd_fused_strided_batched}
        if A.dim() == 2:
            f = single[op]
            rc = f(dt, n, L.data_ptr(), ldl, A.data_ptr(), lda, ctypes.byref(o), wsp, nbytes, ip, stream)
        else:
            f = strided[op]
            sL = L.stride(0) if batch > 1 else ldl * n
            sA = A.stride(0) if batch > 1 else lda * n
            rc = f(dt, n, L.data_ptr(), ldl, sL, A.data_ptr(), lda, sA, batch, ctypes.byref(o), wsp, nbytes, ip,
                   stream)
        _check(rc)
    return A, info_t


def chol_rev(L: torch.Tensor, Lbar: torch.Tensor, *, nb=None, route: str = "auto", out: str = "tril",
             inplace: bool = True, info: bool = False, check: bool = False):
    """Reverse mode (L, Lbar) -> Sigma_bar.  Returns the tensor holding tril(Sigma_bar)
    (Eq. 10 convention; ``out='sym'`` / ``'grad'`` also write the upper triangle, see
    include/choldiff.h).  With ``info=True`` also returns the per-matrix status tensor;
    ``check=True`` synchronises and raises SingularFactorError on a singular factor."""
    L, A, dest = _prep(L, Lbar, inplace)
    A, info_t = _run(CD_OP_REV, L, A, nb, route, out, info or check)
    return _finish(A, dest, info_t, info, check)


def chol_fwd(L: torch.Tensor, Sdot: torch.Tensor, *, nb=None, route: str = "auto", inplace: bool = True,
             info: bool = False, check: bool = False):
    """Forward mode (L, Sigma_dot) -> L_dot (lower triangle of the returned tensor).
    ``info`` / ``check`` as for chol_rev."""
    L, A, dest = _prep(L, Sdot, inplace)
    A, info_t = _run(CD_OP_FWD, L, A, nb, route, "tril", info or check)
    return _finish(A, dest, info_t, info, check)


def chol_rev_fwd(L: torch.Tensor, Lbar: torch.Tensor, Sdot: torch.Tensor, *, nb=None, inplace: bool = True):
    """Both sensitivities of one factor (configs[3]'s workload) in one library call
    (cd_chol_rev_fwd_strided_batched): Sigma_bar = chol_rev(L, Lbar) and L_dot = chol_fwd(L, Sdot),
    the two independent sweeps on two streams inside the library, ordered on the current stream.
    Returns (Sigma_bar, L_dot)."""
    Lc, A, dA = _prep(L, Lbar, inplace)
    _, F, dF = _prep(Lc, Sdot, inplace)
    if F.shape != A.shape or F.dtype != A.dtype:
        raise ValueError("Lbar and Sdot must match")
    Lk = lib()
    n = A.shape[-1]
    batch = A.shape[0] if A.dim() == 3 else 1
    if n == 0 or batch == 0:
        return A, F
    o = _opts(nb, "auto", "tril")
    dt = _dt(A)
    dev = A.device
    with torch.cuda.device(dev):
        nbytes = int(Lk.cd_workspace_size_rev_fwd(dt, n, batch, ctypes.byref(o)))
        ws = _workspace(nbytes, dev)
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        ld = lambda t: max(1, t.stride(-1)) if n > 1 else 1  # noqa: E731
        sb = lambda t: (t.stride(0) if batch > 1 else ld(t) * n) if t.dim() == 3 else ld(t) * n  # noqa: E731
        wsp = ctypes.c_void_p(ws.data_ptr()) if ws is not None else None
        rc = Lk.cd_chol_rev_fwd_strided_batched(dt, n, Lc.data_ptr(), ld(Lc), sb(Lc), A.data_ptr(), ld(A), sb(A),
                                                F.data_ptr(), ld(F), sb(F), batch, ctypes.byref(o), wsp, nbytes,
                                                None, stream)
        _check(rc)
    if dA is not None:
        dA.copy_(A)
        A = dA
    if dF is not None:
        dF.copy_(F)
        F = dF
    return A, F


def chol_fwd_fused(Sigma: torch.Tensor, Sdot: torch.Tensor, *, info: bool = False):
    """Fused factorisation + forward mode (cd_chol_fwd_fused, fp64): in place, tril(Sigma) ->
    L with Sigma = L L^T and tril(Sdot) -> L_dot, in one sweep.
    Both tensors must already be column-major CUDA tensors (they are overwritten).
    Returns (L, L_dot) [, info]."""
    if not (is_colmajor(Sigma) and is_colmajor(Sdot)):
        raise ValueError("chol_fwd_fused works in place: pass column-major tensors (see colmajor())")
    A, Ad = Sigma, Sdot
    if not (A.is_cuda and Ad.is_cuda) or A.shape != Ad.shape or A.dtype != Ad.dtype:
        raise ValueError("chol_fwd_fused takes two CUDA tensors of the same shape and dtype")
    Ad, info_t = _run(CD_OP_CHOL_FWD, A, Ad, None, "auto", "tril", info)
    return (A, Ad, info_t) if info else (A, Ad)


def chol_host(op: str, L_host: torch.Tensor, A_host: torch.Tensor, *, nb=None, device=None) -> torch.Tensor:
    """End-to-end path with HOST buffers (cd_chol_host): dense column-major host arrays
    (pinned for asynchronous copies) are copied to the device, processed and copied
    back into ``A_host`` in place.  Synchronizes the current stream before returning."""
    Lc = lib()
    dev = torch.device(device or "cuda")
    n = A_host.shape[-1]
    dt = _dt(A_host)
    o = _opts(nb, "auto", "tril")
    opc = CD_OP_REV if op == "rev" else CD_OP_FWD
    if not (L_host.stride(-2) == 1 and L_host.stride(-1) == n and A_host.stride(-2) == 1 and A_host.stride(-1) == n):
        raise ValueError("chol_host expects dense column-major (ld = N) host tensors")
    with torch.cuda.device(dev):
        nbytes = int(Lc.cd_workspace_size_host(opc, dt, n, ctypes.byref(o)))
        ws = _workspace(nbytes, dev)
        stream = torch.cuda.current_stream(dev)
        rc = Lc.cd_chol_host(opc, dt, n, L_host.data_ptr(), A_host.data_ptr(), ctypes.byref(o),
                             ctypes.c_void_p(ws.data_ptr()), nbytes, ctypes.c_void_p(stream.cuda_stream))
        _check(rc)
        stream.synchronize()
    return A_host


def host_bytes():
    """(h2d, d2h) bytes moved by the last chol_host call on this thread (cd_host_bytes)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    lib().cd_host_bytes(ctypes.byref(a), ctypes.byref(b))
    return int(a.value), int(b.value)
