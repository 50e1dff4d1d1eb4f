"""CPU oracle for differentiating the Cholesky decomposition (arXiv 1602.07527).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1602_07527_b200``) never imports it and
shares no code with it; the two meet only through the seeded generator in
``synthetic/`` (which holds none of the method's arithmetic).

Contents (each pinned by ``tests/test_oracle.py``; nothing here is "parity
unpinned"):

* ``oracle.c`` (built to ``liboracle.so``, plain C, fp64, ``-O2
  -ffp-contract=off``): the scalar-loop algorithms ``chol_unblocked``
  (PAPER.md:437-445), ``chol_unblocked_fwd``,
  ``chol_unblocked_rev``, a complex-valued
  ``chol_unblocked`` for complex-step differentiation, and the symbolic results
  Eq. 8 / Eq. 9 / Eq. 10 by plain substitution.
* ``jacobian.py``: Eq. 11 element-wise partials and
  derivative-definition checks (finite differences / complex step).
* ``blocked.py``: the paper's blocked algorithms in numpy,
  used only to pin the readings of those algorithms.

All array arguments here are *logical* numpy arrays ``M[i, j]``; the wrappers
lay them out column-major for the C code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile ``oracle.c`` -> ``liboracle.so`` (gcc).  Returns the library path."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            i64, pd, pi = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
            for name, args in {
                "or_chol_unblocked": [i64, pd, i64],
                "or_chol_unblocked_cols": [i64, pd, i64],
                "or_chol_fwd_cols": [i64, pd, i64, pd, i64],
                "or_chol_unblocked_complex": [i64, ctypes.c_void_p, i64],
                "or_chol_fwd": [i64, pd, i64, pd, i64],
                "or_chol_rev": [i64, pd, i64, pd, i64],
                "or_chol_rev_partial": [i64, pd, i64, pd, i64, i64],
                "or_chol_fwd_symbolic": [i64, pd, i64, pd, i64, pd, i64],
                "or_chol_rev_symbolic": [i64, pd, i64, pd, i64, pd, i64],
                "or_chol_rev_symbolic_sym": [i64, pd, i64, pd, i64, pd, i64],
            }.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = ctypes.c_int
            L.or_set_threads.argtypes = [ctypes.c_int]
            L.or_set_threads.restype = None
            for name in ("or_chol_rev_batched", "or_chol_fwd_batched", "or_chol_fwd_cols_batched"):
                f = getattr(L, name)
                f.argtypes = [i64, i64, pd, i64, i64, pd, i64, i64, pi]
                f.restype = None
            _lib = L
    return _lib


def _cm(m, dtype=np.float64):
    """Column-major (Fortran-order) float64 copy of a logical matrix."""
    return np.array(m, dtype=dtype, order="F", copy=True)


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class SingularFactor(ValueError):
    """A diagonal entry of L is zero or non-finite (1-based index in ``.j``)."""

    def __init__(self, j):
        super().__init__(f"L[{j},{j}] (1-based) is zero or non-finite")
        self.j = j


class NotPositiveDefinite(ValueError):
    def __init__(self, j):
        super().__init__(f"matrix not positive definite at column {j} (1-based)")
        self.j = j


def chol(sigma):
    """chol_unblocked of tril(sigma); returns L (logical, upper = 0)."""
    a = _cm(sigma)
    n = a.shape[0]
    info = lib().or_chol_unblocked(n, _p(a), max(1, n))
    if info:
        raise NotPositiveDefinite(info)
    return np.tril(a)


def chol_complex(sigma):
    """chol_unblocked over complex numbers (complex-step pin)."""
    a = np.array(sigma, dtype=np.complex128, order="F", copy=True)
    n = a.shape[0]
    info = lib().or_chol_unblocked_complex(n, a.ctypes.data_as(ctypes.c_void_p), max(1, n))
    if info:
        raise NotPositiveDefinite(info)
    return np.tril(a)


def chol_fwd(L, sigma_dot):
    """chol_unblocked_fwd: returns Ldot (lower; upper copied from input)."""
    l, a = _cm(L), _cm(sigma_dot)
    n = l.shape[0]
    info = lib().or_chol_fwd(n, _p(l), max(1, n), _p(a), max(1, n))
    if info:
        raise SingularFactor(info)
    return np.array(a)


def chol_rev(L, L_bar):
    """chol_unblocked_rev: returns the in-place result array;
    its lower triangle is tril(Sigma_bar) (Eq. 10 convention), upper untouched."""
    l, a = _cm(L), _cm(L_bar)
    n = l.shape[0]
    info = lib().or_chol_rev(n, _p(l), max(1, n), _p(a), max(1, n))
    if info:
        raise SingularFactor(info)
    return np.array(a)


def chol_rev_colmajor_inplace(n, L_cm, Ab_cm, j_lo=0):
    """Raw in-place reverse sweep on column-major buffers (C-contiguous arrays whose
    bytes are column-major, e.g. ``synthetic.to_colmajor``).  Columns j_lo..n-1 only
    when ``j_lo > 0`` (bench sample).  Returns the info code."""
    return lib().or_chol_rev_partial(n, _p(L_cm), max(1, n), _p(Ab_cm), max(1, n), int(j_lo))


def chol_rev_batched_colmajor(n, batch, L_cm, Ab_cm):
    """OpenMP batched reverse sweep over contiguous column-major matrices (ld=n, stride=n*n)."""
    info = np.zeros(batch, dtype=np.int32)
    lib().or_chol_rev_batched(n, batch, _p(L_cm), max(1, n), n * n, _p(Ab_cm), max(1, n), n * n,
                              info.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return info


def chol_fwd_batched_colmajor(n, batch, L_cm, Ad_cm):
    info = np.zeros(batch, dtype=np.int32)
    lib().or_chol_fwd_batched(n, batch, _p(L_cm), max(1, n), n * n, _p(Ad_cm), max(1, n), n * n,
                              info.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return info


def chol_fwd_cols_batched_colmajor(n, batch, L_cm, Ad_cm):
    """As chol_fwd_batched_colmajor, column-ordered evaluation (bit-identical, faster at large n)."""
    info = np.zeros(batch, dtype=np.int32)
    lib().or_chol_fwd_cols_batched(n, batch, _p(L_cm), max(1, n), n * n, _p(Ad_cm), max(1, n), n * n,
                                   info.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return info


def chol_fwd_colmajor_inplace(n, L_cm, Ad_cm):
    """In-place forward sweep on column-major buffers (C-contiguous arrays
    whose bytes are column-major), column-ordered evaluation, OpenMP over rows: bit-identical
    to chol_fwd (tests/test_oracle.py), for the full-size parity tests.  Returns the info code."""
    return lib().or_chol_fwd_cols(n, _p(L_cm), max(1, n), _p(Ad_cm), max(1, n))


def chol_fwd_serial_colmajor_inplace(n, L_cm, Ad_cm):
    """The plain row-wise forward sweep (or_chol_fwd, no OpenMP) on column-major buffers."""
    return lib().or_chol_fwd(n, _p(L_cm), max(1, n), _p(Ad_cm), max(1, n))


def set_threads(t: int) -> None:
    """OpenMP threads of the oracle's parallel loops (0 = all cores).  Scheduling only."""
    lib().or_set_threads(int(t))


def chol_colmajor_inplace(n, A_cm):
    """In-place chol_unblocked on a column-major buffer, column-ordered
    evaluation (bit-identical to chol); returns the info code (0, or the failing 1-based column)."""
    return lib().or_chol_unblocked_cols(n, _p(A_cm), max(1, n))


def chol_fwd_symbolic(L, sigma_dot):
    """Eq. 8 by substitution; reads tril(sigma_dot). Returns Ldot (upper 0)."""
    l, s = _cm(L), _cm(sigma_dot)
    n = l.shape[0]
    out = np.zeros((n, n), order="F")
    info = lib().or_chol_fwd_symbolic(n, _p(l), max(1, n), _p(s), max(1, n), _p(out), max(1, n))
    if info:
        raise SingularFactor(info)
    return np.array(out)


def chol_rev_symbolic(L, L_bar):
    """Eq. 10: tril(Sigma_bar) (upper 0)."""
    l, b = _cm(L), _cm(L_bar)
    n = l.shape[0]
    out = np.zeros((n, n), order="F")
    info = lib().or_chol_rev_symbolic(n, _p(l), max(1, n), _p(b), max(1, n), _p(out), max(1, n))
    if info:
        raise SingularFactor(info)
    return np.array(out)


def chol_rev_symbolic_sym(L, L_bar):
    """Eq. 9: full symmetric Sigma_bar = S + S^T - diag(S)."""
    l, b = _cm(L), _cm(L_bar)
    n = l.shape[0]
    out = np.zeros((n, n), order="F")
    info = lib().or_chol_rev_symbolic_sym(n, _p(l), max(1, n), _p(b), max(1, n), _p(out), max(1, n))
    if info:
        raise SingularFactor(info)
    return np.array(out)


# ---- flop counts (SURVEY.md §8 notation; used by bench.py for GFLOP/s) ----

def rev_flops(n: int) -> int:
    """Exact +,-,*,/ count of chol_unblocked_rev: 2n^3/3 + n^2/2 + 11n/6."""
    return (4 * n ** 3 + 3 * n ** 2 + 11 * n) // 6


def fwd_flops(n: int) -> int:
    """Exact +,-,*,/ count of chol_unblocked_fwd: 2n^3/3 + n^2/2 + 5n/6."""
    return (4 * n ** 3 + 3 * n ** 2 + 5 * n) // 6


def rev_column_flops(n: int, j: int) -> int:
    """Flops of column j (0-based) of the reverse sweep, statement by statement:
    dbar update 2a+1, scaling a+1, rbar 2b(a+1), Bbar 2ab, halving 1 (a = n-1-j, b = j)."""
    a, b = n - 1 - j, j
    return (2 * a + 1) + (a + 1) + 2 * b * (a + 1) + 2 * a * b + 1
