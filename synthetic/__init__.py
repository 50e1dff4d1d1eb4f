"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws random numbers
in a fixed order and lays them out in memory.  Both `oracle/` and the product
path consume its output; neither is imported here.

Recipe (BASELINE.json configs; SURVEY.md §8(d) "Synthetic inputs"):
  * RNG: numpy PCG64, ``np.random.default_rng(seed)``; matrix ``b`` of a batch
    uses ``seed + b`` ("seed+index", BASELINE.json configs[2]).
  * Draw order per matrix (fixed, so that skipping a later draw never changes an
    earlier one):
      1. ``standard_normal((N, N))`` -> strictly-lower part / sqrt(N) -> off-diagonal of L
      2. ``uniform(1, 2, N)``         -> diag(L)
      3. ``standard_normal((N, N))`` -> lower triangle (incl. diagonal) -> Lbar
      4. ``standard_normal((N, N))`` -> lower triangle (incl. diagonal), mirrored -> Sigma_dot
  * Arrays are returned in *logical* orientation ``M[i, j]`` (row i, column j).
    ``to_colmajor`` produces the column-major byte layout the C-ABI consumes
    (element (i, j) of matrix b at offset ``b*stride + j*ld + i``).
"""
from __future__ import annotations

import numpy as np

GENERATOR_VERSION = "pcg64-v1 (L: N(0,1)/sqrt(N) strict-lower, U[1,2] diag; Lbar: tril N(0,1); Sdot: tril N(0,1) mirrored)"


def draw(n: int, seed: int, lbar: bool = True, sdot: bool = False):
    """Return (L, Lbar or None, Sdot or None) for one matrix, logical orientation, float64.

    The upper triangles of L and Lbar are zero; Sdot is full symmetric.
    """
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n)) if n > 0 else np.zeros((0, 0))
    L = np.tril(g, -1) / np.sqrt(n) if n > 0 else g
    L[np.diag_indices(n)] = rng.uniform(1.0, 2.0, n)
    del g
    Lb = Sd = None
    if lbar or sdot:
        Lb = np.tril(rng.standard_normal((n, n)))
    if sdot:
        t = np.tril(rng.standard_normal((n, n)))
        Sd = t + np.tril(t, -1).T
    return L, (Lb if lbar else None), Sd


def draw_batch(n: int, batch: int, seed: int = 0, lbar: bool = True, sdot: bool = False,
               start: int = 0):
    """Batch of matrices ``start .. start+batch-1`` (matrix b uses seed ``seed + b``).

    Returns logical-orientation arrays of shape (batch, n, n) (or None).
    """
    L = np.empty((batch, n, n))
    Lb = np.empty((batch, n, n)) if lbar else None
    Sd = np.empty((batch, n, n)) if sdot else None
    for i in range(batch):
        l, lb, sd = draw(n, seed + start + i, lbar=lbar, sdot=sdot)
        L[i] = l
        if lbar:
            Lb[i] = lb
        if sdot:
            Sd[i] = sd
    return L, Lb, Sd


def to_colmajor(m: np.ndarray, dtype=np.float64) -> np.ndarray:
    """Column-major memory image of a logical (n, n) or (batch, n, n) array.

    The returned C-contiguous array ``c`` satisfies ``c[..., j, i] == m[..., i, j]``,
    i.e. its bytes are the LAPACK column-major layout with ``ld = n``,
    ``stride = n*n``.
    """
    return np.ascontiguousarray(np.swapaxes(m, -1, -2), dtype=dtype)


def from_colmajor(c: np.ndarray) -> np.ndarray:
    """Inverse of :func:`to_colmajor` (returns a logical-orientation view copy)."""
    return np.ascontiguousarray(np.swapaxes(c, -1, -2))


def poison_upper(m: np.ndarray, value=np.nan) -> np.ndarray:
    """Copy of logical array ``m`` with its strict upper triangle set to ``value``
    (used to test that the upper triangle is never read: PAPER.md:448-451)."""
    out = np.array(m, dtype=np.float64, copy=True)
    n = out.shape[-1]
    iu = np.triu_indices(n, 1)
    out[..., iu[0], iu[1]] = value
    return out
