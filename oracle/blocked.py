"""The paper's blocked derivative algorithms in numpy (TEST INFRASTRUCTURE ONLY).

Transcribes ``chol_blocked_fwd`` and ``chol_blocked_rev``
 statement by statement, with numpy matmul / triangular solve
as the library primitives and the diagonal-block routines taken from the C
oracle.  Used by tests/test_oracle.py to pin the readings listed in DESIGN.md §2
(block placement when nb does not divide N, the ``Dbar + Dbar^T`` term, tril
masking) before any kernel relies on them.  Indices below are 0-based:
block [j, k) (the paper's 1-based j..k).
"""
from __future__ import annotations

import numpy as np

from . import chol_fwd, chol_rev


def _solve_right_lower(X, D):
    """X D^{-1} for lower-triangular D (library solve)."""
    return np.linalg.solve(D.T, X.T).T


def chol_blocked_rev(L, Lbar, nb):
    L = np.array(L, dtype=np.float64)
    A = np.array(Lbar, dtype=np.float64)
    n = L.shape[0]
    k = n
    while k > 0:                                   # for k = N to >= 1 in steps of -Nb
        j = max(0, k - nb)                         # j <- max(1, k - Nb + 1)
        R, D, B, C = L[j:k, :j], np.tril(L[j:k, j:k]), L[k:, :j], L[k:, j:k]
        Cb = _solve_right_lower(A[k:, j:k], D)     # Cbar <- Cbar D^{-1}
        A[k:, j:k] = Cb
        A[k:, :j] -= Cb @ R                        # Bbar <- Bbar - Cbar R
        A[j:k, j:k] -= np.tril(Cb.T @ C)           # Dbar <- Dbar - tril(Cbar^T C)
        A[j:k, j:k] = chol_rev(D, A[j:k, j:k])     # Dbar <- chol_unblocked_rev(D, Dbar)
        Db = np.tril(A[j:k, j:k])
        A[j:k, :j] -= Cb.T @ B + (Db + Db.T) @ R   # Rbar <- Rbar - Cbar^T B - (Dbar + Dbar^T) R
        k = j
    return A


def chol_blocked_fwd(L, Sdot, nb):
    L = np.array(L, dtype=np.float64)
    A = np.array(Sdot, dtype=np.float64)
    n = L.shape[0]
    for j in range(0, n, nb):                      # for j = 1 to <= N in steps of Nb
        k = min(n, j + nb)                         # k <- min(N, j + Nb - 1)
        R, D, B, C = L[j:k, :j], np.tril(L[j:k, j:k]), L[k:, :j], L[k:, j:k]
        Rd, Bd = A[j:k, :j], A[k:, :j]
        A[j:k, j:k] -= np.tril(Rd @ R.T + R @ Rd.T)            # Ddot -= tril(Rdot R^T + R Rdot^T)
        A[j:k, j:k] = chol_fwd(D, A[j:k, j:k])                # Ddot <- chol_unblocked_fwd(D, Ddot)
        Dd = np.tril(A[j:k, j:k])
        A[k:, j:k] -= Bd @ R.T + B @ Rd.T                      # Cdot -= Bdot R^T + B Rdot^T
        A[k:, j:k] = _solve_right_lower(A[k:, j:k] - C @ Dd.T, D.T)  # Cdot <- (Cdot - C Ddot^T) D^{-T}
    return A
