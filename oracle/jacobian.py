"""Derivative-definition checks and Eq. 11 (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

* ``jacobian_eq11(L)``: every partial dL_ij/dSigma_kl from Eq. 11,
  as plain loops over (i, j, k, l) - Theta(N^4), small N only.  Row index vech(L)
  position of (i, j); column index vech(Sigma) position of (k, l), with Sigma_kl =
  Sigma_lk treated as ONE variable.
* ``jacobian_complex_step(L)``: the same matrix by complex-step differentiation of
  ``chol_unblocked`` (an independent route: no formula of the paper is used).
* ``fd_rev(L, Lbar)``: central finite differences of f(Sigma) = <Lbar, chol(Sigma)>
  (the north-star pin), returning tril(Sigma_bar) in the paper's convention.
"""
from __future__ import annotations

import numpy as np

from . import chol, chol_complex


def vech_index(n):
    """List of (i, j), i >= j, in vech (column-stacked lower triangle) order."""
    return [(i, j) for j in range(n) for i in range(j, n)]


def jacobian_eq11(L):
    L = np.tril(np.asarray(L, dtype=np.float64))
    n = L.shape[0]
    Li = np.linalg.solve(L, np.eye(n))  # L^{-1}; library primitive (small n)
    idx = vech_index(n)
    J = np.zeros((len(idx), len(idx)))
    for r, (i, j) in enumerate(idx):
        for c, (k, l) in enumerate(idx):
            # (sum_{m>j} L_im Linv_mk + 1/2 L_ij Linv_jk) Linv_jl
            t1 = sum(L[i, m] * Li[m, k] for m in range(j + 1, n)) + 0.5 * L[i, j] * Li[j, k]
            v = t1 * Li[j, l]
            if k != l:  # (1 - delta_kl)(sum_{m>j} L_im Linv_ml + 1/2 L_ij Linv_jl) Linv_jk
                t2 = sum(L[i, m] * Li[m, l] for m in range(j + 1, n)) + 0.5 * L[i, j] * Li[j, l]
                v += t2 * Li[j, k]
            J[r, c] = v
    return J


def _unit_sym(n, k, l):
    V = np.zeros((n, n))
    V[k, l] = 1.0
    V[l, k] = 1.0
    return V


def jacobian_complex_step(L, h=1e-30):
    L = np.tril(np.asarray(L, dtype=np.float64))
    n = L.shape[0]
    sigma = L @ L.T
    idx = vech_index(n)
    J = np.zeros((len(idx), len(idx)))
    for c, (k, l) in enumerate(idx):
        Lc = chol_complex(sigma + 1j * h * _unit_sym(n, k, l))
        d = Lc.imag / h
        J[:, c] = [d[i, j] for (i, j) in idx]
    return J


def ldot_complex_step(L, sigma_dot, h=1e-30):
    """Forward derivative d/dt chol(Sigma + t Sdot) at t=0 by complex step."""
    L = np.tril(np.asarray(L, dtype=np.float64))
    sigma = L @ L.T
    return (chol_complex(sigma + 1j * h * np.asarray(sigma_dot)).imag / h)


def fd_rev(L, Lbar, rel_h=1e-6):
    """Central finite differences of f = <tril(Lbar), chol(Sigma)> w.r.t. each vech(Sigma)
    variable (symmetric perturbation E_kl + E_lk), h = rel_h * max|Sigma|."""
    L = np.tril(np.asarray(L, dtype=np.float64))
    Lb = np.tril(np.asarray(Lbar, dtype=np.float64))
    n = L.shape[0]
    sigma = L @ L.T
    h = rel_h * np.abs(sigma).max()
    out = np.zeros((n, n))
    for (k, l) in vech_index(n):
        V = _unit_sym(n, k, l)
        fp = np.sum(Lb * chol(sigma + h * V))
        fm = np.sum(Lb * chol(sigma - h * V))
        out[k, l] = (fp - fm) / (2 * h)
    return out
