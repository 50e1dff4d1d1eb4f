"""Gaussian-process log-likelihood gradient through the Cholesky derivative (
the paper's motivating use).

    theta = (log ell, log sf, log sn)      K(theta) = sf^2 exp(-|xi - xj|^2 / (2 ell^2)) + sn^2 I
    f(theta) = -1/2 y^T K^{-1} y - 1/2 log|K| - n/2 log(2 pi)

Path: Sigma = K -> (cd.chol_fwd_fused) L -> alpha = L^{-1} y, beta = L^{-T} alpha ->
L_bar = df/dL = tril(beta alpha^T) - diag(1 / L_ii) -> (cd.chol_rev) tril(Sigma_bar) (Eq. 10
convention: Sigma_bar_ij for i > j covers both K_ij and K_ji) -> df/dtheta_k = sum_{i >= j}
Sigma_bar_ij dK_ij/dtheta_k.  The factorisation and the reverse sweep run in libcholdiff; the
two triangular solves with a single right-hand side are torch calls.  The forward sensitivity
L_dot that chol_fwd_fused computes alongside (direction Sigma_dot = dK/dtheta_0) gives a second,
forward-mode value of df/dtheta_0 as a cross-check:
    df = -alpha^T dalpha - sum_i dL_ii / L_ii,   dalpha = -L^{-1} L_dot alpha.

Run:  python examples/gp_loglik_grad.py  (needs a GPU).
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_07527_b200 as cd  # noqa: E402


def kernel_and_derivs(x: torch.Tensor, theta: torch.Tensor):
    """K(theta) and dK/dtheta_k (k = 0, 1, 2), all (n, n), for the squared-exponential kernel."""
    ell, sf, sn = torch.exp(theta)
    d2 = torch.cdist(x, x).pow(2)
    E = torch.exp(-0.5 * d2 / ell**2)
    K = sf**2 * E + sn**2 * torch.eye(x.shape[0], dtype=x.dtype, device=x.device)
    dK = [sf**2 * E * d2 / ell**2, 2.0 * sf**2 * E, 2.0 * sn**2 * torch.eye(x.shape[0], dtype=x.dtype, device=x.device)]
    return K, dK


def loglik_and_grad(x: torch.Tensor, y: torch.Tensor, theta: torch.Tensor):
    """f(theta) and df/dtheta through libcholdiff (fp64, CUDA tensors)."""
    n = x.shape[0]
    K, dK = kernel_and_derivs(x, theta)
    A = cd.colmajor(K)                              # Sigma -> L in place
    Ad = cd.colmajor(torch.tril(dK[0]))             # Sigma_dot = dK/dtheta_0 -> L_dot
    L, Ldot = cd.chol_fwd_fused(A, Ad)
    L = torch.tril(L)
    alpha = torch.linalg.solve_triangular(L, y[:, None], upper=False)
    beta = torch.linalg.solve_triangular(L.T, alpha, upper=True)
    f = -0.5 * float(alpha.square().sum()) - float(torch.log(torch.diagonal(L)).sum()) - 0.5 * n * math.log(2 * math.pi)
    Lbar = torch.tril(beta @ alpha.T) - torch.diag(1.0 / torch.diagonal(L))
    Sbar = torch.tril(cd.chol_rev(cd.colmajor(L), cd.colmajor(Lbar)))
    grad = torch.stack([(Sbar * torch.tril(dk)).sum() for dk in dK])
    # forward mode along theta_0: df = -alpha^T dalpha - sum dL_ii / L_ii, dalpha = -L^{-1} L_dot alpha
    Ldot = torch.tril(Ldot)
    dalpha = -torch.linalg.solve_triangular(L, Ldot @ alpha, upper=False)
    fwd0 = -float((alpha * dalpha).sum()) - float((torch.diagonal(Ldot) / torch.diagonal(L)).sum())
    return f, grad, fwd0


def reference_grad(x: np.ndarray, y: np.ndarray, theta: np.ndarray):
    """Textbook closed form (Rasmussen & Williams 2006, eq. 5.9): df/dtheta_k =
    1/2 tr((beta beta^T - K^{-1}) dK/dtheta_k), beta = K^{-1} y, in numpy fp64."""
    xt = torch.from_numpy(x)
    K, dK = kernel_and_derivs(xt, torch.from_numpy(theta))
    K = K.numpy()
    Ki = np.linalg.inv(K)
    beta = Ki @ y
    W = np.outer(beta, beta) - Ki
    return np.array([0.5 * np.sum(W * dk.numpy()) for dk in dK])


def main():
    rng = np.random.default_rng(0)
    n, d = 1500, 3
    x = rng.uniform(-2, 2, (n, d))
    y = np.sin(x).sum(1) + 0.1 * rng.standard_normal(n)
    theta = np.log(np.array([0.8, 1.2, 0.3]))
    dev = torch.device("cuda")
    f, g, fwd0 = loglik_and_grad(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev), torch.from_numpy(theta).to(dev))
    ref = reference_grad(x, y, theta)
    print(f"f = {f:.6f}\ngrad (libcholdiff)  = {g.cpu().numpy()}\ngrad (closed form)  = {ref}\n"
          f"forward df/dtheta_0 = {fwd0:.10f}")


if __name__ == "__main__":
    main()
