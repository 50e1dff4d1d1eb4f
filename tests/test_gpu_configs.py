"""GPU parity at BASELINE.json's full configurations, in the launch configuration
bench.py times (same entry points, same nb).  Where the oracle cannot finish the
whole output in seconds, it computes a sample exactly (the trailing columns of the
reverse sweep: columns j >= j_lo are final after the sweep reaches j_lo,
tests/test_oracle.py::test_partial_sweep_is_prefix_of_full) and the full output is
checked through properties that hold at any size (Eq. 9 / Eq. 10 identity, adjoint
identity, exact power-of-two scaling)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1602_07527_b200 as cd
import synthetic
from gpu_helpers import fp32_round, nerr, to_dev, to_host

pytestmark = pytest.mark.gpu


def eq10_identity_residual(Ld: torch.Tensor, Lbd: torch.Tensor, T: torch.Tensor) -> float:
    """Eq. 9/10: with T = tril(Sigma_bar) and S = L^{-T} P L^{-1},
    P = Phi(L^T tril(Lbar)):  T + T^T (diagonal doubled) = S + S^T, hence
    L^T (T + T^T) L = P + P^T.  Returns max|residual| / max|P + P^T| (fp64 cuBLAS)."""
    L = torch.tril(Ld)
    T = torch.tril(T)
    X = L.T @ torch.tril(Lbd)
    P = torch.tril(X, -1) + torch.diag(torch.diagonal(X) * 0.5)
    rhs = P + P.T
    lhs = L.T @ (T + T.T) @ L
    return float((lhs - rhs).abs().max() / rhs.abs().max())


def test_config1_rev_n64():
    L, Lb, _ = synthetic.draw(64, 0)
    out = cd.chol_rev(to_dev(L), to_dev(Lb))
    assert nerr(to_host(out), oracle.chol_rev(L, Lb)) < 1e-10


def test_config2_n1024_rev_fwd_adjoint():
    n = 1024
    L, Lb, Sd = synthetic.draw(n, 0, sdot=True)
    Sb = to_host(cd.chol_rev(to_dev(L), to_dev(Lb)))
    Ld = to_host(cd.chol_fwd(to_dev(L), to_dev(np.tril(Sd))))
    assert nerr(Sb, oracle.chol_rev(L, Lb)) < 1e-10
    assert nerr(Ld, oracle.chol_fwd(L, np.tril(Sd))) < 1e-10
    lhs = np.sum(np.tril(Lb) * np.tril(Ld))
    rhs = np.sum(np.tril(Sb) * np.tril(Sd))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(np.tril(Lb)) * np.linalg.norm(np.tril(Ld))


def test_config3_batched_65536_n32_all_matrices():
    n, B = 32, 65536
    L, Lb, _ = synthetic.draw_batch(n, B, seed=0)
    out = to_host(cd.chol_rev(to_dev(L), to_dev(Lb)))
    Lc, Ac = synthetic.to_colmajor(L), synthetic.to_colmajor(Lb)
    assert not oracle.chol_rev_batched_colmajor(n, B, Lc, Ac).any()
    ref = synthetic.from_colmajor(Ac)
    assert nerr(out, ref) < 1e-10
    # upper triangles untouched (TRIL mode): equal to the input's
    iu = np.triu_indices(n, 1)
    assert np.array_equal(out[:, iu[0], iu[1]], Lb[:, iu[0], iu[1]])


def test_config4_batched_f32_1024_n512_rev_fwd():
    n, B = 512, 1024
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=0, sdot=True)
    L, Lb, Sd = fp32_round(L, Lb, Sd)
    Lt = to_dev(L, torch.float32)
    # the bench's call: both sweeps of the same factors on two streams
    Sb, Ldot = cd.chol_rev_fwd(Lt, to_dev(Lb, torch.float32), to_dev(np.tril(Sd), torch.float32))
    Sb, Ldot = to_host(Sb), to_host(Ldot)
    assert np.all(np.isfinite(np.tril(Sb))) and np.all(np.isfinite(np.tril(Ldot)))
    for b in (0, 1, 511, 1023):  # oracle sample (fp64 on the fp32-rounded inputs)
        assert nerr(Sb[b], oracle.chol_rev(L[b], Lb[b])) < 1e-4
        assert nerr(Ldot[b], oracle.chol_fwd(L[b], np.tril(Sd[b]))) < 1e-4
    # adjoint identity on every matrix (fp64 accumulation of the fp32 outputs)
    lhs = np.einsum("bij,bij->b", np.tril(Lb), np.tril(Ldot))
    rhs = np.einsum("bij,bij->b", np.tril(Sb), np.tril(Sd))
    scale = np.linalg.norm(np.tril(Lb), axis=(1, 2)) * np.linalg.norm(np.tril(Ldot), axis=(1, 2))
    assert np.max(np.abs(lhs - rhs) / scale) < 1e-4


@pytest.mark.parametrize("n,nb", [(3000, 128), (16384, 128)])
def test_config5_large_rev(n, nb):
    L, Lb, _ = synthetic.draw(n, 0)
    Lc, Ac = synthetic.to_colmajor(L), synthetic.to_colmajor(Lb)
    del L
    Ld = torch.from_numpy(Lc).cuda().transpose(0, 1)
    Lbd = torch.from_numpy(Ac).cuda().transpose(0, 1)
    out = cd.chol_rev(Ld, Lbd.clone(), nb=nb)
    # (i) exact sample: trailing columns by the oracle's partial sweep
    a = 384
    oracle.chol_rev_colmajor_inplace(n, Lc, Ac, j_lo=n - a)
    ref_cols = np.tril(Ac[n - a:].T, -(n - a))            # logical rows x last a columns
    got_cols = np.tril(out[:, n - a:].cpu().numpy(), -(n - a))
    den = np.linalg.norm(ref_cols)
    assert np.abs(got_cols - ref_cols).max() / den < 1e-10
    # (ii) the whole output through Eq. 10's identity
    assert eq10_identity_residual(Ld, Lbd, out) < 1e-9
    # (iii) exact power-of-two scaling (deterministic kernels)
    out2 = cd.chol_rev(Ld * 2.0, Lbd.clone(), nb=nb)
    assert torch.equal(torch.tril(out2) * 2.0, torch.tril(out))
