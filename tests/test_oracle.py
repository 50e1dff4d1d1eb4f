"""Pins for the CPU oracle (tests -m "not gpu").

The oracle (oracle/) is checked against things OTHER than itself: worked examples
(tests/golden/, each with its citation), closed forms derived from the paper's
equations, the derivative definition (complex step, central finite differences),
Eq. 11's element-wise Jacobian, a second independent route (the symbolic Eqs.
8-10), the adjoint identity, exact power-of-two scaling, linearity, and
upper-triangle poisoning.  A dropped term, wrong sign/index or transposed operand
anywhere in oracle.c fails at least one of these.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synthetic
from oracle import blocked, jacobian

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def nerr(out, ref):
    """max |out - ref| over the lower triangle / ||tril(ref)||_F."""
    out, ref = np.tril(out), np.tril(ref)
    den = np.linalg.norm(ref)
    return np.abs(out - ref).max() / (den if den > 0 else 1.0)


# ---------------------------------------------------------------- worked examples

def test_golden_fwd_2x2_bit_exact():
    g = gold("fwd_2x2_spec.json")
    L, Sd = np.array(g["L"]), np.array(g["Sigma_dot"])
    ref = np.array(g["Ldot_lower"])
    assert np.array_equal(np.tril(oracle.chol_fwd(L, Sd)), ref)
    assert np.array_equal(oracle.chol_fwd_symbolic(L, Sd), ref)


def test_golden_rev_2x2_bit_exact():
    g = gold("rev_2x2_eq10.json")
    L, Lb = np.array(g["L"]), np.array(g["Lbar"])
    assert np.array_equal(np.tril(oracle.chol_rev(L, Lb)), np.array(g["Sigma_bar_tril"]))
    assert np.array_equal(oracle.chol_rev_symbolic(L, Lb), np.array(g["Sigma_bar_tril"]))
    assert np.array_equal(oracle.chol_rev_symbolic_sym(L, Lb), np.array(g["Sigma_bar_sym"]))


def test_golden_scalar():
    g = gold("scalar_n1.json")
    L = np.array(g["L"])
    assert oracle.chol_rev(L, np.array(g["Lbar"]))[0, 0] == g["Sigma_bar"][0][0]
    assert oracle.chol_fwd(L, np.array(g["Sigma_dot"]))[0, 0] == g["Ldot"][0][0]
    assert oracle.chol_rev_symbolic(L, np.array(g["Lbar"]))[0, 0] == g["Sigma_bar"][0][0]
    assert oracle.chol_fwd_symbolic(L, np.array(g["Sigma_dot"]))[0, 0] == g["Ldot"][0][0]


def test_chol_unblocked_worked_example():
    # Sigma = [[4,.],[2,5]] -> L = [[2,0],[1,2]]; and PD failure at column 2.
    assert np.array_equal(oracle.chol(np.array([[4.0, 0.0], [2.0, 5.0]])), np.array([[2.0, 0.0], [1.0, 2.0]]))
    with pytest.raises(oracle.NotPositiveDefinite) as e:
        oracle.chol(np.array([[1.0, 0.0], [2.0, 1.0]]))
    assert e.value.j == 2


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("n", [1, 3, 8, 17])
def test_rev_identity_factor_is_phi(n):
    # Eq. 10 with L = I: tril(Sbar) = Phi(Phi(Lbar) + Phi(Lbar)^T) = Phi(Lbar) exactly.
    Lb = np.tril(np.random.default_rng(n).standard_normal((n, n)))
    phi = np.tril(Lb, -1) + np.diag(np.diag(Lb) / 2)
    assert np.array_equal(np.tril(oracle.chol_rev(np.eye(n), Lb)), phi)


@pytest.mark.parametrize("n", [2, 5, 9])
def test_rev_diagonal_factor(n):
    # L = diag(d): Sbar_ij = Lbar_ij / d_j (i > j), Sbar_ii = Lbar_ii / (2 d_i)   (Eq. 10)
    rng = np.random.default_rng(100 + n)
    d = rng.uniform(1, 2, n)
    Lb = np.tril(rng.standard_normal((n, n)))
    ref = np.tril(Lb / d[None, :], -1) + np.diag(np.diag(Lb) / (2 * d))
    out = np.tril(oracle.chol_rev(np.diag(d), Lb))
    assert np.allclose(out, ref, rtol=0, atol=1e-15 * np.abs(ref).max())


@pytest.mark.parametrize("n", [1, 4, 16, 40])
def test_fwd_sigma_dot_equals_sigma(n):
    # Eq. 8: Sdot = Sigma = L L^T  =>  Ldot = L Phi(I) = L / 2.
    L, _, _ = synthetic.draw(n, n, lbar=False)
    Ld = oracle.chol_fwd(L, np.tril(L @ L.T))
    assert nerr(Ld, L / 2) < 1e-14


@pytest.mark.parametrize("n", [3, 12, 64])
def test_fwd_manufactured_solution(n):
    # Perturbation of Sigma = L L^T: Sdot = Ld0 L^T + L Ld0^T  =>  Ldot = Ld0.
    L, _, _ = synthetic.draw(n, 7 + n, lbar=False)
    Ld0 = np.tril(np.random.default_rng(n).standard_normal((n, n)))
    Sd = Ld0 @ L.T + L @ Ld0.T
    assert nerr(oracle.chol_fwd(L, np.tril(Sd)), Ld0) < 1e-13
    assert nerr(oracle.chol_fwd_symbolic(L, Sd), Ld0) < 1e-13


# ---------------------------------------------------------------- derivative definition

@pytest.mark.parametrize("n", [1, 2, 5, 8])
def test_rev_vs_central_finite_differences(n):
    # north star: FD of f = <Lbar, chol(Sigma)> on N <= 8; h = 1e-6 max|Sigma|.
    L, Lb, _ = synthetic.draw(n, 11 * n)
    ref = jacobian.fd_rev(L, Lb)
    assert nerr(oracle.chol_rev(L, Lb), ref) < 1e-8


@pytest.mark.parametrize("n", [1, 3, 6, 8])
def test_rev_vs_complex_step(n):
    # Sbar_kl = <Lbar, dchol/dSigma_kl>, Sigma_kl = Sigma_lk one variable.
    L, Lb, _ = synthetic.draw(n, 3 * n + 1)
    Jc = jacobian.jacobian_complex_step(L)
    idx = jacobian.vech_index(n)
    g = np.array([Lb[i, j] for (i, j) in idx])
    ref = np.zeros((n, n))
    for c, (k, l) in enumerate(idx):
        ref[k, l] = g @ Jc[:, c]
    assert nerr(oracle.chol_rev(L, Lb), ref) < 1e-13
    assert nerr(oracle.chol_rev_symbolic(L, Lb), ref) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 7, 12])
def test_fwd_vs_complex_step(n):
    L, _, Sd = synthetic.draw(n, 5 * n, sdot=True)
    ref = jacobian.ldot_complex_step(L, Sd)
    assert nerr(oracle.chol_fwd(L, np.tril(Sd)), ref) < 1e-13
    assert nerr(oracle.chol_fwd_symbolic(L, Sd), ref) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 4, 6])
def test_eq11_jacobian_vs_complex_step(n):
    # Eq. 11 against an independent derivative route.
    L, _, _ = synthetic.draw(n, 17 + n, lbar=False)
    Je, Jc = jacobian.jacobian_eq11(L), jacobian.jacobian_complex_step(L)
    assert np.abs(Je - Jc).max() <= 1e-13 * max(1.0, np.abs(Jc).max())


@pytest.mark.parametrize("n", [3, 6])
def test_rev_is_vjp_and_fwd_is_jvp_of_eq11(n):
    L, Lb, Sd = synthetic.draw(n, 23 + n, sdot=True)
    J = jacobian.jacobian_eq11(L)
    idx = jacobian.vech_index(n)
    g = np.array([Lb[i, j] for (i, j) in idx])
    rev = np.zeros((n, n))
    for c, (k, l) in enumerate(idx):
        rev[k, l] = g @ J[:, c]
    assert nerr(oracle.chol_rev(L, Lb), rev) < 1e-13
    v = np.array([Sd[k, l] for (k, l) in idx])  # one variable per (k,l), k >= l
    ld = J @ v
    fwd = np.zeros((n, n))
    for r, (i, j) in enumerate(idx):
        fwd[i, j] = ld[r]
    assert nerr(oracle.chol_fwd(L, np.tril(Sd)), fwd) < 1e-13


# ---------------------------------------------------------------- cross-method / invariants

@pytest.mark.parametrize("n", list(range(1, 11)) + [33, 64, 65])
def test_algorithmic_vs_symbolic(n):
    # all variants agree on N in {1..10, 33, 64, 65}.
    L, Lb, Sd = synthetic.draw(n, n, sdot=True)
    assert nerr(oracle.chol_rev(L, Lb), oracle.chol_rev_symbolic(L, Lb)) < 1e-12
    assert nerr(oracle.chol_fwd(L, np.tril(Sd)), oracle.chol_fwd_symbolic(L, Sd)) < 1e-12


@pytest.mark.parametrize("n", [1, 5, 30])
def test_eq9_symmetric_and_tril_matches_eq10(n):
    L, Lb, _ = synthetic.draw(n, 40 + n)
    s9 = oracle.chol_rev_symbolic_sym(L, Lb)
    assert np.array_equal(s9, s9.T)
    assert nerr(np.tril(s9), oracle.chol_rev_symbolic(L, Lb)) < 1e-13


@pytest.mark.parametrize("n", [8, 64, 200])
def test_adjoint_identity(n):
    # <Lbar, Ldot> = <tril(Sbar), tril(Sdot)>, normalised by ||Lbar|| ||Ldot||.
    L, Lb, Sd = synthetic.draw(n, 0, sdot=True)
    Ld = np.tril(oracle.chol_fwd(L, np.tril(Sd)))
    Sb = np.tril(oracle.chol_rev(L, Lb))
    lhs = np.sum(Lb * Ld)
    rhs = np.sum(Sb * np.tril(Sd))
    assert abs(lhs - rhs) <= 1e-14 * np.linalg.norm(Lb) * np.linalg.norm(Ld)


@pytest.mark.parametrize("s", [-3, 1, 5])
def test_power_of_two_scaling_bit_exact(s):
    # rev(2^s L, Lbar) = 2^-s rev(L, Lbar); rev(L, 2^s Lbar) = 2^s rev(L, Lbar); fwd likewise.
    n = 23
    L, Lb, Sd = synthetic.draw(n, 99, sdot=True)
    r = np.tril(oracle.chol_rev(L, Lb))
    assert np.array_equal(np.tril(oracle.chol_rev(L * 2.0 ** s, Lb)), r * 2.0 ** -s)
    assert np.array_equal(np.tril(oracle.chol_rev(L, Lb * 2.0 ** s)), r * 2.0 ** s)
    f = np.tril(oracle.chol_fwd(L, np.tril(Sd)))
    assert np.array_equal(np.tril(oracle.chol_fwd(L, np.tril(Sd) * 2.0 ** s)), f * 2.0 ** s)
    # Sigma scales by 2^{2s} when L scales by 2^s: Ldot(2^s L, 2^{2s} Sdot) = 2^s Ldot(L, Sdot)
    assert np.array_equal(np.tril(oracle.chol_fwd(L * 2.0 ** s, np.tril(Sd) * 4.0 ** s)), f * 2.0 ** s)


def test_linearity():
    n = 19
    L, Lb, Sd = synthetic.draw(n, 5, sdot=True)
    _, Lb2, Sd2 = synthetic.draw(n, 6, sdot=True)
    a, b = 0.7, -1.3
    r = oracle.chol_rev(L, a * Lb + b * Lb2)
    assert nerr(r, a * oracle.chol_rev(L, Lb) + b * oracle.chol_rev(L, Lb2)) < 1e-14
    f = oracle.chol_fwd(L, np.tril(a * Sd + b * Sd2))
    assert nerr(f, a * oracle.chol_fwd(L, np.tril(Sd)) + b * oracle.chol_fwd(L, np.tril(Sd2))) < 1e-14


def test_upper_triangle_never_read_or_written():
    # only tril is referenced; poison the upper triangles with NaN.
    n = 21
    L, Lb, Sd = synthetic.draw(n, 3, sdot=True)
    r = oracle.chol_rev(synthetic.poison_upper(L), synthetic.poison_upper(Lb))
    assert np.all(np.isfinite(np.tril(r))) and np.all(np.isnan(r[np.triu_indices(n, 1)]))
    assert np.array_equal(np.tril(r), np.tril(oracle.chol_rev(L, Lb)))
    f = oracle.chol_fwd(synthetic.poison_upper(L), synthetic.poison_upper(np.tril(Sd)))
    assert np.array_equal(np.tril(f), np.tril(oracle.chol_fwd(L, np.tril(Sd))))
    assert np.all(np.isnan(f[np.triu_indices(n, 1)]))


def test_singular_factor_reports_index():
    n = 6
    L, Lb, _ = synthetic.draw(n, 1)
    L[3, 3] = 0.0
    with pytest.raises(oracle.SingularFactor) as e:
        oracle.chol_rev(L, Lb)
    assert e.value.j == 4


# ---------------------------------------------------------------- blocked readings

@pytest.mark.parametrize("n,nb", [(1, 1), (5, 2), (5, 3), (17, 4), (33, 7), (33, 32), (33, 33), (33, 38), (70, 16)])
def test_blocked_rev_matches_unblocked(n, nb):
    # PAPER.md:689-707 ("partitioning into columns is arbitrary"; short block at the top-left);
    # checks the readings (Dbar + Dbar^T with tril(Dbar)) and nb-invariance.
    L, Lb, _ = synthetic.draw(n, 2 * n + nb)
    assert nerr(blocked.chol_blocked_rev(L, Lb, nb), oracle.chol_rev(L, Lb)) < 1e-13


@pytest.mark.parametrize("n,nb", [(1, 1), (5, 2), (17, 4), (33, 7), (33, 38), (70, 16)])
def test_blocked_fwd_matches_unblocked(n, nb):
    L, _, Sd = synthetic.draw(n, 3 * n + nb, sdot=True)
    assert nerr(blocked.chol_blocked_fwd(L, np.tril(Sd), nb), oracle.chol_fwd(L, np.tril(Sd))) < 1e-13


# ---------------------------------------------------------------- bench arithmetic

@pytest.mark.parametrize("n", [1, 2, 3, 32, 64, 511, 1024])
def test_flop_formula(n):
    assert sum(oracle.rev_column_flops(n, j) for j in range(n)) == oracle.rev_flops(n)
    assert oracle.rev_flops(32) == 22416 and oracle.rev_flops(16384) == 2932165255168
    assert oracle.fwd_flops(512) + oracle.rev_flops(512) == 179220480


def test_batched_matches_single():
    n, B = 9, 5
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=10, sdot=True)
    Lc, Ac, Dc = synthetic.to_colmajor(L), synthetic.to_colmajor(Lb), synthetic.to_colmajor(np.tril(Sd))
    assert not oracle.chol_rev_batched_colmajor(n, B, Lc, Ac).any()
    assert not oracle.chol_fwd_batched_colmajor(n, B, Lc, Dc).any()
    R, F = synthetic.from_colmajor(Ac), synthetic.from_colmajor(Dc)
    for b in range(B):
        assert np.array_equal(np.tril(R[b]), np.tril(oracle.chol_rev(L[b], Lb[b])))
        assert np.array_equal(np.tril(F[b]), np.tril(oracle.chol_fwd(L[b], np.tril(Sd[b]))))


def test_partial_sweep_is_prefix_of_full():
    n, jlo = 40, 25
    L, Lb, _ = synthetic.draw(n, 8)
    Lc, A1 = synthetic.to_colmajor(L), synthetic.to_colmajor(Lb)
    A2 = A1.copy()
    oracle.chol_rev_colmajor_inplace(n, Lc, A1, j_lo=jlo)
    oracle.chol_rev_colmajor_inplace(n, Lc, A2, j_lo=0)
    # columns >= jlo are final after the partial sweep (the sweep runs j = N..1)
    assert np.array_equal(A1[jlo:], A2[jlo:])


@pytest.mark.parametrize("n", [1, 2, 7, 64, 129, 700, 1100])
def test_fwd_cols_bit_identical(n):
    # the column-ordered evaluation (large-n parity tests) is the same arithmetic as chol_fwd:
    # every sum adds its terms in the same order, so the results agree bit for bit
    L, _, Sd = synthetic.draw(n, 31 + n, lbar=False, sdot=True)
    ref = oracle.chol_fwd(L, np.tril(Sd))
    Lc, Ac = synthetic.to_colmajor(L).copy(), synthetic.to_colmajor(np.tril(Sd)).copy()
    assert oracle.chol_fwd_colmajor_inplace(n, Lc, Ac) == 0
    assert np.array_equal(np.tril(synthetic.from_colmajor(Ac)), np.tril(ref))
    B = 3
    Lb3, _, Sd3 = synthetic.draw_batch(min(n, 64), B, seed=n, lbar=False, sdot=True)
    m = Lb3.shape[-1]
    Lc3, Ac3 = synthetic.to_colmajor(Lb3), synthetic.to_colmajor(np.tril(Sd3))
    assert not oracle.chol_fwd_cols_batched_colmajor(m, B, Lc3, Ac3).any()
    for b in range(B):
        assert np.array_equal(np.tril(synthetic.from_colmajor(Ac3[b])), np.tril(oracle.chol_fwd(Lb3[b], np.tril(Sd3[b]))))


@pytest.mark.parametrize("n", [1, 3, 64, 600, 1100])
def test_chol_cols_bit_identical(n):
    L, _, _ = synthetic.draw(n, 5 + n, lbar=False)
    S = L @ L.T
    ref = oracle.chol(S)
    Sc = synthetic.to_colmajor(S).copy()  # (to_colmajor may alias a 1 x 1 input)
    assert oracle.chol_colmajor_inplace(n, Sc) == 0
    assert np.array_equal(np.tril(synthetic.from_colmajor(Sc)), ref)
    # not positive definite -> the same failing column as chol_unblocked
    S2 = S.copy()
    S2[n // 2, n // 2] = -1.0
    with pytest.raises(oracle.NotPositiveDefinite) as e:
        oracle.chol(S2)
    assert oracle.chol_colmajor_inplace(n, synthetic.to_colmajor(S2).copy()) == e.value.j
