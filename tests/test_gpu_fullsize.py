"""GPU parity at BASELINE.json's full configurations, WHOLE outputs against the oracle.

Every element of the lower triangle of the GPU result is compared with the CPU oracle
(oracle/oracle.c, the paper's unblocked algorithms) on the same seeded inputs, in the launch
configuration bench.py times (same entry points, same nb):

  * configs[4]: chol_rev fp64 N = 16384, nb = 128 (PAPER.md:689-701 vs the unblocked oracle
    PAPER.md:566-578) -- and chol_fwd at the same N (PAPER.md:655-666 vs 489-498), which
    bench.py reports beside it;
  * cd_chol_fwd_fused at N = 4096 (PAPER.md:501-503, 620-666 vs chol_unblocked + chol_unblocked_fwd);
  * configs[3]: all 1024 matrices of the fp32 N = 512 rev + fwd batch, through chol_rev_fwd
    (oracle in fp64 on the fp32-rounded inputs).

Tolerances are the north star's (max |out - ref| over the lower triangle / ||tril(ref)||_F:
1e-10 fp64, 1e-4 fp32).  The oracle runs on the host cores (OpenMP); these are the slow tests
of the suite (a few minutes on 16 cores)."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_1602_07527_b200 as cd
import synthetic
from gpu_helpers import fp32_round, nerr, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL64, TOL32 = 1e-10, 1e-4


def lower_err_img(got: np.ndarray, ref: np.ndarray, chunk: int = 512) -> float:
    """SURVEY c3 on column-major images (img[j, i] = M[i, j]): max over i >= j of
    |got - ref| / ||tril(ref)||_F, computed in row chunks of the image (2 GiB arrays).
    Any non-finite value in the lower triangle of `got` makes the error infinite."""
    n = ref.shape[0]
    num, den2 = 0.0, 0.0
    cols = np.arange(n)
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        mask = cols[None, :] >= np.arange(j0, j1)[:, None]
        g, r = got[j0:j1], ref[j0:j1]
        if not np.all(np.isfinite(g[mask])):
            return math.inf
        num = max(num, float(np.abs(np.where(mask, g - r, 0.0)).max()))
        den2 += float(np.sum(np.where(mask, r, 0.0) ** 2))
    return num / math.sqrt(den2) if den2 > 0 else num


def test_config5_rev_n16384_whole_output():
    n, nb = 16384, 128
    L, Lb, _ = synthetic.draw(n, 0)
    Lc, Ac = synthetic.to_colmajor(L), synthetic.to_colmajor(Lb)
    del L, Lb
    Ld = torch.from_numpy(Lc).cuda().transpose(0, 1)
    A = torch.from_numpy(Ac).cuda().transpose(0, 1)
    cd.chol_rev(Ld, A, nb=nb)  # bench.py's call (configs[4])
    got = A.transpose(0, 1).cpu().numpy()  # column-major image
    del A, Ld
    torch.cuda.empty_cache()
    # the host-buffer call that bench.py's "e2e" times (cd_chol_host, pinned column-major buffers)
    pin_L = torch.from_numpy(Lc).pin_memory().transpose(0, 1)
    pin_A = torch.from_numpy(Ac).pin_memory().transpose(0, 1)
    cd.chol_host("rev", pin_L, pin_A, nb=nb)
    got_host = pin_A.transpose(0, 1).numpy()
    h2d, d2h = cd.host_bytes()
    assert 0 < h2d < 0.7 * 2 * n * n * 8 and 0 < d2h < 0.7 * n * n * 8  # lower triangles only cross the bus
    assert oracle.chol_rev_colmajor_inplace(n, Lc, Ac) == 0  # the whole unblocked sweep, in place
    err = lower_err_img(got, Ac)
    err_host = lower_err_img(got_host, Ac)
    print(f"N={n} chol_rev whole-output error vs oracle: {err:.3e} (device buffers), {err_host:.3e} (cd_chol_host)")
    assert err < TOL64
    assert err_host < TOL64


def test_config5_fwd_n16384_whole_output():
    n, nb = 16384, 128
    L, _, Sd = synthetic.draw(n, 0, lbar=False, sdot=True)
    Lc, Fc = synthetic.to_colmajor(L), synthetic.to_colmajor(np.tril(Sd))
    del L, Sd
    Ld = torch.from_numpy(Lc).cuda().transpose(0, 1)
    F = torch.from_numpy(Fc).cuda().transpose(0, 1)
    cd.chol_fwd(Ld, F, nb=nb)  # bench.py's forward leg
    got = F.transpose(0, 1).cpu().numpy()
    del F, Ld
    torch.cuda.empty_cache()
    assert oracle.chol_fwd_colmajor_inplace(n, Lc, Fc) == 0
    err = lower_err_img(got, Fc)
    print(f"N={n} chol_fwd whole-output error vs oracle: {err:.3e}")
    assert err < TOL64


def test_chol_fwd_fused_n4096_whole_output():
    n = 4096
    L, _, Sd = synthetic.draw(n, 41, lbar=False, sdot=True)
    Sig = L @ L.T  # input construction: Sigma = L L^T
    Sc = synthetic.to_colmajor(Sig)
    Fc = synthetic.to_colmajor(np.tril(Sd))
    A = torch.from_numpy(Sc).cuda().transpose(0, 1)
    Ad = torch.from_numpy(Fc).cuda().transpose(0, 1)
    Lo, Fo = cd.chol_fwd_fused(A, Ad)
    gotL = Lo.transpose(0, 1).cpu().numpy()
    gotF = Fo.transpose(0, 1).cpu().numpy()
    # oracle: chol_unblocked, then chol_unblocked_fwd on the ORACLE's factor
    assert oracle.chol_colmajor_inplace(n, Sc) == 0
    assert oracle.chol_fwd_colmajor_inplace(n, Sc, Fc) == 0
    eL, eF = lower_err_img(gotL, Sc), lower_err_img(gotF, Fc)
    print(f"N={n} fused: L error {eL:.3e}, L_dot error {eF:.3e}")
    assert eL < TOL64 and eF < TOL64


def test_config4_all_1024_matrices_rev_fwd():
    n, B = 512, 1024
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=0, sdot=True)
    L, Lb, Sd = fp32_round(L, Lb, Sd)
    Sd = np.tril(Sd)
    Sb, Ldot = cd.chol_rev_fwd(to_dev(L, torch.float32), to_dev(Lb, torch.float32), to_dev(Sd, torch.float32))
    Sb, Ldot = to_host(Sb), to_host(Ldot)
    Lc = synthetic.to_colmajor(L)
    Ac, Fc = synthetic.to_colmajor(Lb), synthetic.to_colmajor(Sd)
    assert not oracle.chol_rev_batched_colmajor(n, B, Lc, Ac).any()
    assert not oracle.chol_fwd_cols_batched_colmajor(n, B, Lc, Fc).any()
    er = nerr(Sb, synthetic.from_colmajor(Ac))
    ef = nerr(Ldot, synthetic.from_colmajor(Fc))
    print(f"configs[3] all {B} matrices: rev error {er:.3e}, fwd error {ef:.3e}")
    assert er < TOL32 and ef < TOL32
