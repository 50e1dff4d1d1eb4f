"""GPU parity of the fp32 batched schedule with 128-wide panels (the diagonal blocks on
k_rf_diag128 -- the block's own sweep as two 64-wide steps, PAPER.md:689-701 / 655-666 -- and the
128-wide inverses completed by k_rf_inv128) against the oracle, every matrix of the batch, at the
1e-4 fp32 gate; upper triangles untouched."""
import numpy as np
import pytest
import torch

import oracle
import paper_1602_07527_b200 as cd
import synthetic
from gpu_helpers import fp32_round, nerr, to_dev, to_host

pytestmark = pytest.mark.gpu


def _inputs(n, B, seed):
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=seed, sdot=True)
    return fp32_round(L, Lb, Sd)


@pytest.mark.parametrize("n", [256, 384, 512, 640])
def test_rev_fwd_nb128_all_matrices(n):
    B = 5
    L, Lb, Sd = _inputs(n, B, 11 + n)
    Lt = to_dev(L, torch.float32)
    Sb = to_host(cd.chol_rev(Lt, to_dev(Lb, torch.float32), nb=128))
    Ld = to_host(cd.chol_fwd(Lt, to_dev(np.tril(Sd), torch.float32), nb=128))
    iu = np.triu_indices(n, 1)
    for b in range(B):
        assert nerr(Sb[b], oracle.chol_rev(L[b], Lb[b])) < 1e-4
        assert nerr(Ld[b], oracle.chol_fwd(L[b], np.tril(Sd[b]))) < 1e-4
    assert np.array_equal(Sb[:, iu[0], iu[1]], Lb[:, iu[0], iu[1]].astype(np.float32))
    assert np.array_equal(Ld[:, iu[0], iu[1]], np.tril(Sd)[:, iu[0], iu[1]].astype(np.float32))


def test_rev_fwd_shared_inverses_nb128():
    n, B = 512, 7
    L, Lb, Sd = _inputs(n, B, 5)
    Lt = to_dev(L, torch.float32)
    Sb, Ld = cd.chol_rev_fwd(Lt, to_dev(Lb, torch.float32), to_dev(np.tril(Sd), torch.float32), nb=128)
    Sb, Ld = to_host(Sb), to_host(Ld)
    for b in range(B):
        assert nerr(Sb[b], oracle.chol_rev(L[b], Lb[b])) < 1e-4
        assert nerr(Ld[b], oracle.chol_fwd(L[b], np.tril(Sd[b]))) < 1e-4


def test_nb128_matches_nb64_closely():
    # two partitions of the same sweep: both within the gate of each other
    n, B = 384, 9
    L, Lb, Sd = _inputs(n, B, 3)
    Lt = to_dev(L, torch.float32)
    a = to_host(cd.chol_rev(Lt, to_dev(Lb, torch.float32), nb=128))
    c = to_host(cd.chol_rev(Lt, to_dev(Lb, torch.float32), nb=64))
    for b in range(B):
        assert nerr(a[b], c[b].astype(np.float64)) < 1e-4
