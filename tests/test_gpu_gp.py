"""GP log-likelihood gradient end to end: libcholdiff's fused factorisation
+ forward mode and reverse mode inside a whole computation, against the textbook closed form
and against central finite differences of f (both fp64)."""
import math
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples"))
from gp_loglik_grad import loglik_and_grad, reference_grad  # noqa: E402

pytestmark = pytest.mark.gpu


def _f(x, y, theta):
    """f(theta) in numpy fp64 (for finite differences)."""
    from gp_loglik_grad import kernel_and_derivs
    K = kernel_and_derivs(torch.from_numpy(x), torch.from_numpy(theta))[0].numpy()
    c = np.linalg.cholesky(K)
    a = np.linalg.solve(c, y)
    return -0.5 * a @ a - np.log(np.diag(c)).sum() - 0.5 * len(y) * math.log(2 * math.pi)


@pytest.mark.parametrize("n", [100, 300, 700])
def test_gp_gradient(n):
    rng = np.random.default_rng(n)
    x = rng.uniform(-2, 2, (n, 2))
    y = np.cos(x).sum(1) + 0.1 * rng.standard_normal(n)
    theta = np.log(np.array([0.7, 1.1, 0.4]))
    dev = torch.device("cuda")
    f, g, fwd0 = loglik_and_grad(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev),
                                 torch.from_numpy(theta).to(dev))
    g = g.cpu().numpy()
    ref = reference_grad(x, y, theta)
    assert abs(f - _f(x, y, theta)) < 1e-8 * max(1.0, abs(f))
    assert np.max(np.abs(g - ref)) < 1e-8 * np.max(np.abs(ref))
    assert abs(fwd0 - ref[0]) < 1e-8 * np.max(np.abs(ref))  # forward mode agrees with reverse
    h = 1e-5
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        fd = (_f(x, y, theta + e) - _f(x, y, theta - e)) / (2 * h)
        assert abs(fd - g[k]) < 1e-5 * max(1.0, abs(g[k]))
