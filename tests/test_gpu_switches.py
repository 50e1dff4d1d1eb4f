"""GPU parity of the alternative panel schedules that measurement switches select (read once per
process by the library, so they run in child processes): the reverse panel's phase 1 on whole
128-row tiles / the 32 x 32 staged path (CD_PR_SPLIT=1) or on 64-row halves only (=2), and the
forward panel's phase 0 likewise (CD_PF_SPLIT).  The defaults (sub-tiles up to quarters) are what
every other -m gpu test exercises.  Same gate as tests/test_gpu_parity.py: 1e-10 (fp64) against the
oracle (PAPER.md:689-701 reverse, 655-666 forward)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1602_07527_b200 as cd
import synthetic
from gpu_helpers import nerr, to_dev, to_host

pytestmark = pytest.mark.gpu
child_only = pytest.mark.skipif(os.environ.get("CD_TEST_SWITCH_CHILD") != "1", reason="run by test_switches_in_subprocess")
TOL64 = 1e-10


@child_only
@pytest.mark.parametrize("n", [700, 1100, 2500])
def test_panel_schedules(n):
    L, Lb, Sd = synthetic.draw(n, 3 * n + 1, sdot=True)
    Lp, Ap, Fp = (synthetic.poison_upper(x) for x in (L, Lb, np.tril(Sd)))
    r = to_host(cd.chol_rev(to_dev(Lp), to_dev(Ap)))
    f = to_host(cd.chol_fwd(to_dev(Lp), to_dev(Fp)))
    assert nerr(r, oracle.chol_rev(L, Lb)) < TOL64
    assert nerr(f, oracle.chol_fwd(L, np.tril(Sd))) < TOL64
    iu = np.triu_indices(n, 1)
    assert np.all(np.isnan(r[iu])) and np.all(np.isnan(f[iu]))  # upper triangles never written


@pytest.mark.parametrize("split", ["1", "2"])
def test_switches_in_subprocess(split):
    if os.environ.get("CD_TEST_SWITCH_CHILD") == "1":
        pytest.skip("already in a child")
    env = dict(os.environ, CD_TEST_SWITCH_CHILD="1", CD_PR_SPLIT=split, CD_PF_SPLIT=split)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "test_panel_schedules", __file__],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
