"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck) runs (measurement / QA tool, not the product path).  Round 2: compute-sanitizer is
refused on this GPU pool (the runner exits 86 before starting it), so these cases were last run
under it in round 1; the round-2 kernels are covered by the NaN-guarded parity tests instead."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def dev(m, dt=torch.float64):
    return torch.from_numpy(synthetic.to_colmajor(m)).to(dt).cuda().transpose(-1, -2)


def main():
    for n, B in ((300, 1), (300, 2), (32, 37), (24, 5), (64, 3), (517, 1)):
        L, Lb, Sd = (synthetic.draw(n, n, sdot=True) if B == 1 else synthetic.draw_batch(n, B, seed=n, sdot=True))
        cd.chol_rev(dev(L), dev(Lb))
        cd.chol_fwd(dev(L), dev(np.tril(Sd)))
        cd.chol_rev(dev(L, torch.float32), dev(Lb, torch.float32))
        cd.chol_fwd(dev(L, torch.float32), dev(np.tril(Sd), torch.float32))
        if n <= 64:
            cd.chol_rev(dev(L), dev(Lb), route="symbolic")
        S = np.einsum("...ij,...kj->...ik", L, L)
        cd.chol_fwd_fused(dev(S), dev(np.tril(Sd)))
    # panel phase 1 on 64-row sub-tiles (7 tiles per panel at most) and the batched N = 32 kernel
    L, Lb, Sd = synthetic.draw(1024, 1, sdot=True)
    cd.chol_rev(dev(L), dev(Lb))
    cd.chol_fwd(dev(L), dev(np.tril(Sd)))  # k_fwd_sk with the deferred stream-K fixup (few output tiles)
    if os.environ.get("CD_SAN_BIG", "1") != "0":  # k_symm_ll: in-kernel and deferred fixups, short first block
        L, Lb, Sd = synthetic.draw(2048 + 40, 2, sdot=True)
        cd.chol_rev(dev(L), dev(Lb))
        cd.chol_fwd(dev(L), dev(np.tril(Sd)))
    L, Lb, _ = synthetic.draw_batch(32, 1000, seed=1)
    cd.chol_rev(dev(L), dev(Lb))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
