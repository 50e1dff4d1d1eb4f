"""Print the fp32 path's normalised error against the fp64 oracle on fp32-rounded inputs
(measurement tool; test infrastructure may import the oracle).   python tools/f32_error.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402
from gpu_helpers import fp32_round, nerr, to_dev, to_host  # noqa: E402


def main():
    cases = [(512, 4, 64), (512, 4, 128), (1100, 1, 0), (2048, 1, 0)]
    for n, B, nb in cases:
        L, Lb, Sd = synthetic.draw_batch(n, B, seed=31 + n, sdot=True)
        L, Lb, Sd = fp32_round(L, Lb, Sd)
        kw = {"nb": nb} if nb else {}
        r = cd.chol_rev(to_dev(L, torch.float32), to_dev(Lb, torch.float32), **kw)
        er = nerr(to_host(r), np.stack([oracle.chol_rev(L[b], Lb[b]) for b in range(B)]))
        f = cd.chol_fwd(to_dev(L, torch.float32), to_dev(np.tril(Sd), torch.float32), **kw)
        ef = nerr(to_host(f), np.stack([oracle.chol_fwd(L[b], Sd[b]) for b in range(B)]))
        print(f"n={n} B={B} nb={nb or 'auto'}: rev {er:.3e}  fwd {ef:.3e}  (gate 1e-4)", flush=True)


if __name__ == "__main__":
    main()
