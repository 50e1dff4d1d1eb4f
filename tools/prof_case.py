"""Run one small case of the hot path for ncu captures (measurement tool, not the product path).

  python tools/prof_case.py --case rev --n 8192      # blocked reverse sweep, single matrix
  python tools/prof_case.py --case batched --n 32 --batch 65536
  python tools/prof_case.py --case fwd --n 4096
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="rev")
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dt = torch.float64 if a.dtype == "f64" else torch.float32
    if a.batch == 1:
        L, Lb, Sd = synthetic.draw(a.n, 0, sdot=a.case == "fwd")
    else:
        L, Lb, Sd = synthetic.draw_batch(a.n, a.batch, seed=0, sdot=a.case == "fwd")
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).to(dt).cuda().transpose(-1, -2)  # noqa: E731
    Ld = to(L)
    A0 = to(Lb if a.case != "fwd" else np.tril(Sd))
    for _ in range(a.reps):
        A = A0.clone()
        if a.case == "fwd":
            cd.chol_fwd(Ld, A, nb=a.nb)
        else:
            cd.chol_rev(Ld, A, nb=a.nb)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
