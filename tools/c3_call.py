"""configs[3] (1024 x N=512 fp32): two cd.chol_rev_fwd calls and nothing else, for an ncu launch
list (measurement tool).   python tools/c3_call.py [--calls 2]"""
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
    ap.add_argument("--calls", type=int, default=2)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--batch", type=int, default=1024)
    a = ap.parse_args()
    L, Lb, Sd = synthetic.draw_batch(a.n, a.batch, seed=0, sdot=True)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).float().cuda().transpose(-1, -2)  # noqa: E731
    Ld, A, F = to(L), to(Lb), to(np.tril(Sd))
    for _ in range(a.calls):
        cd.chol_rev_fwd(Ld, A, F)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
