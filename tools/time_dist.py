"""Time the distributed reverse schedule (paper_1602_07527_b200/dist.py) for P simulated ranks on one
GPU (loopback: the ranks' steps run back to back, so the time is the sum of all ranks' work plus the
schedule's launches) against the single-GPU left-looking sweep (measurement tool).
    python tools/time_dist.py --n 8192 --nb 128 --world 1 2 4"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402
from paper_1602_07527_b200 import dist as cdd  # noqa: E402


def timed(fn, reps):
    ts = []
    for i in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--world", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = a.n
    L, Lb, _ = synthetic.draw(n, 0)
    Ld = torch.from_numpy(L).cuda()
    Lbd = torch.from_numpy(Lb).cuda()
    flops = (2 * n ** 3 / 3 + n * n / 2 + 11 * n / 6)
    Lc = cd.colmajor(Ld)
    t = timed(lambda: cd.chol_rev(Lc, cd.colmajor(Lbd)), a.reps)
    print(f"single-GPU chol_rev n={n}: {t:.2f} ms  {flops / t / 1e9:.1f} TFLOP/s")
    for P in a.world:
        t = timed(lambda: cdd.chol_rev_loopback(Ld, Lbd, a.nb, P), a.reps)
        print(f"distributed schedule, {P} simulated rank(s), nb={a.nb}: {t:.2f} ms  {flops / t / 1e9:.1f} TFLOP/s"
              " (all ranks' work serialised on one GPU, incl. storage split / assembly)")


if __name__ == "__main__":
    main()
