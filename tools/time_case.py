"""Time one hot-path case with CUDA events (measurement tool, not the product path).

  python tools/time_case.py --case rev --n 512 --batch 1024 --dtype f32 --nb 64 --reps 5
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
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--nb", type=int, nargs="+", default=[128])
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dt = torch.float64 if a.dtype == "f64" else torch.float32
    if a.batch == 1:
        L, Lb, Sd = synthetic.draw(a.n, 0, sdot=a.case in ("fwd", "fused"))
    else:
        L, Lb, Sd = synthetic.draw_batch(a.n, a.batch, seed=0, sdot=a.case in ("fwd", "fused"))
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).to(dt).cuda().transpose(-1, -2)  # noqa: E731
    Ld = to(L)
    A0 = to(Lb if a.case not in ("fwd", "fused") else np.tril(Sd))
    if a.case == "fused":
        S = Ld @ Ld.transpose(-1, -2)  # Sigma = L L^T on the device
        S = S.transpose(-1, -2).contiguous().transpose(-1, -2)
    for nb in a.nb:
        ts = []
        for i in range(a.reps + 2):
            A = A0.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            if a.case == "fused":  # Sigma in A0's slot is replaced by a copy of L L^T
                cd.chol_fwd_fused(S.clone(), A)
            elif a.case == "fwd":
                cd.chol_fwd(Ld, A, nb=nb)
            else:
                cd.chol_rev(Ld, A, nb=nb)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"{a.case} n={a.n} batch={a.batch} {a.dtype} nb={nb}: min {min(ts):.3f} ms  med {sorted(ts)[len(ts)//2]:.3f} ms")


if __name__ == "__main__":
    main()
