"""configs[3] step through cd.chol_rev_fwd (measurement tool).   python tools/time_rev_fwd.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def main():
    n, B = 512, 1024
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=0, sdot=True)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).float().cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0, F0 = to(L), to(Lb), to(np.tril(Sd))
    ts = []
    for i in range(12):
        A, F = A0.clone(), F0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cd.chol_rev_fwd(Ld, A, F)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    print(f"chol_rev_fwd 1024 x 512 fp32: median {sorted(ts)[len(ts) // 2]:.3f} ms  min {min(ts):.3f} ms")


if __name__ == "__main__":
    main()
