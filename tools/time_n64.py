"""configs[0] latency the way bench.py times it (L2 flushed before every call, CUDA events around
the call and around a CUDA-graph replay of it), plus the in-kernel phase clocks (measurement tool).
    python tools/time_n64.py [--n 64]"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    a = ap.parse_args()
    L, Lb, _ = synthetic.draw(a.n, 0)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0 = to(L), to(Lb)
    A = A0.clone()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn, reps=50):
        ts = []
        for i in range(reps + 5):
            A.copy_(A0)
            flush.fill_(i & 255)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    t = timed(lambda: cd.chol_rev(Ld, A))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cd.chol_rev(Ld, A)
    tg = timed(g.replay)
    print(f"n={a.n}: {t:.2f} us per call, {tg:.2f} us under graph replay (L2 flushed)")


if __name__ == "__main__":
    main()
