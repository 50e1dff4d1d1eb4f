"""configs[3] step (1024 x N=512 fp32, rev + fwd) with the two independent sweeps on one stream vs on two
streams (measurement tool).   python tools/time_c3_streams.py"""
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
    A, F = A0.clone(), F0.clone()
    s_main = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()

    def seq():
        cd.chol_rev(Ld, A)
        cd.chol_fwd(Ld, F)

    def two():
        s2.wait_stream(s_main)
        cd.chol_rev(Ld, A)
        with torch.cuda.stream(s2):
            cd.chol_fwd(Ld, F)
        s_main.wait_stream(s2)

    ss = [torch.cuda.Stream() for _ in range(4)]

    def four(parts=2):
        h = B // parts
        for x in ss:
            x.wait_stream(s_main)
        for i in range(parts):
            with torch.cuda.stream(ss[2 * i % 4]):
                cd.chol_rev(Ld[i * h:(i + 1) * h], A[i * h:(i + 1) * h])
            with torch.cuda.stream(ss[(2 * i + 1) % 4]):
                cd.chol_fwd(Ld[i * h:(i + 1) * h], F[i * h:(i + 1) * h])
        for x in ss:
            s_main.wait_stream(x)

    for name, fn in (("one stream", seq), ("two streams", two), ("four streams (halves)", four),
                     ("one stream", seq), ("two streams", two), ("four streams (halves)", four)):
        ts = []
        for i in range(7):
            A.copy_(A0)
            F.copy_(F0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"{name}: median {sorted(ts)[len(ts) // 2]:.3f} ms  min {min(ts):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
