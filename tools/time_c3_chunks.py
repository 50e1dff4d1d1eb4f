"""configs[3] (1024 x N=512 fp32, rev + fwd) split into batch chunks spread over several streams, so that
the working set of the kernels in flight stays in L2 (measurement tool).
    python tools/time_c3_chunks.py [--nb 128]"""
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
    ap.add_argument("--nb", type=int, default=None)
    a = ap.parse_args()
    n, B = 512, 1024
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=0, sdot=True)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).float().cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0, F0 = to(L), to(Lb), to(np.tril(Sd))
    A, F = A0.clone(), F0.clone()
    s_main = torch.cuda.current_stream()
    ss = [torch.cuda.Stream() for _ in range(16)]
    ref_a = ref_f = None

    def run(chunk, nstreams, mode):
        nch = B // chunk
        for x in ss[:nstreams]:
            x.wait_stream(s_main)
        for i in range(nch):
            sl = slice(i * chunk, (i + 1) * chunk)
            if mode == "pair":
                with torch.cuda.stream(ss[i % nstreams]):
                    cd.chol_rev_fwd(Ld[sl], A[sl], F[sl], nb=a.nb)
            else:
                with torch.cuda.stream(ss[(2 * i) % nstreams]):
                    cd.chol_rev(Ld[sl], A[sl], nb=a.nb)
                with torch.cuda.stream(ss[(2 * i + 1) % nstreams]):
                    cd.chol_fwd(Ld[sl], F[sl], nb=a.nb)
        for x in ss[:nstreams]:
            s_main.wait_stream(x)

    for chunk, nst, mode in ((1024, 1, "pair"), (512, 2, "pair"), (256, 4, "pair"), (128, 4, "pair"), (128, 8, "pair"),
                             (64, 8, "pair"), (64, 16, "pair"), (256, 4, "split"), (128, 8, "split"), (64, 16, "split"),
                             (1024, 1, "pair")):
        ts = []
        for i in range(7):
            A.copy_(A0)
            F.copy_(F0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(chunk, nst, mode)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        if ref_a is None:
            ref_a, ref_f = A.clone(), F.clone()
        da = (A - ref_a).abs().max().item()
        df = (F - ref_f).abs().max().item()
        print(f"chunk {chunk:5d} streams {nst:2d} {mode:5s}: median {sorted(ts)[len(ts) // 2]:.3f} ms  "
              f"min {min(ts):.3f} ms  (max diff vs first {da:.2e} {df:.2e})", flush=True)


if __name__ == "__main__":
    main()
