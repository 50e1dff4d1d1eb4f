"""configs[3] (1024 x N=512 fp32) warm per-launch timeline of chol_rev and chol_fwd run alone, and
the chol_rev_fwd step (measurement tool).   CD_PROF_DUMP=1 python tools/prof_c3.py [--n 512 --batch 1024]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402

NAMES = ["gemm", "reduce", "sweep", "trinv", "other", "symm", "panel"]


def timed(fn, reps=7):
    ts = []
    for i in range(reps + 2):
        fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(-1)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--nb", type=int, default=None)
    a = ap.parse_args()
    n, B = a.n, a.batch
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=0, sdot=True)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).float().cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0, F0 = to(L), to(Lb), to(np.tril(Sd))
    A, F = A0.clone(), F0.clone()

    def reset(i):
        if i >= 0:
            A.copy_(A0)
            F.copy_(F0)

    def rev(i):
        reset(i)
        if i < 0:
            cd.chol_rev(Ld, A, nb=a.nb)

    def fwd(i):
        reset(i)
        if i < 0:
            cd.chol_fwd(Ld, F, nb=a.nb)

    def both(i):
        reset(i)
        if i < 0:
            cd.chol_rev_fwd(Ld, A, F, nb=a.nb)

    print(f"n {n} batch {B}: rev {timed(rev):.3f} ms  fwd {timed(fwd):.3f} ms  rev_fwd {timed(both):.3f} ms", flush=True)
    lib = cd.lib()
    lib.cd_profile_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_int64)]
    for name, fn in (("rev", rev), ("fwd", fwd), ("rev_fwd", both)):
        fn(0)
        torch.cuda.synchronize()
        lib.cd_profile_reset()
        lib.cd_profile_enable(1)
        fn(-1)
        torch.cuda.synchronize()
        lib.cd_profile_enable(0)
        print(f"--- {name}", flush=True)
        for cls in range(7):
            ms, fl, cnt = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
            lib.cd_profile_read(cls, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(cnt))
            sys.stderr.flush()
            if cnt.value:
                print(f"{NAMES[cls]:7s} {cnt.value:4d} launches {ms.value:8.3f} ms", flush=True)
        lib.cd_profile_reset()


if __name__ == "__main__":
    main()
