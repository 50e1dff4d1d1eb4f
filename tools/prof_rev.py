"""Per-launch timeline (start, duration, stream) of one single-matrix reverse call, from the library's
event brackets (measurement tool):   CD_PROF_DUMP=1 python tools/prof_rev.py --n 8192"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    a = ap.parse_args()
    L, Lb, _ = synthetic.draw(a.n, 0)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0 = to(L), to(Lb)
    lib = cd.lib()
    lib.cd_profile_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_int64)]
    A = A0.clone()
    cd.chol_rev(Ld, A)
    torch.cuda.synchronize()
    A = A0.clone()
    torch.cuda.synchronize()
    lib.cd_profile_reset()
    lib.cd_profile_enable(1)
    cd.chol_rev(Ld, A)
    torch.cuda.synchronize()
    lib.cd_profile_enable(0)
    ms, fl, cnt = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    lib.cd_profile_read(0, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(cnt))
    sys.stderr.flush()


if __name__ == "__main__":
    main()
