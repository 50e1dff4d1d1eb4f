"""Phase clocks of the on-chip reverse sweep for one small matrix (CTA 0; measurement tool).
    python tools/clk_small.py [--n 64]"""
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
    ap.add_argument("--n", type=int, default=64)
    a = ap.parse_args()
    L, Lb, _ = synthetic.draw(a.n, 0)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0 = to(L), to(Lb)
    lib = cd.lib()
    lib.cd_debug_phase_clocks.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = (ctypes.c_longlong * 40)()
    for cold in (False, True):
        for rep in range(4):
            A = A0.clone()
            if cold:
                flush.fill_(rep)
            torch.cuda.synchronize()
            lib.cd_debug_phase_clocks(1, None, 0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cd.chol_rev(Ld, A)
            e1.record()
            torch.cuda.synchronize()
            lib.cd_debug_phase_clocks(0, out, 40)
        c = [out[i] - out[0] for i in range(40)]
        steps = [c[3 + 4 * s] for s in range(8)] + [c[35]]
        print(f"n={a.n} {'cold' if cold else 'warm'}: event {e0.elapsed_time(e1)*1e3:.1f} us; cycles stage {c[1]} inv {c[2]-c[1]} "
              f"steps {[steps[i+1]-steps[i] for i in range(8)]} (s1/s23/s4/s5 of step 0: "
              f"{[c[4]-c[3], c[5]-c[4], c[6]-c[5], c[7]-c[6]]}) store {c[36]-c[35]} total {c[36]}; "
              f"stage L issued {c[37]} A issued {c[38]} landed {c[39]}")


if __name__ == "__main__":
    main()
