"""configs[3] step (1024 x N=512 fp32, rev + fwd) through chol_rev_fwd: the fused kernel vs the
layered schedule (the default; CD_RF32=1 selects the fused kernel).  Measurement tool:  python tools/time_rf32.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def main():
    n = int(os.environ.get("N", "512"))
    B = int(os.environ.get("B", "1024"))
    L, Lb, Sd = synthetic.draw_batch(n, B, seed=0, sdot=True)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).float().cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0, F0 = to(L), to(Lb), to(np.tril(Sd))
    A, F = A0.clone(), F0.clone()
    for name, fn in (("rev+fwd", lambda: cd.chol_rev_fwd(Ld, A, F)), ("rev", lambda: cd.chol_rev(Ld, A)),
                     ("fwd", lambda: cd.chol_fwd(Ld, F))):
        ts = []
        for i in range(8):
            A.copy_(A0)
            F.copy_(F0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        print(f"{'fused' if os.environ.get('CD_RF32') else 'layered'} n={n} B={B} {name}: "
              f"median {np.median(ts):.3f} ms  min {min(ts):.3f} ms", flush=True)
        if os.environ.get("CD_RF32_PROF") and os.environ.get("CD_RF32"):
            import ctypes
            out = (ctypes.c_longlong * 8)()
            cd.lib().cd_rf32_prof_read(out, 148)
            items = max(1, out[7])
            names = ["wait-acc", "loads", "s1 (R2-R4 | F3)", "s2 (Dbar' | F4)", "s3 (R5)", "publish"]
            print("   per item (matrix sweep), cycles: " + "  ".join(f"{nm} {out[i] / items:.0f}" for i, nm in
                                                                  enumerate(names)) + f"  (items {items})", flush=True)


if __name__ == "__main__":
    main()
