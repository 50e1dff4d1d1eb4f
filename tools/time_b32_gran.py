"""configs[2] (65536 x N=32 fp64 reverse) under different L2 fetch granularities
(cudaLimitMaxL2FetchGranularity = 32 / 64 / 128 bytes): the lower triangles touch partial 128-byte
lines at every column start.  Measurement tool:  python tools/time_b32_gran.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402


def cudart():
    import glob
    for pat in ("libcudart.so*",):
        for d in [os.path.join(os.path.dirname(torch.__file__), "lib")] + sys.path:
            for f in glob.glob(os.path.join(d, "nvidia", "cuda_runtime", "lib", pat)) + glob.glob(os.path.join(d, pat)):
                try:
                    return ctypes.CDLL(f)
                except OSError:
                    pass
    return ctypes.CDLL("libcudart.so")


def main():
    n, B = 32, 65536
    L, Lb, _ = synthetic.draw_batch(n, B, seed=0)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(-1, -2)  # noqa: E731
    Ld, A0 = to(L), to(Lb)
    A = A0.clone()
    rt = cudart()
    for gran in (128, 64, 32, 128):
        v = ctypes.c_size_t(gran)
        rc = rt.cudaDeviceSetLimit(ctypes.c_int(0x05), v)  # cudaLimitMaxL2FetchGranularity
        got = ctypes.c_size_t(0)
        rt.cudaDeviceGetLimit(ctypes.byref(got), ctypes.c_int(0x05))
        ts = []
        for i in range(25):
            A.copy_(A0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cd.chol_rev(Ld, A)
            b.record()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b))
        t = float(np.median(ts))
        print(f"L2 fetch granularity {gran} (rc {rc}, now {got.value}): {t * 1e3:.1f} us, "
              f"{B / (t * 1e-3):.3e} matrices/s, {B * 12672 / (t * 1e-3) / 1e9 / 6536.4:.3f} of HBM", flush=True)


if __name__ == "__main__":
    main()
