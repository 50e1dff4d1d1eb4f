"""One call of a BASELINE.json configuration, for ncu counter captures (measurement tool).
CFG = c0 (N=64 rev) | c1r / c1f (N=1024 rev / fwd) | c2 (65536 x 32 rev) | c3 (1024 x 512 fp32 rev+fwd)
| c4 (N=16384 rev).  A warm-up call precedes the measured one; use ncu -s to skip it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402

cfg = os.environ.get("CFG", "c4")
to = lambda m, dt=torch.float64: torch.from_numpy(synthetic.to_colmajor(m)).to(dt).cuda().transpose(-1, -2)  # noqa: E731
if cfg in ("c0", "c1r", "c1f", "c4"):
    n = {"c0": 64, "c1r": 1024, "c1f": 1024, "c4": 16384}[cfg]
    L, Lb, Sd = synthetic.draw(n, 0, sdot=cfg == "c1f")
    Ld, A0 = to(L), to(np.tril(Sd) if cfg == "c1f" else Lb)
    del L, Lb, Sd
    for _ in range(2):
        A = A0.clone()
        (cd.chol_fwd if cfg == "c1f" else cd.chol_rev)(Ld, A)
elif cfg == "c2":
    L, Lb, _ = synthetic.draw_batch(32, 65536, seed=0)
    Ld, A0 = to(L), to(Lb)
    for _ in range(2):
        cd.chol_rev(Ld, A0.clone())
elif cfg == "c3":
    L, Lb, Sd = synthetic.draw_batch(512, 1024, seed=0, sdot=True)
    Ld, A0, F0 = to(L, torch.float32), to(Lb, torch.float32), to(np.tril(Sd), torch.float32)
    for _ in range(2):
        cd.chol_rev_fwd(Ld, A0.clone(), F0.clone())
torch.cuda.synchronize()
print("ok", cfg)
