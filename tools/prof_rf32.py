"""One configs[3]-shaped fused call (1024 x N=512 fp32, rev + fwd) for ncu captures (measurement tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402

n, B = int(os.environ.get("N", "512")), int(os.environ.get("B", "1024"))
L, Lb, Sd = synthetic.draw_batch(n, min(B, 64), seed=0, sdot=True)
rep = (B + L.shape[0] - 1) // L.shape[0]
to = lambda m: torch.from_numpy(synthetic.to_colmajor(np.concatenate([m] * rep)[:B])).float().cuda().transpose(-1, -2)  # noqa: E731
Ld, A, F = to(L), to(Lb), to(np.tril(Sd))
for _ in range(int(os.environ.get("REPS", "2"))):
    cd.chol_rev_fwd(Ld, A.clone(), F.clone())
torch.cuda.synchronize()
print("ok")
