"""configs[1]-shaped timing: fp64 N (default 1024) reverse and forward, CUDA events, L2 flushed
between calls.  Run under CD_DEBUG_PANEL_SKIP=<mask> to time the panel phases by omission (results
then wrong).  Measurement tool:  N=1024 python tools/time_mid.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_07527_b200 as cd  # noqa: E402
import synthetic  # noqa: E402

n = int(os.environ.get("N", "1024"))
L, Lb, Sd = synthetic.draw(n, 0, sdot=True)
to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(0, 1)  # noqa: E731
Ld, A0, F0 = to(L), to(Lb), to(np.tril(Sd))
A = A0.clone()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name, fn, src in ((("rev", cd.chol_rev, A0), ("fwd", cd.chol_fwd, F0)) if os.environ.get("ONLY") is None else [x for x in (("rev", cd.chol_rev, A0), ("fwd", cd.chol_fwd, F0)) if x[0] == os.environ["ONLY"]]):
    ts = []
    for i in range(25):
        A.copy_(src)
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(Ld, A)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b))
    print(f"N={n} {name} skip={os.environ.get('CD_DEBUG_PANEL_SKIP', '0')}: median {np.median(ts) * 1e3:.1f} us",
          flush=True)
