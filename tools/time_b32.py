import sys, torch, numpy as np
sys.path.insert(0, '.')
import synthetic, paper_1602_07527_b200 as cd
n, B = 32, 65536
L, Lb, _ = synthetic.draw_batch(n, B, seed=0)
to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(-1, -2)
Ld, A0 = to(L), to(Lb)
A = A0.clone()
ts = []
for i in range(25):
    A.copy_(A0); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); cd.chol_rev(Ld, A); e1.record(); torch.cuda.synchronize()
    if i >= 5: ts.append(e0.elapsed_time(e1))
print("batched 65536x32 rev: median %.4f ms min %.4f" % (sorted(ts)[10], min(ts)))
