"""Single-matrix latency of the two routes under CUDA-graph replay (measurement tool):
python tools/latency_routes.py"""
import sys, torch
sys.path.insert(0, ".")
import paper_1602_07527_b200 as cd, synthetic
for n in (16, 32, 48, 64):
    L, Lb, _ = synthetic.draw(n, 0)
    to = lambda m: torch.from_numpy(synthetic.to_colmajor(m)).cuda().transpose(0, 1)
    Ld, A0 = to(L), to(Lb)
    A = A0.clone()
    for route in ("algorithmic", "symbolic"):
        g = torch.cuda.CUDAGraph()
        cd.chol_rev(Ld, A, route=route)
        with torch.cuda.graph(g):
            cd.chol_rev(Ld, A, route=route)
        ts = []
        for i in range(30):
            A.copy_(A0); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            if i > 3: ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(n, route, "%.2f us" % (1e3 * ts[len(ts) // 2]))
