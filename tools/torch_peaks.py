"""Measure torch (cuBLAS) fp64 / fp32 / tf32 matmul peaks on the box (context for the roofline)."""
import json, time, torch
def bench(dtype, n=8192, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype); b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained 4 s
    t0 = time.time(); cnt = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    while time.time() - t0 < 4.0:
        a @ b; cnt += 1
        if cnt % 8 == 0: torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sus = e0.elapsed_time(e1) / cnt
    fl = 2.0 * n ** 3
    return {"burst_tflops": fl / best / 1e9, "sustained_tflops": fl / sus / 1e9}
out = {"fp64": bench(torch.float64), "fp32": bench(torch.float32), "tf32": bench(torch.float32, tf32=True)}
print(json.dumps(out))
