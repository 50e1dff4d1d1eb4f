#!/usr/bin/env python
"""bench.py -- throughput of the Cholesky-derivative hot path on B200 (arXiv 1602.07527).

Default workload (BASELINE.json metric "chol_rev GFLOP/s (fp64, N=16384) ..."; configs[4]):
one reverse-mode sweep (L, Lbar) -> tril(Sigma_bar) of a single fp64 N=16384 matrix
(PAPER.md:689-701), seed 0, nb=128.  A "step" is one complete chol_rev call.  At
--gpus N > 1 every rank runs its own replica (the single-matrix sweep does not shard,
DESIGN.md §7): scaling "weak", value = sum over ranks.

The same JSON line carries, measured in the same run:
  * "batched": configs[2], 65536 x N=32 fp64 reverse, matrices/s, sharded by matrix
    across ranks (NCCL all_gather of the results timed separately), HBM roofline;
  * "roofline": the dominant kernel (the DMMA GEMM of the blocked sweep), achieved
    algorithmic TFLOP/s from per-launch CUDA events inside the timed steps;
  * "e2e": the same metric through the host-buffer C-ABI call (cd_chol_host), with
    the H2D copies of L and Abar and the D2H copy of the result inside the timing;
  * "cpu_baseline": the CPU oracle (oracle/, plain C, OpenMP) on the host cores,
    on a bounded sample of the same workload (rank 0, N=1 only);
  * "clocks": NVML SM clocks / throttle reasons sampled during the timed steps.

--impl reference: the CPU oracle (the reference arm for this tier) timed on the
same metric / config, each step a bounded sample (the trailing columns of the
sweep), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chol_rev GFLOP/s (fp64, N=16384) and batched matrices/s; % of roofline"
FP64_PEAK_TFLOPS = 37.0     # measured DMMA issue-rate peak (tools/microbench_fp64.cu, profiles/r01_microbench_fp64.txt)
CUBLAS_DGEMM_TFLOPS = 35.5  # measured torch.matmul fp64 8192^3 (profiles/r01_torch_peaks.json), context only
TF32_PEAK_TFLOPS = 1638.4 / 2  # MEASURED_PEAKS bf16 dense x the guide's nominal tf32:bf16 ratio (1:2)


def rev_flops(n: int) -> int:
    return (4 * n ** 3 + 3 * n ** 2 + 11 * n) // 6


def fwd_flops(n: int) -> int:
    return (4 * n ** 3 + 3 * n ** 2 + 5 * n) // 6


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while running."""

    REASONS = {
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4,
    }

    def __init__(self, torch_device):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            uuid = str(torch.cuda.get_device_properties(torch_device).uuid)
            try:
                self._h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU") else uuid)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(torch_device.index or 0)
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.error = str(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._h is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- distributed
class Dist:
    def __init__(self, want: int):
        import torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.want = want
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist
        self.device = torch.device("cuda", self.local)

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------- timing
def timed_steps(step, restore, K: int, W: int, dist: Dist, stream, before_timed=None):
    """W untimed warm-ups; then K steps, each bracketed by CUDA events on `stream`
    (restore() runs before each step, outside the events).  Barrier + synchronize
    on both sides.  Returns per-step ms (this rank)."""
    import torch
    for _ in range(W):
        restore()
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    if before_timed:
        before_timed()
    evs = []
    for _ in range(K):
        restore()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def colmajor_dev(m: np.ndarray, device, dtype=None):
    import torch
    import synthetic
    t = torch.from_numpy(synthetic.to_colmajor(m))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device).transpose(-1, -2)


# ----------------------------------------------------------------------------- workloads
def bench_single_rev(args, dist: Dist):
    """configs[4]: single fp64 reverse sweep, N = args.n (16384)."""
    import torch
    import paper_1602_07527_b200 as cd
    import synthetic

    n, nb = args.n, args.nb
    t0 = time.time()
    L, Lb, _ = synthetic.draw(n, args.seed)
    Lcm = synthetic.to_colmajor(L)
    Acm = synthetic.to_colmajor(Lb)
    del L, Lb
    gen_s = time.time() - t0
    dev = dist.device
    Ld = torch.from_numpy(Lcm).to(dev).transpose(0, 1)
    A0 = torch.from_numpy(Acm).to(dev).transpose(0, 1)
    A = A0.clone()
    stream = torch.cuda.current_stream(dev)

    def step():
        cd.chol_rev(Ld, A, nb=nb)

    def restore():
        A.copy_(A0)

    # the same steps, with per-kernel-class event timing switched on (roofline evidence)
    Lib = cd.lib()

    def start_timed():
        cd.reset_launch_count()
        Lib.cd_profile_reset()
        Lib.cd_profile_enable(1)

    # the timed steps carry no instrumentation (per-launch event pairs cost ~1.5 % here); the
    # same steps are then repeated with per-kernel-class events for the roofline evidence
    with ClockSampler(dev) as clk:
        ms = timed_steps(step, restore, args.steps, args.warmup, dist, stream, before_timed=cd.reset_launch_count)
    launches = cd.launch_count()  # library kernel launches inside the timed steps
    timed_steps(step, restore, max(1, min(args.steps, 3)), 0, dist, stream, before_timed=start_timed)
    Lib.cd_profile_enable(0)
    prof = read_profile(Lib)
    Lib.cd_profile_reset()

    mean_ms = statistics.mean(ms)
    worst = dist.max(mean_ms)
    fl = rev_flops(n)
    value = fl * dist.world / (worst * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(worst, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded PCG64 generator, synthetic/; no dataset)",
        "config": {"workload": f"configs[4]: chol_rev fp64 single matrix N={n}, seed {args.seed}, nb={nb}",
                   "n": n, "nb": nb, "batch": 1,
                   "parallelism": "replicas" if dist.world > 1 else "single-gpu",
                   "l2": "inputs larger than L2 (2 GiB per matrix); Abar restored from a pristine device copy "
                         "before every step, outside the timed events"},
        "step_ms": {"min": round(min(ms), 3), "median": round(statistics.median(ms), 3),
                    "max": round(max(ms), 3)},
        "gpu_launches": int(launches),
        "input_generation_s": round(gen_s, 1),
    }
    total_ms = sum(v[0] for v in prof.values())
    # dominant kernel class = the largest device-time share among the tensor-core classes
    dom = max(("symm", "gemm", "panel"), key=lambda k: prof[k][0])
    g_ms, g_fl, g_n = prof[dom]
    if g_n:
        per_launch_ms = g_ms / g_n
        achieved = g_fl / (g_ms * 1e-3) / 1e12
        peaks = measured_peaks()
        out["roofline"] = {
            "kernel": KERNEL_NAMES[dom] + ", all launches of the timed steps",
            "bound": "tensor", "achieved": round(achieved, 2), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
            "peak_source": "measured fp64 DMMA issue rate on this pool (tools/microbench_fp64.cu -> "
                           "profiles/r01_microbench_fp64.txt); MEASURED_PEAKS.json has no fp64 entry",
            "frac_of_cublas_dgemm": round(achieved / CUBLAS_DGEMM_TFLOPS, 4),
            "traffic": load_traffic(dom),
            "per_launch_ms": round(per_launch_ms, 4), "launches": int(g_n),
            "share_of_step": round(g_ms / max(total_ms, 1e-9), 4),
            "whole_step_frac": round(value / dist.world / 1e3 / FP64_PEAK_TFLOPS, 4),
        }
        out["kernel_shares"] = {k: round(v[0] / max(total_ms, 1e-9), 4) for k, v in prof.items()}
        if peaks:
            out["roofline"]["hbm_peak_gbs"] = peaks.get("hbm_gbs")
    out["clocks"] = clk.summary()

    # ---- the blocked forward sweep alongside, same N and L; Sigma_dot's
    # lower triangle is an N(0,1) draw like L_bar's, so tril(L_bar) serves as its input
    if args.fwd_steps > 0:
        def fstep():
            cd.chol_fwd(Ld, A, nb=nb)

        fms = timed_steps(fstep, restore, args.fwd_steps, 1, dist, stream)
        fw = dist.max(statistics.mean(fms))
        out["fwd"] = {"workload": f"chol_fwd fp64 single matrix N={n} (same L), nb={nb}",
                      "ms_per_step": round(fw, 3), "value": round(fwd_flops(n) / (fw * 1e-3) / 1e9, 2),
                      "unit": "GFLOP/s", "frac_of_fp64_peak": round(fwd_flops(n) / (fw * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                      "steps": args.fwd_steps}

    # ---- factorisation + forward mode fused in one sweep (Sigma = L L^T as input)
    if args.fused_steps > 0:
        S0 = (Ld @ Ld.transpose(0, 1)).transpose(0, 1).contiguous().transpose(0, 1)  # column-major Sigma
        Sw = torch.empty_like(S0).transpose(0, 1).contiguous().transpose(0, 1)

        def ustep():
            cd.chol_fwd_fused(Sw, A)

        def urestore():
            Sw.copy_(S0)
            A.copy_(A0)

        ums = timed_steps(ustep, urestore, args.fused_steps, 1, dist, stream)
        uw = dist.max(statistics.mean(ums))
        ufl = n ** 3 / 3 + fwd_flops(n)
        out["chol_fwd_fused"] = {"workload": f"cd_chol_fwd_fused fp64 N={n}: Sigma -> L and Sigma_dot -> L_dot in one sweep",
                                 "ms_per_step": round(uw, 3), "value": round(ufl / (uw * 1e-3) / 1e9, 2),
                                 "unit": "GFLOP/s (N^3/3 factorisation + fwd(N))", "steps": args.fused_steps}
        del S0, Sw

    # ---- e2e through the host-buffer C-ABI call
    if args.e2e_steps > 0:
        pin_L = torch.from_numpy(Lcm).pin_memory().transpose(0, 1)
        pin_A0 = torch.from_numpy(Acm).pin_memory()
        pin_A = pin_A0.clone().pin_memory().transpose(0, 1)
        del Ld, A0, A
        torch.cuda.empty_cache()

        def e2e_step():
            cd.chol_host("rev", pin_L, pin_A, nb=nb, device=dev)

        def e2e_restore():
            pin_A.transpose(0, 1).copy_(pin_A0)

        ems = timed_steps(e2e_step, e2e_restore, args.e2e_steps, 1, dist, stream)
        e_worst = dist.max(statistics.mean(ems))
        h2d, d2h = cd.host_bytes()  # counted by the library from the copies it issued
        out["e2e"] = {"value": round(fl * dist.world / (e_worst * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                      "ms_per_step": round(e_worst, 3),
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "path": "cd_chol_host: pinned host L, Abar; the lower part of each 128-column block "
                              "streams in on a copy stream as the left-looking sweep reaches it and streams "
                              "out when final (only the lower triangles cross the bus)"}
    # ---- CPU oracle sample
    if dist.world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_sample_rev(Lcm, Acm, n, args.cpu_seconds)
    return out


KERNEL_NAMES = {
    "symm": "k_symm_ll (left-looking trailing update Cbar -= (T+T^T) L, DMMA.8x8x4 via mma.sync m8n8k4 f64, "
            "TMA-fed, stream-K)",
    "gemm": "k_gemm_tma<double> (mma.sync m8n8k4 f64 -> DMMA.8x8x4)",
    "panel": "k_panel_rev (panel solve + tril correction, cooperative)",
}


def read_profile(Lib):
    import ctypes
    names = {0: "gemm", 1: "splitk_reduce", 2: "sweep", 3: "trinv", 4: "other", 5: "symm", 6: "panel"}
    res = {}
    for cls, name in names.items():
        ms, fl, cnt = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        Lib.cd_profile_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
        rc = Lib.cd_profile_read(cls, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(cnt))
        if rc != 0:
            raise RuntimeError("cd_profile_read failed")
        res[name] = (ms.value, fl.value, cnt.value)
    return res


def load_traffic(kind: str):
    """dram bytes per launch from the committed ncu --set full capture, if present."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kind)
    except Exception:
        return None


def cpu_sample_rev(Lcm, Acm, n, seconds):
    """Oracle (plain C, OpenMP over the columns of each rank-1 step) on the trailing
    columns of the same N=16384 sweep: columns n-1 .. n-a."""
    ncores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(ncores))
    import oracle
    A = Acm.copy()
    # calibrate on 128 columns, then size the sample for ~`seconds`
    a0 = 128
    t0 = time.perf_counter()
    oracle.chol_rev_colmajor_inplace(n, Lcm, A, j_lo=n - a0)
    dt0 = time.perf_counter() - t0
    f0 = sum(oracle.rev_column_flops(n, j) for j in range(n - a0, n))
    rate = f0 / max(dt0, 1e-6)
    a = a0
    while a < n and sum_cols(n, a * 2) / rate < seconds:
        a *= 2
    A = Acm.copy()
    t0 = time.perf_counter()
    oracle.chol_rev_colmajor_inplace(n, Lcm, A, j_lo=n - a)
    dt = time.perf_counter() - t0
    fl = sum_cols(n, a)
    return {"value": round(fl / dt / 1e9, 3), "unit": "GFLOP/s", "cores": ncores,
            "threads": int(os.environ.get("OMP_NUM_THREADS", ncores)), "kind": "oracle",
            "sample": f"trailing {a} columns (j = {n - 1}..{n - a}) of the N={n} reverse sweep, "
                      f"{fl / 1e9:.1f} GFLOP in {dt:.1f} s (oracle/oracle.c or_chol_rev_partial, OpenMP over columns)"}


def sum_cols(n, a):
    # exact flops of columns n-1..n-a (oracle.rev_column_flops summed in closed form)
    tot = 0
    for j in range(n - a, n):
        aa, b = n - 1 - j, j
        tot += (2 * aa + 1) + (aa + 1) + 2 * b * (aa + 1) + 2 * aa * b + 1
    return tot


def bench_batched(args, dist: Dist, n=32, total=65536, seed=0, gather=True):
    """configs[2]: 65536 independent fp64 N=32 matrices (seed + index), sharded by matrix."""
    import torch
    import paper_1602_07527_b200 as cd
    import synthetic

    from paper_1602_07527_b200.shard import gather_batches, shard_range
    P, r = dist.world, dist.rank
    lo, hi = shard_range(total, P, r)
    B = hi - lo
    L, Lb, _ = synthetic.draw_batch(n, B, seed=seed, start=lo)
    dev = dist.device
    Ld = colmajor_dev(L, dev)
    A0 = colmajor_dev(Lb, dev)
    A = A0.clone()
    stream = torch.cuda.current_stream(dev)

    def step():
        cd.chol_rev(Ld, A)

    def restore():
        A.copy_(A0)

    with ClockSampler(dev) as clk:
        ms = timed_steps(step, restore, args.steps_batched, args.warmup, dist, stream,
                         before_timed=cd.reset_launch_count)
    launches = cd.launch_count()
    worst = dist.max(statistics.mean(ms))
    mats = total / (worst * 1e-3)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6536.0)
    algo_bytes = 3 * n * (n + 1) // 2 * 8
    achieved_gbs = mats / P * algo_bytes / 1e9  # per GPU
    out = {"workload": f"configs[2]: chol_rev fp64, {total} x N={n} (seed+index), contiguous column-major, "
                       f"sharded by matrix over {P} GPU(s)",
           "value": round(mats, 1), "unit": "matrices/s", "ms_per_step": round(worst, 4),
           "gflops": round(mats * rev_flops(n) / 1e9, 1), "steps": args.steps_batched,
           "roofline": {"kernel": "k_rev_bulk32<4> (one warp per matrix, N_b=8 DMMA tiles, cp.async-staged conflict-free smem columns)", "bound": "hbm", "achieved": round(achieved_gbs, 1),
                        "peak": hbm, "unit": "GB/s", "frac": round(achieved_gbs / hbm, 4),
                        "algorithmic_bytes_per_matrix": algo_bytes,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs", "traffic": load_traffic("bulk32")},
           "gpu_launches": int(launches), "clocks": clk.summary()}
    # the symbolic route (Eq. 10 on the whole matrix, north star (d)) on the same inputs, for
    # the route choice "by measurement" (AUTO = algorithmic)
    sms = timed_steps(lambda: cd.chol_rev(Ld, A, route="symbolic"), restore, 5, 2, dist, stream)
    out["symbolic_route"] = {"ms_per_step": round(dist.max(statistics.mean(sms)), 4),
                             "matrices_per_s": round(total / (dist.max(statistics.mean(sms)) * 1e-3), 1),
                             "kernel": "k_symbolic_cta (one CTA per matrix, Eq. 10 on 8x8 DMMA tiles)"}
    if gather and P > 1:
        # NCCL used only to gather the sharded results (north star), timed separately
        torch.cuda.synchronize()
        dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gathered = gather_batches(A, total)
        b.record(stream)
        torch.cuda.synchronize()
        g = dist.max(a.elapsed_time(b))
        del gathered
        out["gather"] = {"ms": round(g, 3), "bytes": total * n * n * 8,
                         "GBps": round(total * n * n * 8 / (g * 1e-3) / 1e9, 1),
                         "collective": "all_gather_into_tensor (paper_1602_07527_b200/shard.py)"}
    if dist.world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_sample_batched(L, Lb, n)
    return out


def cpu_sample_batched(L, Lb, n, sample=16384):
    ncores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(ncores))
    import oracle
    import synthetic
    s = min(sample, L.shape[0])
    Lc = synthetic.to_colmajor(L[:s])
    Ac = synthetic.to_colmajor(Lb[:s])
    t0 = time.perf_counter()
    oracle.chol_rev_batched_colmajor(n, s, Lc, Ac)
    dt = time.perf_counter() - t0
    return {"value": round(s / dt, 1), "unit": "matrices/s", "cores": ncores,
            "threads": int(os.environ.get("OMP_NUM_THREADS", ncores)), "kind": "oracle",
            "sample": f"first {s} of the 65536 N={n} matrices, oracle/oracle.c or_chol_rev_batched (OpenMP over matrices)"}


def bench_small_configs(args, dist: Dist):
    """configs[0] (N=64 rev latency), configs[1] (N=1024 rev + fwd) and configs[3]
    (1024 x N=512 fp32 rev + fwd, sharded by matrix), same timing rules."""
    import torch
    import paper_1602_07527_b200 as cd
    import synthetic

    dev = dist.device
    stream = torch.cuda.current_stream(dev)
    out = {}
    # configs[0]: single fp64 N=64 reverse (latency)
    L, Lb, _ = synthetic.draw(64, 0)
    Ld, A0 = colmajor_dev(L, dev), colmajor_dev(Lb, dev)
    A = A0.clone()
    ms = timed_steps(lambda: cd.chol_rev(Ld, A), lambda: A.copy_(A0), 50, args.warmup, dist, stream)
    t = dist.max(statistics.median(ms))
    # the same call captured once in a CUDA graph and replayed (host launch overhead removed)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cd.chol_rev(Ld, A)
    gms = timed_steps(g.replay, lambda: A.copy_(A0), 50, args.warmup, dist, stream)
    tg = dist.max(statistics.median(gms))
    out["n64_rev"] = {"workload": "configs[0]: chol_rev fp64 N=64, seed 0", "us_per_call": round(t * 1e3, 2),
                      "gflops": round(rev_flops(64) / (t * 1e-3) / 1e9, 2),
                      "us_per_call_cuda_graph": round(tg * 1e3, 2)}
    # configs[1]: N=1024 reverse and forward
    L, Lb, Sd = synthetic.draw(1024, 0, sdot=True)
    Ld, A0, F0 = colmajor_dev(L, dev), colmajor_dev(Lb, dev), colmajor_dev(np.tril(Sd), dev)
    A, F = A0.clone(), F0.clone()
    tr = dist.max(statistics.median(timed_steps(lambda: cd.chol_rev(Ld, A), lambda: A.copy_(A0), 10, args.warmup,
                                                dist, stream)))
    tf = dist.max(statistics.median(timed_steps(lambda: cd.chol_fwd(Ld, F), lambda: F.copy_(F0), 10, args.warmup,
                                                dist, stream)))
    ts = dist.max(statistics.median(timed_steps(lambda: cd.chol_rev(Ld, A, route="symbolic"), lambda: A.copy_(A0),
                                                5, args.warmup, dist, stream)))
    out["n1024"] = {"workload": "configs[1]: fp64 N=1024, seed 0", "rev_ms": round(tr, 3), "fwd_ms": round(tf, 3),
                    "rev_symbolic_route_ms": round(ts, 3),
                    "rev_gflops": round(rev_flops(1024) / (tr * 1e-3) / 1e9, 1),
                    "fwd_gflops": round(fwd_flops(1024) / (tf * 1e-3) / 1e9, 1)}
    # configs[3]: 1024 x N=512 fp32, reverse + forward per step, sharded by matrix
    n, total = 512, 1024
    from paper_1602_07527_b200.shard import shard_range
    P, r = dist.world, dist.rank
    lo, hi = shard_range(total, P, r)
    L, Lb, Sd = synthetic.draw_batch(n, hi - lo, seed=0, sdot=True, start=lo)
    Ld = colmajor_dev(L, dev, torch.float32)
    A0 = colmajor_dev(Lb, dev, torch.float32)
    F0 = colmajor_dev(np.tril(Sd), dev, torch.float32)
    del L, Lb, Sd
    A, F = A0.clone(), F0.clone()

    def step():  # both sweeps of the same factors; chol_rev_fwd runs them on two streams
        cd.chol_rev_fwd(Ld, A, F)

    def restore():
        A.copy_(A0)
        F.copy_(F0)

    t = dist.max(statistics.median(timed_steps(step, restore, 5, args.warmup, dist, stream)))
    fl = (rev_flops(n) + fwd_flops(n)) * total
    out["batched_f32_n512"] = {
        "workload": f"configs[3]: fp32 rev + fwd, {total} x N={n}, sharded by matrix over {P} GPU(s); "
                    "cd.chol_rev_fwd (the two independent sweeps on two streams)",
        "ms_per_step": round(t, 3), "matrices_per_s": round(total / (t * 1e-3), 1),
        "gflops": round(fl / (t * 1e-3) / 1e9, 1),
        # engines: tcgen05 kind::tf32 GEMMs + fp64-DMMA on-chip diagonal blocks.  Roofline =
        # max(bytes / HBM, flops / tf32 peak); the HBM term wins: 5 T(512) fp32 triangles per
        # matrix moved once (L shared by rev and fwd), 0.41 ms for the batch
        "roofline": {"bound": "hbm", "unit": "GB/s",
                     "algorithmic_bytes_per_matrix": 5 * (n * (n + 1) // 2) * 4,
                     "achieved": round(5 * (n * (n + 1) // 2) * 4 * total / P / (t * 1e-3) / 1e9, 1),
                     "peak": measured_peaks().get("hbm_gbs", 6536.0),
                     "frac": round(5 * (n * (n + 1) // 2) * 4 * total / P / (t * 1e-3) / 1e9
                                   / measured_peaks().get("hbm_gbs", 6536.0), 4),
                     "compute_floor_ms": round(fl / P / TF32_PEAK_TFLOPS / 1e9, 3),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs; tf32 peak = measured bf16 dense x 1/2 "
                                    "(profiling guide's nominal ratio)"}}
    return out


# ----------------------------------------------------------------------------- reference arm
def reference_arm(args):
    """The CPU oracle as the reference implementation (this tier has no reference code):
    same workload, metric and unit; each step = the trailing `a` columns of the N=16384
    reverse sweep, restored from a pristine copy between steps (untimed)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    ncores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(ncores))
    import oracle
    import synthetic
    n = args.n
    L, Lb, _ = synthetic.draw(n, args.seed)
    Lcm, A0 = synthetic.to_colmajor(L), synthetic.to_colmajor(Lb)
    del L, Lb
    a = args.ref_cols
    A = A0.copy()
    for _ in range(max(0, args.warmup)):
        np.copyto(A, A0)
        oracle.chol_rev_colmajor_inplace(n, Lcm, A, j_lo=n - a)
        break  # one warm-up sample is enough for a CPU loop
    times = []
    for _ in range(args.steps):
        np.copyto(A, A0)
        t0 = time.perf_counter()
        oracle.chol_rev_colmajor_inplace(n, Lcm, A, j_lo=n - a)
        times.append(time.perf_counter() - t0)
    fl = sum_cols(n, a)
    ms = statistics.mean(times) * 1e3
    value = fl / (ms * 1e-3) / 1e9
    sample = (f"trailing {a} columns (j = {n - 1}..{n - a}) of the N={n} reverse sweep per step, "
              f"{fl / 1e9:.2f} GFLOP per step")
    return {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded PCG64 generator, synthetic/)",
            "config": {"workload": f"configs[4]: chol_rev fp64 single matrix N={n}, seed {args.seed}",
                       "n": n, "batch": 1, "parallelism": "host cores (oracle)"},
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": ncores,
                             "threads": int(os.environ.get("OMP_NUM_THREADS", ncores)), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--steps-batched", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--fwd-steps", type=int, default=2, help="timed chol_fwd steps at the same N (0 = skip)")
    ap.add_argument("--fused-steps", type=int, default=2, help="timed chol_fwd_fused steps at the same N (0 = skip)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-cols", type=int, default=1024)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-batched", action="store_true")
    ap.add_argument("--no-aux", action="store_true", help="skip configs[0], [1], [3] sub-measurements")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3

    if args.impl == "reference":
        res = reference_arm(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA GPU (the product path has no CPU fallback)")
    dist = Dist(args.gpus)
    torch.cuda.set_device(dist.device)
    import paper_1602_07527_b200 as cd
    cd.lib()  # fail loudly if the extension is missing
    res = bench_single_rev(args, dist)
    if not args.no_batched:
        res["batched"] = bench_batched(args, dist)
    if not args.no_aux:
        res["other_configs"] = bench_small_configs(args, dist)
    if dist.rank == 0:
        print(json.dumps(res), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
