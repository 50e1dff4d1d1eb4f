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

Multi-GPU: ``python bench.py --gpus N`` (N > 1) started without a torchrun environment
re-executes itself under ``torch.distributed.run`` with N ranks (one per GPU, NCCL,
rendezvous on 127.0.0.1), and every rank checks WORLD_SIZE == --gpus.  The batched
configs shard by matrix; their compute is timed as the max over ranks and the NCCL
gather of the results is timed separately ("gather").  NCCL_DEBUG=INFO is set for
the ranks, its output written to nccl_logs/ (the JSON line stays the only stdout).
``--dry-run`` runs the same rank/shard/gather plumbing on the CPU with gloo (no GPU,
no kernels, no timing numbers): ``python bench.py --gpus 2 --dry-run``.
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


def _generator_version():
    sys.path.insert(0, ROOT)
    import synthetic
    return synthetic.GENERATOR_VERSION


GEN = _generator_version()


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
    """One process per GPU (torchrun environment).  NCCL on the GPUs; gloo on the CPU for
    --dry-run.  Fails loudly when the launched world size is not the requested --gpus."""

    def __init__(self, want: int, dry_run: bool = False):
        import torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.want = want
        self.dry = dry_run
        if self.world != want:
            raise SystemExit(f"bench.py: --gpus {want} but the launch has WORLD_SIZE={self.world} "
                             "(start it as `python bench.py --gpus N`, or under torchrun with N ranks)")
        self.pg = None
        self.device = torch.device("cpu") if dry_run else torch.device("cuda", self.local)
        if self.world > 1:
            import torch.distributed as dist
            if dry_run:
                dist.init_process_group("gloo")
            else:
                nccl_env()
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist
        self.backend = (self.pg.get_backend() if self.pg else None)

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def _reduce(self, x: float, op) -> float:
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.MAX) if self.pg else x

    def sum(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.SUM) if self.pg else x

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


NCCL_LOG_DIR = os.path.join(ROOT, "nccl_logs")


def nccl_env():
    """NCCL_DEBUG=INFO for the ranks (communicator setup and ranks visible), written to
    nccl_logs/ so that stdout carries only the JSON line."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    if "NCCL_DEBUG_FILE" not in os.environ:
        os.makedirs(NCCL_LOG_DIR, exist_ok=True)
        os.environ["NCCL_DEBUG_FILE"] = os.path.join(NCCL_LOG_DIR, "nccl.%h.%p.log")


def relaunch_under_torchrun(nranks: int) -> int:
    """`python bench.py --gpus N` without a torchrun environment: start N ranks of this very
    command under torch.distributed.run (127.0.0.1 rendezvous) and return their exit code."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    nccl_env()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ))


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
    L, Lb, Sd = synthetic.draw(n, args.seed, sdot=args.fwd_steps > 0 or args.fused_steps > 0)
    Lcm = synthetic.to_colmajor(L)
    Acm = synthetic.to_colmajor(Lb)
    Fcm = synthetic.to_colmajor(np.tril(Sd)) if Sd is not None else None
    del L, Lb, Sd
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
        "generator": GEN,
    }
    if dist.world > 1:
        out["nccl"] = {"backend": dist.backend, "world_size": dist.world,
                       "debug": os.environ.get("NCCL_DEBUG"), "debug_file": os.environ.get("NCCL_DEBUG_FILE")}
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
                           "profiles/r01_microbench_fp64.txt; with its clock record, sustained 1965 MHz, in "
                           "profiles/r02_microbench_fp64.txt); MEASURED_PEAKS.json has no fp64 entry",
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

    # ---- the blocked forward sweep alongside, same N and L, the generator's
    # Sigma_dot (its 4th draw, synthetic/)
    if args.fwd_steps > 0:
        F0 = torch.from_numpy(Fcm).to(dev).transpose(0, 1)

        def fstep():
            cd.chol_fwd(Ld, A, nb=nb)

        def frestore():
            A.copy_(F0)

        fms = timed_steps(fstep, frestore, args.fwd_steps, 1, dist, stream)
        fw = dist.max(statistics.mean(fms))
        out["fwd"] = {"workload": f"chol_fwd fp64 single matrix N={n} (same L), nb={nb}",
                      "ms_per_step": round(fw, 3), "value": round(fwd_flops(n) / (fw * 1e-3) / 1e9, 2),
                      "unit": "GFLOP/s", "frac_of_fp64_peak": round(fwd_flops(n) / (fw * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                      "steps": args.fwd_steps}
        del F0

    # ---- factorisation + forward mode fused in one sweep (Sigma = L L^T as input)
    if args.fused_steps > 0:
        S0 = (Ld @ Ld.transpose(0, 1)).transpose(0, 1).contiguous().transpose(0, 1)  # column-major Sigma
        Sw = torch.empty_like(S0).transpose(0, 1).contiguous().transpose(0, 1)

        def ustep():
            cd.chol_fwd_fused(Sw, A)

        F0 = torch.from_numpy(Fcm).to(dev).transpose(0, 1)

        def urestore():
            Sw.copy_(S0)
            A.copy_(F0)

        ums = timed_steps(ustep, urestore, args.fused_steps, 1, dist, stream)
        uw = dist.max(statistics.mean(ums))
        ufl = n ** 3 / 3 + fwd_flops(n)
        out["chol_fwd_fused"] = {"workload": f"cd_chol_fwd_fused fp64 N={n}: Sigma -> L and Sigma_dot -> L_dot in one sweep",
                                 "ms_per_step": round(uw, 3), "value": round(ufl / (uw * 1e-3) / 1e9, 2),
                                 "unit": "GFLOP/s (N^3/3 factorisation + fwd(N))", "steps": args.fused_steps}
        del S0, Sw, F0

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
           "gpu_launches": int(launches), "clocks": clk.summary(), "generator": GEN,
           "l2": "inputs larger than L2 (512 MiB per array)"}
    # the symbolic route (Eq. 10 on the whole matrix, north star (d)) on the same inputs, for
    # the route choice "by measurement" (AUTO = algorithmic)
    sms = timed_steps(lambda: cd.chol_rev(Ld, A, route="symbolic"), restore, 5, 2, dist, stream)
    out["symbolic_route"] = {"ms_per_step": round(dist.max(statistics.mean(sms)), 4),
                             "matrices_per_s": round(total / (dist.max(statistics.mean(sms)) * 1e-3), 1),
                             "kernel": "k_symbolic_cta (one CTA per matrix, Eq. 10 on 8x8 DMMA tiles)"}
    if gather and P > 1:
        out["gather"] = timed_gather(dist, stream, [A], total)
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


class L2Flush:
    """Writes a buffer larger than the 126 MB L2 (outside the timed events) so that every
    timed iteration of a small configuration starts from a cold L2 (timing rules)."""

    def __init__(self, device, nbytes=256 << 20):
        import torch
        self.buf = torch.empty(nbytes // 4, dtype=torch.float32, device=device)
        self.k = 0

    def __call__(self):
        self.k += 1
        self.buf.fill_(float(self.k))


def graph_device_us(call, flush, restore, stream, dist, pairs=20, reps=10):
    """Device microseconds per call: a CUDA graph of `pairs` (flush, call) pairs against a graph
    of the flushes alone, both replayed `reps` times between CUDA events (median each)."""
    import torch
    restore()
    torch.cuda.synchronize()
    g_both, g_flush = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_both):
        for _ in range(pairs):
            flush()
            call()
    with torch.cuda.graph(g_flush):
        for _ in range(pairs):
            flush()

    def med(g):
        ts = []
        for _ in range(reps + 2):
            restore()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts[2:])

    return dist.max(1e3 * (med(g_both) - med(g_flush)) / pairs)


def cpu_oracle_single(kind: str, L, X, reps_seconds=2.0):
    """Oracle (plain C, ONE thread) on one matrix, repeated for about `reps_seconds`:
    kind 'rev' or 'fwd'.  Returns seconds per call."""
    import oracle
    n = L.shape[0]
    Lc = synthetic_cm(L)
    X0 = synthetic_cm(X)
    f = oracle.chol_rev_colmajor_inplace if kind == "rev" else oracle.chol_fwd_serial_colmajor_inplace
    oracle.set_threads(1)
    try:
        reps, t_tot = 0, 0.0
        while t_tot < reps_seconds or reps < 3:
            A = X0.copy()
            t0 = time.perf_counter()
            f(n, Lc, A)
            t_tot += time.perf_counter() - t0
            reps += 1
    finally:
        oracle.set_threads(0)
    return t_tot / reps, reps


def synthetic_cm(m):
    import synthetic
    return synthetic.to_colmajor(m).copy()


def bench_small_configs(args, dist: Dist):
    """configs[0] (N=64 rev latency), configs[1] (N=1024 rev + fwd) and configs[3]
    (1024 x N=512 fp32 rev + fwd, sharded by matrix), same timing rules; each with the
    oracle timed beside it on the host cores (rank 0 at N=1)."""
    import torch
    import paper_1602_07527_b200 as cd
    import synthetic

    dev = dist.device
    stream = torch.cuda.current_stream(dev)
    flush = L2Flush(dev)
    cpu = dist.world == 1 and not args.no_cpu
    out = {}
    # configs[0]: single fp64 N=64 reverse (latency); L2 flushed before every timed call
    L, Lb, _ = synthetic.draw(64, 0)
    Ld, A0 = colmajor_dev(L, dev), colmajor_dev(Lb, dev)
    A = A0.clone()

    def r0():
        A.copy_(A0)
        flush()

    ms = timed_steps(lambda: cd.chol_rev(Ld, A), r0, 50, args.warmup, dist, stream)
    t = dist.max(statistics.median(ms))
    # the same call captured once in a CUDA graph and replayed (host launch overhead removed)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cd.chol_rev(Ld, A)
    gms = timed_steps(g.replay, r0, 50, args.warmup, dist, stream)
    tg = dist.max(statistics.median(gms))
    # device time per call: one CUDA graph holding 20 (L2 flush, call) pairs, minus a graph of the 20
    # flushes alone (no host submission gap between the events; the calls still start cold)
    td = graph_device_us(lambda: cd.chol_rev(Ld, A), lambda: flush(), r0, stream, dist)
    out["n64_rev"] = {"workload": "configs[0]: chol_rev fp64 N=64, seed 0", "us_per_call": round(t * 1e3, 2),
                      "gflops": round(rev_flops(64) / (t * 1e-3) / 1e9, 2),
                      "us_per_call_cuda_graph": round(tg * 1e3, 2),
                      "us_per_call_device": round(td, 2),
                      "device_method": "20 (L2 flush, call) pairs captured in one CUDA graph, minus the same "
                                       "graph of flushes alone, / 20 (median of 10 replays each)",
                      "l2": "flushed before every timed call", "generator": GEN}
    if cpu:
        sec, reps = cpu_oracle_single("rev", L, Lb)
        out["n64_rev"]["cpu_baseline"] = {"value": round(sec * 1e6, 2), "unit": "us per call", "cores": 1,
                                          "threads": 1, "kind": "oracle",
                                          "sample": f"the whole N=64 reverse sweep, {reps} calls, "
                                                    "oracle/oracle.c or_chol_rev_partial (single thread)"}
    # configs[1]: N=1024 reverse and forward
    L, Lb, Sd = synthetic.draw(1024, 0, sdot=True)
    Ld, A0, F0 = colmajor_dev(L, dev), colmajor_dev(Lb, dev), colmajor_dev(np.tril(Sd), dev)
    A, F = A0.clone(), F0.clone()

    def ra():
        A.copy_(A0)
        flush()

    def rf():
        F.copy_(F0)
        flush()

    tr = dist.max(statistics.median(timed_steps(lambda: cd.chol_rev(Ld, A), ra, 10, args.warmup, dist, stream)))
    tf = dist.max(statistics.median(timed_steps(lambda: cd.chol_fwd(Ld, F), rf, 10, args.warmup, dist, stream)))
    ts = dist.max(statistics.median(timed_steps(lambda: cd.chol_rev(Ld, A, route="symbolic"), ra,
                                                5, args.warmup, dist, stream)))
    tdr = graph_device_us(lambda: cd.chol_rev(Ld, A), lambda: flush(), ra, stream, dist, pairs=10) * 1e-3
    tdf = graph_device_us(lambda: cd.chol_fwd(Ld, F), lambda: flush(), rf, stream, dist, pairs=10) * 1e-3
    out["n1024"] = {"workload": "configs[1]: fp64 N=1024, seed 0", "rev_ms": round(tr, 3), "fwd_ms": round(tf, 3),
                    "rev_ms_device": round(tdr, 3), "fwd_ms_device": round(tdf, 3),
                    "device_method": "10 (L2 flush, call) pairs in one CUDA graph minus the flushes alone, / 10",
                    "rev_symbolic_route_ms": round(ts, 3),
                    "rev_gflops": round(rev_flops(1024) / (tr * 1e-3) / 1e9, 1),
                    "fwd_gflops": round(fwd_flops(1024) / (tf * 1e-3) / 1e9, 1),
                    "rev_frac_of_fp64_peak": round(rev_flops(1024) / (tr * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                    "fwd_frac_of_fp64_peak": round(fwd_flops(1024) / (tf * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                    "l2": "flushed before every timed call", "generator": GEN}
    if cpu:
        sr, nr = cpu_oracle_single("rev", L, Lb)
        sf, nf = cpu_oracle_single("fwd", L, np.tril(Sd))
        out["n1024"]["cpu_baseline"] = {
            "value": round((rev_flops(1024) + fwd_flops(1024)) / (sr + sf) / 1e9, 3), "unit": "GFLOP/s",
            "rev_ms": round(sr * 1e3, 1), "fwd_ms": round(sf * 1e3, 1), "cores": 1, "threads": 1, "kind": "oracle",
            "sample": f"the whole N=1024 reverse ({nr} calls) and forward ({nf} calls) sweeps, oracle/oracle.c "
                      "(single thread)"}
    # configs[3]: 1024 x N=512 fp32, reverse + forward per step, sharded by matrix
    n, total = 512, 1024
    from paper_1602_07527_b200.shard import gather_batches, shard_range
    P, r = dist.world, dist.rank
    lo, hi = shard_range(total, P, r)
    L, Lb, Sd = synthetic.draw_batch(n, hi - lo, seed=0, sdot=True, start=lo)
    Ld = colmajor_dev(L, dev, torch.float32)
    A0 = colmajor_dev(Lb, dev, torch.float32)
    F0 = colmajor_dev(np.tril(Sd), dev, torch.float32)
    A, F = A0.clone(), F0.clone()

    def step():  # both sweeps of the same factors in one library call
        cd.chol_rev_fwd(Ld, A, F)

    def restore():
        A.copy_(A0)
        F.copy_(F0)

    with ClockSampler(dev) as clk:
        ms3 = timed_steps(step, restore, args.steps_c3, args.warmup, dist, stream,
                          before_timed=cd.reset_launch_count)
    launches = cd.launch_count()
    t = dist.max(statistics.median(ms3))
    fl = (rev_flops(n) + fwd_flops(n)) * total
    algo = 5 * (n * (n + 1) // 2) * 4
    hbm = measured_peaks().get("hbm_gbs", 6536.0)
    achieved = algo * total / P / (t * 1e-3) / 1e9  # per GPU
    out["batched_f32_n512"] = {
        "workload": f"configs[3]: fp32 rev + fwd, {total} x N={n}, sharded by matrix over {P} GPU(s); "
                    "cd.chol_rev_fwd (cd_chol_rev_fwd_strided_batched)",
        "ms_per_step": round(t, 3), "matrices_per_s": round(total / (t * 1e-3), 1),
        "gflops": round(fl / (t * 1e-3) / 1e9, 1), "steps": args.steps_c3,
        "step_ms": {"min": round(min(ms3), 3), "median": round(statistics.median(ms3), 3),
                    "max": round(max(ms3), 3)},
        "gpu_launches": int(launches) // max(1, args.steps_c3), "clocks": clk.summary(), "generator": GEN,
        "l2": "inputs larger than L2 (1 GiB per array)",
        # roofline = max(bytes / HBM, flops / tf32 peak); the HBM term wins: 5 T(512) fp32
        # triangles per matrix moved once (L shared by rev and fwd), 0.41 ms for the batch
        "roofline": {"bound": "hbm", "unit": "GB/s", "algorithmic_bytes_per_matrix": algo,
                     "achieved": round(achieved, 1), "peak": hbm, "frac": round(achieved / hbm, 4),
                     "compute_floor_ms": round(fl / P / TF32_PEAK_TFLOPS / 1e9, 3),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs; tf32 peak = measured bf16 dense x 1/2 "
                                    "(profiling guide's nominal ratio)"}}
    if P > 1:
        out["batched_f32_n512"]["gather"] = timed_gather(dist, stream, [A, F], total)
    if cpu:
        out["batched_f32_n512"]["cpu_baseline"] = cpu_sample_c3(L, Lb, Sd, n)
    return out


def timed_gather(dist: Dist, stream, shards, total: int):
    """NCCL all_gather of the per-rank result shards (north star: NCCL only to gather),
    timed on the device as the max over ranks, outside the compute timing."""
    import torch
    from paper_1602_07527_b200.shard import gather_batches
    torch.cuda.synchronize()
    dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    outs = [gather_batches(x, total) for x in shards]
    b.record(stream)
    torch.cuda.synchronize()
    g = dist.max(a.elapsed_time(b))
    nbytes = sum(o.numel() * o.element_size() for o in outs)
    del outs
    return {"ms": round(g, 3), "bytes": nbytes, "GBps": round(nbytes / (g * 1e-3) / 1e9, 1),
            "collective": "all_gather_into_tensor over NCCL (paper_1602_07527_b200/shard.py)",
            "timed": "device events around the gathers, max over ranks, separate from compute"}


def cpu_sample_c3(L, Lb, Sd, n, sample=48):
    """configs[3] oracle beside the GPU: the first `sample` matrices of the batch, reverse and
    forward, fp64 on the fp32-rounded inputs, OpenMP over matrices on all cores."""
    ncores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(ncores))
    import oracle
    import synthetic
    s = min(sample, L.shape[0])
    r32 = lambda x: x[:s].astype(np.float32).astype(np.float64)  # noqa: E731
    Lc = synthetic.to_colmajor(r32(L))
    Ac = synthetic.to_colmajor(r32(Lb))
    Fc = synthetic.to_colmajor(np.tril(r32(Sd)))
    t0 = time.perf_counter()
    oracle.chol_rev_batched_colmajor(n, s, Lc, Ac)
    oracle.chol_fwd_cols_batched_colmajor(n, s, Lc, Fc)
    dt = time.perf_counter() - t0
    return {"value": round(s / dt, 2), "unit": "matrices/s (rev + fwd)", "cores": ncores,
            "threads": int(os.environ.get("OMP_NUM_THREADS", ncores)), "kind": "oracle",
            "gflops": round(s * (rev_flops(n) + fwd_flops(n)) / dt / 1e9, 3),
            "sample": f"first {s} of the 1024 N={n} matrices, reverse + forward in fp64 on the fp32-rounded "
                      "inputs, oracle/oracle.c (OpenMP over matrices)"}


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
    ap.add_argument("--steps-c3", type=int, default=10, help="timed steps of configs[3] (1024 x N=512 fp32)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: exercise the rank / shard / gather plumbing with gloo (no kernels, no timings)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours" and not args.dry_run:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this command as N torchrun ranks
        raise SystemExit(relaunch_under_torchrun(args.gpus))

    if args.impl == "reference":
        res = reference_arm(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    if args.dry_run:
        dist = Dist(args.gpus, dry_run=True)
        res = dry_run(args, dist)
        if dist.rank == 0:
            print(json.dumps(res), flush=True)
        dist.close()
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


def dry_run(args, dist: Dist):
    """The multi-rank plumbing of the batched configs without a GPU: every rank takes its
    shard_range of configs[2] / configs[3] (reduced totals), draws its own inputs (seed + index),
    passes them through unchanged in place of the kernel, and the shards are all-gathered over
    gloo (the same gather_batches the GPU run uses over NCCL); rank 0 checks the gathered batch
    equals a single-process draw (partition order).  No kernel runs and nothing is timed as a
    throughput: "value" is null."""
    import torch
    import synthetic
    from paper_1602_07527_b200.shard import gather_batches, shard_range
    P, r = dist.world, dist.rank
    out = {"metric": METRIC, "value": None, "unit": "GFLOP/s", "n_gpus": P, "dry_run": True,
           "backend": dist.backend, "steps": 0, "warmup": 0, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64 generator, synthetic/)",
           "generator": GEN, "config": {"workload": "dry run: shard + gather plumbing of configs[2] / configs[3]",
                                        "parallelism": f"by matrix over {P} ranks"}}
    for name, n, total in (("batched", 32, 96), ("batched_f32_n512", 16, 24)):
        lo, hi = shard_range(total, P, r)
        _, Lb, _ = synthetic.draw_batch(n, hi - lo, seed=0, start=lo)
        local = torch.from_numpy(synthetic.to_colmajor(Lb)).transpose(-1, -2)  # column-major per matrix
        dist.barrier()
        t0 = time.perf_counter()
        g = gather_batches(local, total)
        dt = time.perf_counter() - t0
        gmax = dist.max(dt)
        ok = True
        if r == 0:
            _, ref, _ = synthetic.draw_batch(n, total, seed=0)
            ok = bool(np.array_equal(g.numpy(), ref))
        out[name] = {"shards": [list(shard_range(total, P, q)) for q in range(P)], "total": total, "n": n,
                     "gather": {"ms": round(gmax * 1e3, 3), "bytes": int(g.numel() * g.element_size()),
                                "collective": f"all_gather over {dist.backend} (paper_1602_07527_b200/shard.py)",
                                "order_ok": ok}}
    return out


if __name__ == "__main__":
    main()
