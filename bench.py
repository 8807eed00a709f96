"""Benchmark: compressed-NeNMF outer iterations/s on BASELINE config 2 (B200).

One step = the hot path over one synthetic input: the randomized-subspace-
iteration sketch (``subspace_iteration_pair``, q=4, p'=30) charged to the run
as the reference CLI does (cli.py:159-168), then ``factorize_compressed`` for
100 outer iterations with inner Max_iter=500 (the reference default) in FP32
on n = m = 10^4, p = 20 (BASELINE.json configs[1]).  metric value =
outer iterations completed / wall time of the step on the device.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (the reference algorithm restated in
NumPy, oracle/nenmf_oracle.py; the reference is pure Python, so there is
nothing to compile into oracle/_ref) on the host cores, on a bounded sample
of the same workload.  N > 1 (torchrun): independent replicas (weak scaling),
rank 0 prints; the path has no cross-GPU exchange in this configuration.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "compressed-NeNMF outer iters/s (cfg2 n=m=1e4 p=20 p'=30 q=4, fp32, 100 outer, inner<=500, sketch charged)"
UNIT = "outer_iter/s"
CFG = 2
OUTER = 100


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg5"],
                    help="cfg2: the headline (1 problem per GPU, replicas for N > 1); "
                         "cfg5: 100k x 100k fp32 generated on device, X row-sharded over the N GPUs")
    ap.add_argument("--outer", type=int, default=None, help="override the outer-iteration count (probes only)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi needs a moment before its first line: wait for it so the
        # periodic samples fall inside the timed region, then drop it
        t0 = time.time()
        while not self.rows and time.time() - t0 < 3.0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.rows.clear()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 4:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.rows:
            # a timed region shorter than the sampling period: one sample at its end
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
                for line in out.stdout.splitlines():
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) == 4:
                        self.rows.append(parts)
            except (OSError, subprocess.TimeoutExpired):
                pass
        sm, mx, reasons = [], None, set()
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
        for s, m, _pw, act in self.rows:
            try:
                sm.append(float(s))
                mx = float(m)
                bits = int(act, 16)
            except ValueError:
                continue
            for b, nm in names.items():
                if bits & b and b != 0x1:
                    reasons.add(nm)
        busy = [v for v in sm if mx is None or v > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline
def cpu_sample(w, outer_sample: int = 1):
    """Oracle (reference algorithm, NumPy/OpenBLAS, all host threads) on a
    bounded sample of the same workload: the full sketch + compression and
    ``outer_sample`` outer iterations; extrapolated to OUTER iterations."""
    sys.path.insert(0, str(REPO / "oracle"))
    import nenmf_oracle as orc

    t0 = time.perf_counter()
    L, R = orc.rsi(w.X, w.nu, w.q, w.sketch_seed)
    t_sketch = time.perf_counter() - t0
    t1 = time.perf_counter()
    res = orc.nenmf(w.X, w.G0, w.F0, L=L, R=R, max_outer=outer_sample, max_iter=w.inner,
                    trace_every=outer_sample + 1)
    t_loop = time.perf_counter() - t1
    # the loop includes compress + 2 emits; charge them once like the GPU step does
    per_outer = t_loop / outer_sample
    total = t_sketch + OUTER * per_outer
    return {"value": OUTER / total, "t_sketch_s": t_sketch, "t_outer_s": per_outer,
            "inner_iters": [[g.iterations, f.iterations] for g, f in res.inner]}


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# -------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1812_04315_b200 import workloads

    w = workloads.make_workload(CFG, dtype=args.dtype)
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(w, outer_sample=1)
        if i >= args.warmup:
            vals.append(r)
    value = statistics.median(v["value"] for v in vals)
    ms = 1e3 * OUTER / value
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE cfg2 generator, seed 1234)",
        "impl": "reference",
        "config": {"workload": "cfg2", "n": w.n, "m": w.m, "p": w.p, "p_prime": w.nu, "q": w.q,
                   "outer": OUTER, "inner_max_iter": w.inner, "parallelism": "host cores (OpenBLAS threads)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port",
                         "sample": "per step: full RSI sketch+compress on cfg2 X and 1 outer iteration "
                                   "(inner<=500), extrapolated to 100 outer; reference algorithm restated in "
                                   "NumPy (oracle/nenmf_oracle.py), float64 as the reference"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_detail": vals[-1],
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1812_04315_b200 as nm
    from paper_1812_04315_b200 import _lib, _ops, workloads
    from paper_1812_04315_b200.compression import rsi_device

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    lib = _lib.load_library()
    w = workloads.make_workload(CFG, dtype=args.dtype)
    tdt = _lib.torch_dtype(args.dtype)
    Xd = torch.from_numpy(w.X.astype(np.float32 if args.dtype == "fp32" else np.float64)).to("cuda")
    G0d = torch.from_numpy(w.G0.astype(Xd.numpy().dtype if False else (np.float32 if args.dtype == "fp32" else np.float64))).to("cuda")
    F0d = torch.from_numpy(w.F0.astype(np.float32 if args.dtype == "fp32" else np.float64)).to("cuda")
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                         max_outer_iterations=OUTER, trace_every=OUTER)
    stream = torch.cuda.current_stream()

    def step_device():
        sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
        init = nm.FactorPair(G=G0d, F=F0d, p=w.p)
        return nm.factorize_compressed(Xd, sk, init, cfg, return_device=True)

    # pinned host copies for the end-to-end leg
    Xh = torch.from_numpy(w.X.astype(np.float32 if args.dtype == "fp32" else np.float64)).pin_memory()
    G0h = torch.from_numpy(w.G0.astype(np.float32 if args.dtype == "fp32" else np.float64)).pin_memory()
    F0h = torch.from_numpy(w.F0.astype(np.float32 if args.dtype == "fp32" else np.float64)).pin_memory()
    h2d = Xh.numel() * Xh.element_size() + G0h.numel() * G0h.element_size() + F0h.numel() * F0h.element_size()
    d2h = (w.n * w.p + w.p * w.m) * Xh.element_size()

    def step_e2e():
        X = Xh.to("cuda", non_blocking=True)
        G0 = G0h.to("cuda", non_blocking=True)
        F0 = F0h.to("cuda", non_blocking=True)
        sk = nm.subspace_iteration_pair(X, w.nu, w.q, w.sketch_seed)
        out = nm.factorize_compressed(X, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True)
        G = out.G.to("cpu")
        F = out.F.to("cpu")
        return G, F

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k):
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
        b.record(stream)
        barrier()
        ms = a.elapsed_time(b)
        if dist is not None:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = lib.nenmf_launch_count()
    ms = timed(step_device, args.steps)
    launches = lib.nenmf_launch_count() - launches0
    clocks = sampler.stop()
    ms_step = ms / args.steps
    value = world * OUTER / (ms_step / 1e3)

    # end-to-end through the public API with host buffers
    step_e2e()
    ms_e2e = timed(step_e2e, max(1, min(args.steps, 3))) / max(1, min(args.steps, 3))
    e2e_value = world * OUTER / (ms_e2e / 1e3)

    # roofline of the kernels, timed on the launching stream with CUDA events
    roof = kernel_rooflines(w, Xd, args.dtype)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = cpu_sample(w, outer_sample=1)
        cpu = {"value": r["value"], "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": "full RSI sketch+compress on cfg2 X + 1 outer iteration (inner<=500) of the NumPy "
                         "restatement of the reference (float64, OpenBLAS all threads), extrapolated to 100 outer",
               "t_sketch_s": r["t_sketch_s"], "t_outer_s": r["t_outer_s"]}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64",
        "data": "synthetic (BASELINE cfg2 generator: U[0,1) G,F + 1% |N| noise, seed 1234; X resident in HBM)",
        "config": {"workload": "cfg2", "n": w.n, "m": w.m, "p": w.p, "p_prime": w.nu, "q": w.q,
                   "outer": OUTER, "inner_max_iter": w.inner, "grad_tol": 1e-4,
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (X = 400 MB fp32)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": ms_e2e},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roof["rsi"],
        "solver": roof["solver"],
        "kernels": roof["table"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6555.8), d.get("bf16_tflops", 1693.5), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def _traffic(kernel: str):
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(kernel)
    return None


def kernel_rooflines(w, Xd, dtype):
    """Time the RSI dual pass and one compressed solve in isolation (CUDA
    events on the current stream; inputs larger than L2 for the pass)."""
    import torch

    from paper_1812_04315_b200 import _lib, _ops, workloads
    from paper_1812_04315_b200.compression import compress_device, rsi_device

    hbm, _bf16, src = _peaks()
    stream = torch.cuda.current_stream()
    L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
    Yt = torch.empty((w.nu, w.n), dtype=Xd.dtype, device="cuda")
    Zt = torch.empty((w.nu, w.m), dtype=Xd.dtype, device="cuda")

    def ev_time(fn, reps):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    Xp = _ops.prepare_x(Xd, w.nu)
    if Xp is not None:
        # FP32: the passes of a sketch stream the prepared (tile-major bf16 hi/lo) copy of X,
        # 4 bytes per element like X itself; it is made once per sketch (timed separately)
        ms_prep = ev_time(lambda: _ops.prepare_x(Xd, w.nu), 5)
        ms_op = ev_time(lambda: _ops.dual_pass_prepared(Xp, w.n, w.m, Rt, L, Yt, Zt), 20)
        # the kernel alone: CUDA events around each k_dual_bulk launch on its stream
        import ctypes
        lib = _lib.load_library()
        lib.nenmf_debug_xpass_ms(None)
        lib.nenmf_debug_xpass_timing(1)
        for _ in range(20):
            _ops.dual_pass_prepared(Xp, w.n, w.m, Rt, L, Yt, Zt)
        tot = ctypes.c_double(0.0)
        cnt = lib.nenmf_debug_xpass_ms(ctypes.byref(tot))
        lib.nenmf_debug_xpass_timing(0)
        ms_pass = tot.value / max(cnt, 1)
        kname = "RSI X-pass (k_dual_bulk: bulk-copy stream of the prepared X -> X*A and X^T*B, tcgen05 BF16x3)"
    else:
        ms_prep = 0.0
        ms_pass = ev_time(lambda: _ops.dual_pass(Xd, Rt, L, Yt, Zt), 10)
        ms_op = ms_pass
        kname = "RSI X-pass (k_dual: one read of X -> X*A and X^T*B)"
    del Xp
    pass_bytes = w.n * w.m * Xd.element_size()
    ms_rsi = ev_time(lambda: rsi_device(Xd, w.nu, w.q, w.sketch_seed), 3)
    rsi_bytes = workloads.rsi_bytes(w.n, w.m, w.q, Xd.element_size())
    # compressed F-half solve at cfg2 (the dominant kernel of the step)
    XL, XRt = compress_device(Xd, L, Rt)
    F0 = _lib.to_device(w.F0, dtype)
    Gt = _lib.to_device(w.G0.T.copy(), dtype)
    GLt = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
    _ops.abt(Gt, L, GLt)
    Fo = torch.empty_like(F0)
    status = _lib.new_status()

    def solve():
        status.zero_()
        _ops.solve(GLt, XL, F0, Fo, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                   status=status)

    ms_solve = ev_time(solve, 5)
    iters = int(_lib.read_status(status)[0]["inner_iters"])
    s = Xd.element_size()
    pass_gbs = pass_bytes / (ms_pass * 1e-3) / 1e9
    rsi = {"bound": "hbm", "kernel": kname,
           "achieved": pass_gbs, "peak": hbm, "unit": "GB/s", "frac": pass_gbs / hbm,
           "traffic": _traffic("k_dual_bulk"), "peak_source": src,
           "algorithmic_bytes_per_launch": pass_bytes, "ms_per_launch": ms_pass,
           "ms_per_launch_source": "CUDA events around each k_dual_bulk launch on its stream (20 passes)",
           "ms_per_pass_op": ms_op,
           "pass_op_gbs": pass_bytes / (ms_op * 1e-3) / 1e9,
           "pass_op_includes": "skinny-operand split + k_dual_bulk + slab reduction (3 launches)",
           "prepare_x_ms_once_per_sketch": ms_prep,
           "rsi_total_ms": ms_rsi, "rsi_effective_gbs": rsi_bytes / (ms_rsi * 1e-3) / 1e9,
           "rsi_bytes_model": "(2q+2)*n*m*s_X (SURVEY 8d)"}
    # the inner solver is latency-bound (state lives in registers; one
    # dependent iteration after another), so its figure is time per iteration
    # next to the floors of SURVEY 8(d): HBM if the state were streamed, and
    # the tensor-pipe flops of W*F
    us_it = 1e3 * ms_solve / max(iters, 1)
    flops_it = 2 * w.p * w.p * w.m
    stream_bytes_it = 9 * w.p * w.m * s
    solver = {"bound": "latency", "kernel": "k_nnls_mma (persistent inner solver, F-half at cfg2)",
              "ms_per_launch": ms_solve, "inner_iters": iters, "us_per_inner_iter": us_it,
              "flops_per_iter": flops_it, "achieved_tflops": flops_it / (us_it * 1e-6) / 1e12,
              "hbm_floor_us_if_streamed": stream_bytes_it / (hbm * 1e9) * 1e6,
              "traffic": _traffic("k_nnls_mma")}
    table = {"dual_pass_kernel_ms": ms_pass, "dual_pass_op_ms": ms_op, "prepare_x_ms": ms_prep, "rsi_ms": ms_rsi,
             "solve_F_half_ms": ms_solve}
    return {"rsi": rsi, "solver": solver, "table": table}


# ------------------------------------------------- row-sharded arm (cfg5)
def run_sharded(args, rank, world, local_rank):
    """BASELINE cfg 5 (n = m = 1e5, p = 16, p' = 26, q = 4, fp32, 40 GB X
    generated on the device) with X row-sharded across the ranks (sharded.py):
    total work is fixed as N grows ("strong").  One step = sharded RSI sketch
    + compressed NeNMF (inner <= 500)."""
    import socket

    import torch
    import torch.distributed as dist

    import paper_1812_04315_b200 as nm
    from paper_1812_04315_b200 import _lib, _ops, sharded, workloads

    if "MASTER_ADDR" not in os.environ:  # N = 1 without torchrun
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]), RANK="0", WORLD_SIZE="1")
        s.close()
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    lib = _lib.load_library()
    Xl, r0, n, m, p, nu, q, inner, outer, G0, F0, sseed = workloads.device_shard(5, world, rank)
    outer = args.outer or outer
    comm = sharded.Comm()
    init = nm.FactorPair(G=G0, F=F0, p=p)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=inner), time_budget_seconds=0.0,
                         max_outer_iterations=outer, trace_every=outer)
    stream = torch.cuda.current_stream()
    rsi_ms = []

    def step():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sk = sharded.subspace_iteration_pair_sharded(Xl, n, nu, q, sseed, comm=comm)
        b.record(stream)
        sharded.factorize_compressed_sharded(Xl, n, sk, init, cfg, comm=comm, return_device=True)
        rsi_ms.append((a, b))

    def timed(fn, k):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
        b.record(stream)
        dist.barrier()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    rsi_ms.clear()
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = lib.nenmf_launch_count()
    ms = timed(step, args.steps)
    launches = lib.nenmf_launch_count() - launches0
    clocks = sampler.stop()
    ms_step = ms / args.steps
    rsi_step = statistics.median(a.elapsed_time(b) for a, b in rsi_ms)
    # roofline: one RSI pass over this rank's prepared rows
    hbm, _bf16, src = _peaks()
    Xp = _ops.prepare_x(Xl, nu)
    At = torch.randn((nu, m), device="cuda")
    Bt = torch.randn((nu, Xl.shape[0]), device="cuda")
    Yt = torch.empty((nu, Xl.shape[0]), device="cuda")
    Zt = torch.empty((nu, m), device="cuda")
    _ops.dual_pass_prepared(Xp, Xl.shape[0], m, At, Bt, Yt, Zt)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(5):
        _ops.dual_pass_prepared(Xp, Xl.shape[0], m, At, Bt, Yt, Zt)
    b.record(stream)
    torch.cuda.synchronize()
    ms_pass = a.elapsed_time(b) / 5
    pass_gbs = Xl.numel() * 4 / (ms_pass * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": "compressed-NeNMF outer iters/s (cfg5 n=m=1e5 p=16 p'=26 q=4, fp32, X row-sharded, sketch charged)",
            "value": outer / (ms_step / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic, generated on device (cfg5: U(0,1) G, F from derive_seed(1234,0); X = G F)",
            "config": {"workload": "cfg5", "n": n, "m": m, "p": p, "p_prime": nu, "q": q, "outer": outer,
                       "inner_max_iter": inner, "parallelism": f"row-sharded x{world} (NCCL)",
                       "l2": "inputs larger than L2 (X = 40 GB fp32)"},
            "e2e": None, "e2e_note": "cfg5 X is generated on the device by definition (40 GB never on host)",
            "gpu_launches": int(launches), "clocks": clocks, "rsi_ms_per_step": rsi_step,
            "roofline": {"bound": "hbm", "kernel": "RSI X-pass over this rank's prepared rows (k_dual_bulk)",
                         "achieved": pass_gbs, "peak": hbm, "unit": "GB/s", "frac": pass_gbs / hbm,
                         "traffic": None, "peak_source": src, "ms_per_launch": ms_pass,
                         "algorithmic_bytes_per_launch": Xl.numel() * 4},
            "cpu_baseline": None,
            "cpu_baseline_note": "the CPU oracle at cfg5 needs 80 GB of host RAM per copy of X (SURVEY 8(d)); "
                                 "the cfg2 line carries the CPU baseline",
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "cfg5":
        run_sharded(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
