"""Benchmark: compressed-NeNMF outer iterations/s on BASELINE config 2 (B200).

One step = the hot path over one synthetic input: the randomized-subspace-
iteration sketch (``subspace_iteration_pair``, q=4, p'=30) charged to the run
as the reference CLI does (cli.py:159-168), then ``factorize_compressed`` for
100 outer iterations with inner Max_iter=500 (the reference default) on
n = m = 10^4, p = 20 (BASELINE.json configs[1]).  metric value = outer
iterations completed / device time of the step.

The headline (``value``, ``e2e``) runs in FP64 mode -- the reference's own
arithmetic (matrix.py:31-36), parity 1e-5 -- so it compares like for like
with the reference arm; ``fp32_mode`` reports the same workload in FP32 mode
(parity 1e-3) beside it, with its final RRE against the FP64 run's.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1: bench.py re-executes itself under torch.distributed.run with N
ranks (one per GPU) unless it already runs under it (WORLD_SIZE must then
equal N).  X is split into row blocks (sharded.py) and the ONE
problem runs across the ranks ("scaling": "strong"); ``cfg5_sharded``
reports BASELINE cfg 5 (10^5 x 10^5, 40 GB fp32, generated on the device) the
same way at every N.

--impl reference times the UNMODIFIED reference package (baseline/_ref, pip
installed from /root/reference; pure Python/NumPy, float64) through its
public API on the host cores: each step is one bounded sample (sketch +
compression + one outer iteration), reported as the same metric; rank 0 only.
If the package is missing, the NumPy restatement in oracle/ stands in
("kind": "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

UNIT = "outer_iter/s"
CFG = 2
OUTER = 100
L2_BYTES = 126 * 1024 * 1024


def metric_name(dtype: str) -> str:
    return (f"compressed-NeNMF outer iters/s (cfg2 n=m=1e4 p=20 p'=30 q=4, {dtype}, 100 outer, inner<=500, "
            f"sketch charged)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="fp64", choices=["fp64", "fp32"], help="headline arithmetic (default fp64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the fp32_mode and cfg5_sharded blocks")
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


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------ CPU baseline
def _reference_package():
    """The unmodified reference package installed in baseline/_ref, or None."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "nenmf" / "__init__.py").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import nenmf
    except Exception:  # noqa: BLE001 - any import failure means "not available"
        return None
    finally:
        sys.path.remove(str(ref))
    if not str(getattr(nenmf, "__file__", "")).startswith(str(ref)):
        return None
    return nenmf


def cpu_sample(w):
    """One bounded sample of the cfg2 workload on the host cores, timed through
    the UNMODIFIED reference package when it is installed (kind "reference"),
    else through the oracle's NumPy restatement (kind "port").  Measured: the
    sketch, a separate compression, and factorize_compressed with ONE outer
    iteration (its MonotonicClock = compression + the outer iteration, emits
    excluded, factorize.py:136-152; its wall time adds the two full-X RRE
    emits).  The rate of the 100-outer step is extrapolated from those parts:
    sketch + wall(1 outer) + 99 x (solver(1 outer) - compression)."""
    nenmf = _reference_package()
    t0 = time.perf_counter()
    if nenmf is not None:
        sk = nenmf.subspace_iteration_pair(w.X, w.nu, w.q, w.sketch_seed)
        t1 = time.perf_counter()
        nenmf.compress_problem(w.X, sk)
        t2 = time.perf_counter()
        clock = nenmf.MonotonicClock()
        cfg = nenmf.OuterConfig(inner=nenmf.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                                max_outer_iterations=1)
        nenmf.factorize_compressed(w.X, sk, nenmf.FactorPair(G=w.G0, F=w.F0, p=w.p), cfg, clock=clock)
        t3 = time.perf_counter()
        solver = clock.elapsed()
        kind = "reference"
    else:
        sys.path.insert(0, str(REPO / "oracle"))
        import nenmf_oracle as orc

        L, R = orc.rsi(w.X, w.nu, w.q, w.sketch_seed)
        t1 = time.perf_counter()
        orc.compress(w.X, L, R)
        t2 = time.perf_counter()
        ts = time.perf_counter()
        orc.nenmf(w.X, w.G0, w.F0, L=L, R=R, max_outer=1, max_iter=w.inner, trace_every=2)
        t3 = time.perf_counter()
        solver = t3 - ts  # includes the final emit: an upper bound
        kind = "port"
    t_sketch, t_compress, t_fc = t1 - t0, t2 - t1, t3 - t2
    t_outer = max(solver - t_compress, 1e-9)
    total = t_sketch + t_fc + (OUTER - 1) * t_outer
    return {"value": OUTER / total, "kind": kind, "sample_s": t3 - t0, "t_sketch_s": t_sketch,
            "t_compress_s": t_compress, "t_factorize_1outer_wall_s": t_fc, "t_outer_solver_s": t_outer,
            "extrapolated_100_outer_s": total}


# -------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1812_04315_b200 import workloads

    w = workloads.make_workload(CFG, dtype="fp64")
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(w)
        if i >= args.warmup:
            vals.append(r)
            walls.append(r["sample_s"])
    value = statistics.median(v["value"] for v in vals)
    kind = vals[-1]["kind"]
    what = ("the unmodified reference package (baseline/_ref: nenmf.subspace_iteration_pair, compress_problem, "
            "factorize_compressed with MonotonicClock)" if kind == "reference" else
            "the oracle's NumPy restatement of the reference (baseline/_ref not installed)")
    sample = (f"per step: {what} on cfg2 X (float64): the sketch, one compression, and 1 outer iteration "
              f"(inner<=500); the 100-outer rate is extrapolated as sketch + wall(1 outer incl. 2 RRE emits) "
              f"+ 99 x (solver-clock outer - compression)")
    line = {
        "metric": metric_name("fp64"), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE cfg2 generator, seed 1234)", "impl": "reference",
        "config": {"workload": "cfg2", "n": w.n, "m": w.m, "p": w.p, "p_prime": w.nu, "q": w.q,
                   "outer": OUTER, "inner_max_iter": w.inner, "parallelism": "host cores (OpenBLAS threads)"},
        "ms_per_step_meaning": "measured wall time of one sample (what a step of this arm runs)",
        "extrapolation": {"outer_measured_per_step": 1, "outer_in_metric": OUTER,
                          "extrapolated_step_s": statistics.median(v["extrapolated_100_outer_s"] for v in vals)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "samples": vals,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ helpers
def _peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6555.8), d.get("bf16_tflops", 1693.5), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def _fp64_peak():
    p = REPO / "profiles" / "fp64_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["fp64_dmma_tflops"], "measured on this pool's B200 by tools/micro/fp64_peak.cu (profiles/fp64_peak.json)"
    return 37.0, "fallback: nominal B200 FP64 tensor figure (no measurement committed)"


class Timer:
    """CUDA-event timing on the current stream with a synchronize on both sides."""

    def __init__(self, torch, dist=None):
        self.torch, self.dist = torch, dist

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def __call__(self, fn, k, between=None):
        torch = self.torch
        stream = torch.cuda.current_stream()
        self.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
            if between is not None:
                between()
        b.record(stream)
        self.barrier()
        ms = a.elapsed_time(b)
        if self.dist is not None:
            t = torch.tensor([ms], device="cuda")
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms


class Problem:
    """The cfg2 problem on this rank: the whole X (world 1) or its row block
    (sharded.py), resident in HBM, plus pinned host copies for the e2e leg."""

    def __init__(self, w, dtype, world, rank):
        import numpy as np
        import torch

        from paper_1812_04315_b200 import sharded

        self.w, self.dtype, self.world, self.rank = w, dtype, world, rank
        npdt = np.float32 if dtype == "fp32" else np.float64
        self.row0, self.rows = sharded.row_block(w.n, world, rank)
        Xl = np.ascontiguousarray(w.X[self.row0:self.row0 + self.rows].astype(npdt))
        self.Xh = torch.from_numpy(Xl).pin_memory()
        self.G0h = torch.from_numpy(w.G0.astype(npdt)).pin_memory()
        self.F0h = torch.from_numpy(w.F0.astype(npdt)).pin_memory()
        self.Xd = self.Xh.to("cuda")
        self.G0d = self.G0h.to("cuda")
        self.F0d = self.F0h.to("cuda")
        self.h2d = sum(t.numel() * t.element_size() for t in (self.Xh, self.G0h, self.F0h))
        self.d2h = (w.n * w.p + w.p * w.m) * self.Xh.element_size()
        self.flush = None
        if self.Xd.numel() * self.Xd.element_size() < 2 * L2_BYTES:
            # this rank's X would stay in L2 between steps: overwrite L2 after each step
            self.flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")

    def l2_flush(self):
        if self.flush is not None:
            from paper_1812_04315_b200 import _lib

            _lib.zero_(self.flush)

    def cfg(self, outer, trace_every=None):
        import paper_1812_04315_b200 as nm

        return nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=self.w.inner), time_budget_seconds=0.0,
                              max_outer_iterations=outer, trace_every=trace_every or outer)

    def step(self, X, G0, F0, cfg, comm=None, observer=None):
        """sketch + factorize through the public API (device tensors in and out)."""
        import paper_1812_04315_b200 as nm
        from paper_1812_04315_b200 import sharded

        w = self.w
        init = nm.FactorPair(G=G0, F=F0, p=w.p)
        if self.world == 1:
            sk = nm.subspace_iteration_pair(X, w.nu, w.q, w.sketch_seed)
            return nm.factorize_compressed(X, sk, init, cfg, observer=observer, return_device=True)
        sk = sharded.subspace_iteration_pair_sharded(X, w.n, w.nu, w.q, w.sketch_seed, comm=comm)
        return sharded.factorize_compressed_sharded(X, w.n, sk, init, cfg, observer=observer, comm=comm,
                                                    return_device=True)

    def step_e2e(self, cfg, comm=None):
        X = self.Xh.to("cuda", non_blocking=True)
        G0 = self.G0h.to("cuda", non_blocking=True)
        F0 = self.F0h.to("cuda", non_blocking=True)
        out = self.step(X, G0, F0, cfg, comm)
        return out.G.to("cpu"), out.F.to("cpu")

    def final_rre(self, outer, comm=None):
        import paper_1812_04315_b200 as nm

        rec = nm.TraceRecorder()
        self.step(self.Xd, self.G0d, self.F0d, self.cfg(outer), comm, observer=rec)
        return rec.records[-1].rre


def measure_workload(args, w, dtype, world, rank, dist, comm, outer):
    """value / e2e / launches / clocks of cfg2 in one arithmetic mode."""
    import torch

    from paper_1812_04315_b200 import _lib

    lib = _lib.load_library()
    timer = Timer(torch, dist)
    P = Problem(w, dtype, world, rank)
    cfg = P.cfg(outer)
    run = lambda: P.step(P.Xd, P.G0d, P.F0d, cfg, comm)  # noqa: E731
    for _ in range(args.warmup):
        run()
        P.l2_flush()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    launches0 = lib.nenmf_launch_count()
    ms = timer(run, args.steps, between=P.l2_flush)
    launches = (lib.nenmf_launch_count() - launches0) // args.steps
    clocks = sampler.stop()
    ms_step = ms / args.steps
    P.step_e2e(cfg, comm)
    k = max(1, min(args.steps, 3))
    ms_e2e = timer(lambda: P.step_e2e(cfg, comm), k) / k
    rre = P.final_rre(outer, comm)
    res = {"value": outer / (ms_step / 1e3), "ms_per_step": ms_step,
           "e2e": {"value": outer / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": P.h2d,
                   "d2h_bytes_per_step": P.d2h, "ms_per_step": ms_e2e},
           "gpu_launches": int(launches), "clocks": clocks, "final_rre": rre,
           "l2": ("inputs larger than L2 (this rank's X: %.0f MB)" % (P.Xd.numel() * P.Xd.element_size() / 1e6)
                  if P.flush is None else "L2 flushed after every step (this rank's X: %.0f MB < 2 x L2)"
                  % (P.Xd.numel() * P.Xd.element_size() / 1e6))}
    return res, P


def rsi_roofline(P, dtype):
    """The RSI X-pass (the kernel north_star's roofline target names) and the
    whole sketch + compression, on this rank's X, CUDA events on the stream
    the kernels run on."""
    import ctypes

    import torch

    from paper_1812_04315_b200 import _lib, _ops, workloads
    from paper_1812_04315_b200.compression import compress_device, rsi_device

    w = P.w
    Xd = P.Xd
    n, m = Xd.shape
    hbm, _bf16, src = _peaks()
    timer = Timer(torch)
    L, Rt, _ = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
    Yt = torch.empty((w.nu, n), dtype=Xd.dtype, device="cuda")
    Zt = torch.empty((w.nu, m), dtype=Xd.dtype, device="cuda")
    pass_bytes = n * m * Xd.element_size()
    pass_flops = 2 * 2 * n * m * w.nu  # Y = X A and Z = X^T B
    Xp = _ops.prepare_x(Xd, w.nu)
    lib = _lib.load_library()
    if Xp is not None:
        ms_prep = timer(lambda: _ops.prepare_x(Xd, w.nu), 5) / 5
        ms_op = timer(lambda: _ops.dual_pass_prepared(Xp, n, m, Rt, L, Yt, Zt), 20) / 20
        kname = "k_dual_bulk (RSI X-pass: bulk-copy stream of the prepared X -> X*A and X^T*B, tcgen05 BF16x3)"
        op = lambda: _ops.dual_pass_prepared(Xp, n, m, Rt, L, Yt, Zt)  # noqa: E731
    else:
        ms_prep = 0.0
        ms_op = timer(lambda: _ops.dual_pass(Xd, Rt, L, Yt, Zt), 10) / 10
        kname = ("k_dual64t (RSI X-pass in FP64: one TMA read of X feeds X*A and X^T*B on the DMMA tensor pipe)"
                 if os.environ.get("NENMF_DUAL64", "")[:1] != "o" else
                 "k_xv64 + k_ux64 (RSI X-pass in FP64 on the DMMA tensor pipe, two reads of X)")
        op = lambda: _ops.dual_pass(Xd, Rt, L, Yt, Zt)  # noqa: E731
    # the kernel(s) alone: CUDA events the library records around each X-pass
    # launch on its own stream
    lib.nenmf_debug_xpass_ms(None)
    lib.nenmf_debug_xpass_timing(1)
    for _ in range(20):
        op()
    tot = ctypes.c_double(0.0)
    cnt = lib.nenmf_debug_xpass_ms(ctypes.byref(tot))
    lib.nenmf_debug_xpass_timing(0)
    # per pass; a path without the hook (FP64 before the fused pass) reports the whole pass op
    ms_pass = tot.value / 20.0 if cnt > 0 else ms_op
    del Xp

    def sketch_and_compress():
        L2, Rt2, _ = rsi_device(Xd, w.nu, w.q, w.sketch_seed, check=False)
        compress_device(Xd, L2, Rt2)

    ms_rsi = timer(sketch_and_compress, 3) / 3
    rsi_bytes = workloads.rsi_bytes(n, m, w.q, Xd.element_size())
    rsi_gbs = rsi_bytes / (ms_rsi * 1e-3) / 1e9
    if dtype == "fp32":
        ach = pass_bytes / (ms_pass * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_source": src, "algorithmic_bytes_per_launch": pass_bytes}
    else:
        peak, psrc = _fp64_peak()
        ach = pass_flops / (ms_pass * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": kname, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "peak_source": psrc, "algorithmic_flops_per_pass": pass_flops,
                "hbm_gbs_same_pass": pass_bytes / (ms_pass * 1e-3) / 1e9,
                "hbm_frac_same_pass": pass_bytes / (ms_pass * 1e-3) / 1e9 / hbm}
    roof.update({
        "traffic": None,
        "traffic_note": "dram bytes per launch come from the committed ncu --set full capture (profiles/)",
        "ms_per_launch": ms_pass,
        "ms_per_launch_source": "CUDA events around each X-pass launch on the library's stream (20 passes)",
        "ms_per_pass_op": ms_op, "prepare_x_ms_once_per_sketch": ms_prep,
        "rsi_total": {"ms": ms_rsi, "bytes": rsi_bytes, "gbs": rsi_gbs, "frac_hbm": rsi_gbs / hbm,
                      "what": "sketch (2q+1 passes) + compression (1 pass) timed together; "
                              "bytes = (2q+2) n m s_X (SURVEY 8(d))"},
    })
    return roof


def solver_probe(P, dtype):
    """One compressed F-half solve at cfg2 (the kernel that dominates the step)."""
    import torch

    from paper_1812_04315_b200 import _lib, _ops
    from paper_1812_04315_b200.compression import compress_device, rsi_device

    w = P.w
    Xd = P.Xd
    timer = Timer(torch)
    L, Rt, _ = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
    XL, XRt = compress_device(Xd, L, Rt)
    F0 = _lib.to_device(w.F0, dtype)
    Gt = _lib.to_device(w.G0[P.row0:P.row0 + P.rows].T.copy(), dtype)
    GLt = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
    _ops.abt(Gt, L, GLt)
    Fo = torch.empty_like(F0)
    status = _lib.new_status()

    def solve():
        _lib.zero_(status)
        _ops.solve(GLt, XL, F0, Fo, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                   status=status)

    solve()
    ms = timer(solve, 5) / 5
    iters = int(_lib.read_status(status)[0]["inner_iters"])
    us_it = 1e3 * ms / max(iters, 1)
    flops_it = 2 * w.p * w.p * w.m
    hbm, _, _ = _peaks()
    out = {"bound": "latency", "kernel": f"k_nnls_mma<{'double' if dtype == 'fp64' else 'float'}> "
                                         "(persistent inner solver, F-half at cfg2)",
           "ms_per_launch": ms, "inner_iters": iters, "us_per_inner_iter": us_it, "flops_per_iter": flops_it,
           "achieved_tflops": flops_it / (us_it * 1e-6) / 1e12,
           "hbm_floor_us_if_streamed": 9 * w.p * w.m * Xd.element_size() / (hbm * 1e9) * 1e6}
    if dtype == "fp64":
        peak, _ = _fp64_peak()
        out["frac_fp64_tensor_peak"] = out["achieved_tflops"] / peak
    return out


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1812_04315_b200 import _lib, sharded, workloads

    torch.cuda.set_device(local_rank)
    dist = comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        comm = sharded.Comm()
    _lib.load_library()
    outer = args.outer or OUTER
    dtype = args.dtype
    w = workloads.make_workload(CFG, dtype=dtype)
    head, P = measure_workload(args, w, dtype, world, rank, dist, comm, outer)
    roof = rsi_roofline(P, dtype)
    solver = solver_probe(P, dtype)
    del P
    torch.cuda.empty_cache()

    fp32 = None
    if not args.no_secondary and dtype == "fp64":
        w32 = workloads.make_workload(CFG, dtype="fp32")
        res32, P32 = measure_workload(args, w32, "fp32", world, rank, dist, comm, outer)
        res32["roofline"] = rsi_roofline(P32, "fp32")
        res32["solver"] = solver_probe(P32, "fp32")
        res32["metric"] = metric_name("fp32")
        res32["final_rre_rel_diff_vs_fp64_run"] = abs(res32["final_rre"] - head["final_rre"]) / head["final_rre"]
        fp32 = res32
        del P32
        torch.cuda.empty_cache()

    vanilla = vanilla32 = None
    if not args.no_secondary:
        vanilla = run_vanilla(args, w, dtype, rank, world)
        if dtype == "fp64":
            vanilla32 = run_vanilla(args, workloads.make_workload(CFG, dtype="fp32"), "fp32", rank, world,
                                    cpu_leg=False)

    cfg5 = None
    if not args.no_secondary:
        cfg5 = run_cfg5(args, rank, world, local_rank, dist, comm)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        w64 = w if dtype == "fp64" else workloads.make_workload(CFG, dtype="fp64")
        r = cpu_sample(w64)
        cpu = {"value": r["value"], "unit": UNIT, "cores": cores(), "kind": r["kind"],
               "sample": ("one sample of cfg2 on the host cores: the sketch, one compression and 1 outer iteration "
                          "(inner<=500) of " + ("the unmodified reference package (baseline/_ref), float64, "
                                                "OpenBLAS on all threads" if r["kind"] == "reference" else
                                                "the oracle's NumPy restatement, float64") +
                          "; the 100-outer rate extrapolated from the measured parts"),
               "detail": r}
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    line = {
        "metric": metric_name(dtype), "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if dtype == "fp64" else "f32",
        "data": "synthetic (BASELINE cfg2 generator: U[0,1) G,F + 1% |N| noise, seed 1234; X resident in HBM)",
        "config": {"workload": "cfg2", "n": w.n, "m": w.m, "p": w.p, "p_prime": w.nu, "q": w.q, "outer": outer,
                   "inner_max_iter": w.inner, "grad_tol": 1e-4, "arithmetic": f"{dtype} mode",
                   "parallelism": f"X row-sharded x{world} (sharded.py)" if world > 1 else "1 GPU",
                   "l2": head["l2"]},
        "e2e": head["e2e"], "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
        "final_rre": head["final_rre"],
        "roofline": roof, "solver": solver,
        "fp32_mode": fp32, "vanilla": vanilla, "vanilla_fp32": vanilla32, "cfg5_sharded": cfg5,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ------------------------------------------------------ vanilla cfg2 block
def run_vanilla(args, w, dtype, rank, world, cpu_leg=True):
    """Vanilla NeNMF (factorize_vanilla, factorize.py:186-194) on BASELINE cfg 2
    (1 GPU as BASELINE.json states): 100 outer iterations, inner <= 500, on
    the full X; value = outer it/s.  FP32 forms V = A^T X with the tcgen05 pass
    over the prepared X; FP64 on the DMMA pipe.  Beside it, the reference
    package's factorize_vanilla timed for one outer iteration on the host."""
    import numpy as np
    import torch

    import paper_1812_04315_b200 as nm

    if world > 1 or rank != 0:
        return None
    npdt = np.float32 if dtype == "fp32" else np.float64
    Xd = torch.from_numpy(w.X.astype(npdt)).cuda()
    G0 = torch.from_numpy(w.G0.astype(npdt)).cuda()
    F0 = torch.from_numpy(w.F0.astype(npdt)).cuda()
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                         max_outer_iterations=OUTER, trace_every=OUTER)
    run = lambda: nm.factorize_vanilla(Xd, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True)  # noqa: E731
    run()
    timer = Timer(torch)
    k = max(1, min(args.steps, 2))
    ms = timer(run, k) / k
    out = {"metric": f"vanilla NeNMF outer iters/s (cfg2 n=m=1e4 p=20, {dtype}, 100 outer, inner<=500)",
           "value": OUTER / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": k, "dtype": dtype,
           "v_products": "tcgen05 BF16x3 pass over the prepared X" if dtype == "fp32" else "DMMA (FP64 tensor pipe)",
           "tie_break_residuals": ("tcgen05 pair pass over the prepared X (k_resid_bulk)" if dtype == "fp32"
                                   else "DMMA (k_resid64)")}
    if cpu_leg and not args.no_cpu_baseline:
        nenmf = _reference_package()
        if nenmf is not None:
            t0 = time.perf_counter()
            clock = nenmf.MonotonicClock()
            ccfg = nenmf.OuterConfig(inner=nenmf.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                                     max_outer_iterations=1)
            nenmf.factorize_vanilla(w.X, nenmf.FactorPair(G=w.G0, F=w.F0, p=w.p), ccfg, clock=clock)
            wall = time.perf_counter() - t0
            solver = clock.elapsed()
            out["cpu_baseline"] = {"value": OUTER / (wall + (OUTER - 1) * solver), "unit": UNIT, "cores": cores(),
                                   "kind": "reference",
                                   "sample": "the unmodified reference package's factorize_vanilla, 1 outer iteration "
                                             "(float64, OpenBLAS all threads); 100-outer rate = wall(1 outer incl. 2 "
                                             "emits) + 99 x solver-clock outer",
                                   "t_wall_s": wall, "t_outer_solver_s": solver}
    del Xd
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------- row-sharded cfg5 block
def run_cfg5(args, rank, world, local_rank, dist, comm):
    """BASELINE cfg 5 (n = m = 1e5, p = 16, p' = 26, q = 4, fp32, 40 GB X
    generated on the device) with X row-sharded across the ranks (sharded.py):
    total work is fixed as N grows ("strong").  One step = sharded RSI sketch
    + compressed NeNMF (inner <= 500, 50 outer)."""
    import os
    import socket

    import torch
    import torch.distributed as tdist

    import paper_1812_04315_b200 as nm
    from paper_1812_04315_b200 import _lib, sharded, workloads

    own_pg = False
    if comm is None:
        if "MASTER_ADDR" not in os.environ:
            s = socket.socket()
            s.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
            s.close()
        tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local_rank))
        comm, own_pg = sharded.Comm(), True
    lib = _lib.load_library()
    Xl, r0, n, m, p, nu, q, inner, outer, G0, F0, sseed = workloads.device_shard(5, world, rank)
    outer = min(outer, args.outer or outer)
    init = nm.FactorPair(G=G0, F=F0, p=p)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=inner), time_budget_seconds=0.0,
                         max_outer_iterations=outer, trace_every=outer)
    stream = torch.cuda.current_stream()
    rsi_ev = []

    def step():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sk = sharded.subspace_iteration_pair_sharded(Xl, n, nu, q, sseed, comm=comm)
        b.record(stream)
        sharded.factorize_compressed_sharded(Xl, n, sk, init, cfg, comm=comm, return_device=True)
        rsi_ev.append((a, b))

    timer = Timer(torch, dist)
    for _ in range(max(1, min(args.warmup, 2))):
        step()
    rsi_ev.clear()
    launches0 = lib.nenmf_launch_count()
    k = max(1, min(args.steps, 3))
    ms = timer(step, k)
    launches = (lib.nenmf_launch_count() - launches0) // k
    ms_step = ms / k
    rsi_step = statistics.median(a.elapsed_time(b) for a, b in rsi_ev)
    hbm, _, _ = _peaks()
    rsi_bytes = workloads.rsi_bytes(Xl.shape[0], m, q, 4) - Xl.shape[0] * m * 4  # 2q+1 sketch passes
    out = {"metric": "compressed-NeNMF outer iters/s (cfg5 n=m=1e5 p=16 p'=26 q=4, fp32, 50 outer, X row-sharded, "
                     "sketch charged)",
           "value": outer / (ms_step / 1e3), "unit": UNIT, "ms_per_step": ms_step, "steps": k, "n_gpus": world,
           "scaling": "strong", "gpu_launches": int(launches), "rsi_ms_per_step": rsi_step,
           "rsi_sketch_gbs_per_rank": rsi_bytes / (rsi_step * 1e-3) / 1e9,
           "rsi_sketch_frac_hbm": rsi_bytes / (rsi_step * 1e-3) / 1e9 / hbm,
           "data": "synthetic, generated on the device (cfg5: U(0,1) G, F from derive_seed(1234,0); X = G F)",
           "l2": "inputs larger than L2 (X = 40 GB fp32 in total)"}
    del Xl
    torch.cuda.empty_cache()
    if own_pg:
        tdist.destroy_process_group()
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torch.distributed.run (rank 0 prints)
        import socket

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
