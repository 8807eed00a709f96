"""GPU driver of the paper's comparison: time to a target RRE, vanilla vs
compressed NeNMF, sketch construction charged to the compressed method
(the reference's ``nenmf-bench run``, cli.py:145-181
and its summary, cli.py:189-269 and 299-364).

Per seed, as the reference CLI does: the instance is ``generate_problem(n, m,
p, snr_db, seed)`` (here generated on the device, bit-identical draws); the
initial factors come from ``derive_seed(seed, 1)``; the sketch from
``derive_seed(seed, 2)``; with the real clock the sketch build time (measured
after a device synchronisation) is the MonotonicClock's offset, so the
compressed method's trace starts at the cost of its sketch (cli.py:159-168).
Every method's trace is written as the reference's CSV (tracing.py:89-110)
and a summary with the reference's fields (time/iterations to each target,
per seed and medians) goes to ``summary.json``; ``compare`` adds the ratio
compressed / vanilla of the median time to each target (the paper's Fig. 1
claim; the reference's acceptance criterion 8 asks for <= 0.5).

  python -m paper_1812_04315_b200.timebench --n 2000 --m 2000 --p 15 --nu 25 --q 4 \\
      --snr-db 30 --seeds 1 2 3 --targets 0.05 --budget-s 5 --out /tmp/cmp
"""

from __future__ import annotations

import argparse
import json
import statistics
import time
from dataclasses import dataclass, field
from pathlib import Path

from . import _lib
from .compression import power_iteration_pair, subspace_iteration_pair
from .factorize import OuterConfig, factorize_compressed, factorize_vanilla, init_factors
from .nnls import InnerSolverConfig
from .synthetic import generate_problem_device
from .tracing import (IterationClock, MonotonicClock, TraceRecorder, iterations_to_target, time_to_target,
                      write_trace_csv)
from .workloads import derive_seed

METHODS = ("vanilla", "power", "subspace")
_INIT_STREAM, _SKETCH_STREAM = 1, 2  # cli.py:50-52


@dataclass
class RunSpec:
    n: int
    m: int
    p: int
    nu: int = 25
    q: int = 4
    snr_db: float = 30.0
    seeds: tuple = (1,)
    targets: tuple = (0.05,)
    budget_s: float = 15.0
    max_outer: int = 0
    max_inner: int = 500
    grad_tol: float = 1e-4
    trace_every: int = 1
    clock: str = "real"
    dtype: str = "fp64"
    extra: dict = field(default_factory=dict)


def run_seed(spec: RunSpec, method: str, seed: int, inst=None) -> dict:
    """One seed of one method (cli.py:_run_one_seed) on the GPU."""
    _, torch = _lib.require_device()
    if inst is None:
        inst = generate_problem_device(spec.n, spec.m, spec.p, spec.snr_db, seed, dtype=spec.dtype)
    init = init_factors(spec.n, spec.m, spec.p, derive_seed(seed, _INIT_STREAM))
    cfg = OuterConfig(inner=InnerSolverConfig(max_iter=spec.max_inner, grad_tol=spec.grad_tol),
                      time_budget_seconds=spec.budget_s, max_outer_iterations=spec.max_outer,
                      trace_every=spec.trace_every)
    rec = TraceRecorder()
    sketch, build_s = None, 0.0
    X = inst.X
    if method != "vanilla":
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        make = power_iteration_pair if method == "power" else subspace_iteration_pair
        sketch = make(X, spec.nu, spec.q, derive_seed(seed, _SKETCH_STREAM))
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
    clock = IterationClock() if spec.clock == "iteration" else MonotonicClock(offset=build_s)
    if sketch is None:
        factorize_vanilla(X, init, cfg, observer=rec, clock=clock, dtype=spec.dtype)
    else:
        factorize_compressed(X, sketch, init, cfg, observer=rec, clock=clock, dtype=spec.dtype)
    recs = rec.records
    final = recs[-1]
    return {
        "seed": seed, "status": "ok", "error": None, "records": recs,
        "final_rre": final.rre, "final_objective": final.objective, "outer_iterations": final.outer_iter,
        "solver_elapsed_s": final.solver_elapsed_s, "wall_elapsed_s": final.wall_elapsed_s,
        "sketch_build_s": build_s,
        "time_to_target": {str(t): time_to_target(recs, t) for t in spec.targets},
        "iterations_to_target": {str(t): iterations_to_target(recs, t) for t in spec.targets},
        "realized_snr_db": inst.snr_db_realized,
    }


def _median(values):
    values = [v for v in values if v is not None]
    return statistics.median(values) if values else None


def summarize(spec: RunSpec, method: str, per_seed: list) -> dict:
    """The reference's summary fields (cli.py:_write_summary)."""
    ok = [s for s in per_seed if s["status"] == "ok"]
    return {
        "method": method, "n": spec.n, "m": spec.m, "p": spec.p, "nu": spec.nu, "q": spec.q,
        "snr_db": spec.snr_db, "budget_s": spec.budget_s, "max_inner": spec.max_inner, "clock": spec.clock,
        "targets": list(spec.targets), "seeds": list(spec.seeds), "dtype": spec.dtype,
        "per_seed": [{k: v for k, v in s.items() if k != "records"} for s in per_seed],
        "medians": {
            "final_rre": _median([s["final_rre"] for s in ok]),
            "solver_elapsed_s": _median([s["solver_elapsed_s"] for s in ok]),
            "sketch_build_s": _median([s["sketch_build_s"] for s in ok]),
            "time_to_target": {str(t): _median([s["time_to_target"][str(t)] for s in ok]) for t in spec.targets},
            "iterations_to_target": {str(t): _median([s["iterations_to_target"][str(t)] for s in ok])
                                     for t in spec.targets},
        },
        "failed_seeds": [s["seed"] for s in per_seed if s["status"] != "ok"],
    }


def compare(spec: RunSpec, methods=("vanilla", "subspace"), out=None) -> dict:
    """Run every method on every seed (the same device instance per seed),
    write traces and summaries under ``out`` if given, and return the
    summaries with the compressed / vanilla ratios of the median times."""
    results = {m: [] for m in methods}
    for seed in spec.seeds:
        inst = generate_problem_device(spec.n, spec.m, spec.p, spec.snr_db, seed, dtype=spec.dtype)
        for method in methods:
            res = run_seed(spec, method, seed, inst)
            results[method].append(res)
            if out is not None:
                d = Path(out) / method
                d.mkdir(parents=True, exist_ok=True)
                write_trace_csv(res["records"], d / f"trace_{method}_seed{seed}.csv")
        del inst
    summaries = {m: summarize(spec, m, results[m]) for m in methods}
    ratios = {}
    if "vanilla" in summaries:
        van = summaries["vanilla"]["medians"]["time_to_target"]
        for m in methods:
            if m == "vanilla":
                continue
            mine = summaries[m]["medians"]["time_to_target"]
            ratios[m] = {t: (mine[t] / van[t] if mine[t] is not None and van[t] else None) for t in van}
    report = {"summaries": summaries, "time_to_target_ratio_vs_vanilla": ratios}
    if out is not None:
        for m, summ in summaries.items():
            (Path(out) / m / "summary.json").write_text(json.dumps(summ, sort_keys=True, indent=2) + "\n")
        (Path(out) / "comparison.json").write_text(
            json.dumps({"time_to_target_ratio_vs_vanilla": ratios}, sort_keys=True, indent=2) + "\n")
    return report


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--p", type=int, required=True)
    ap.add_argument("--nu", type=int, default=25)
    ap.add_argument("--q", type=int, default=4)
    ap.add_argument("--snr-db", type=float, default=30.0)
    ap.add_argument("--seeds", type=int, nargs="+", default=[1])
    ap.add_argument("--targets", type=float, nargs="+", default=[0.05])
    ap.add_argument("--budget-s", type=float, default=15.0)
    ap.add_argument("--max-outer", type=int, default=0)
    ap.add_argument("--max-inner", type=int, default=500)
    ap.add_argument("--methods", nargs="+", default=["vanilla", "subspace"], choices=METHODS)
    ap.add_argument("--dtype", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--clock", default="real", choices=["real", "iteration"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    spec = RunSpec(a.n, a.m, a.p, a.nu, a.q, a.snr_db, tuple(a.seeds), tuple(a.targets), a.budget_s, a.max_outer,
                   a.max_inner, clock=a.clock, dtype=a.dtype)
    rep = compare(spec, tuple(a.methods), a.out)
    print(json.dumps({"medians": {m: s["medians"] for m, s in rep["summaries"].items()},
                      "time_to_target_ratio_vs_vanilla": rep["time_to_target_ratio_vs_vanilla"]}, indent=2))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
