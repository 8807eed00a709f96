"""BASELINE cfg1 (fp64, n = m = 1000, inner 10, 50 outer) wall rate through the public API; development aid."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads
w = workloads.make_workload(1, dtype="fp64")
for rep in range(3):
    t0 = time.perf_counter()
    sk = nm.subspace_iteration_pair(w.X, w.nu, w.q, w.sketch_seed)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0, max_outer_iterations=50, trace_every=50)
    out = nm.factorize_compressed(w.X, sk, nm.FactorPair(G=w.G0, F=w.F0, p=w.p), cfg)
    t1 = time.perf_counter()
    print(f"cfg1 fp64: sketch + 50 outer {1e3*(t1-t0):.1f} ms -> {50/(t1-t0):.0f} outer it/s (wall, host numpy in/out)", flush=True)
