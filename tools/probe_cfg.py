"""RSI + a few outer iterations at BASELINE cfg3 / cfg4 (timing probe)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, _lib
from paper_1812_04315_b200.compression import rsi_device
cfgn = int(sys.argv[1]); outer = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time()
w = workloads.make_workload(cfgn, dtype="fp32")
print(f"cfg{cfgn} gen {time.time()-t0:.1f}s  n={w.n} m={w.m} p={w.p} nu={w.nu}", flush=True)
Xd = _lib.to_device(w.X, "fp32")
G0 = _lib.to_device(w.G0, "fp32"); F0 = _lib.to_device(w.F0, "fp32")
def ev(fn, reps=1):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ms = ev(lambda: rsi_device(Xd, w.nu, w.q, w.sketch_seed))
print(f"  RSI {ms:.2f} ms -> {workloads.rsi_bytes(w.n, w.m, w.q, 4)/ms/1e6:.0f} GB/s effective", flush=True)
sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                     max_outer_iterations=outer, trace_every=outer)
ms = ev(lambda: nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True))
print(f"  compress + {outer} outer: {ms:.1f} ms -> {outer/(ms/1e3):.2f} outer it/s", flush=True)
