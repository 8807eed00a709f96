"""Vanilla NeNMF outer-iteration rate at BASELINE cfg2 (timing probe)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, _lib
dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = workloads.make_workload(2, dtype=dtype)
Xd = _lib.to_device(w.X, dtype); G0 = _lib.to_device(w.G0, dtype); F0 = _lib.to_device(w.F0, dtype)
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                     max_outer_iterations=outer, trace_every=outer)
tv = len(sys.argv) > 3
run = lambda: nm.factorize_vanilla(Xd, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True, tensor_v=tv)
run(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); run(); b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(f"vanilla cfg2 {dtype}: {outer} outer in {ms:.1f} ms -> {outer/(ms/1e3):.1f} outer it/s")
