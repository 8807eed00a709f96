"""One bench-like step (RSI + compressed NeNMF, cfg2 fp32) with few outer iterations, for ncu launch lists."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads
outer = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dtype = sys.argv[2] if len(sys.argv) > 2 else "fp32"
w = workloads.make_workload(2, dtype=dtype)
npdt = np.float32 if dtype == "fp32" else np.float64
Xd = torch.from_numpy(w.X.astype(npdt)).cuda()
G0 = torch.from_numpy(w.G0.astype(npdt)).cuda(); F0 = torch.from_numpy(w.F0.astype(npdt)).cuda()
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0, max_outer_iterations=outer, trace_every=outer)
for _ in range(2):
    sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
    out = nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True)
torch.cuda.synchronize()
print("ok")
