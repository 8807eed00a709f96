"""cfg5 proxy (n = m = 10^4, noiseless rank 16, p' = 26), FP32: one-step parity of the plain device
path (factorize_compressed) against the oracle, and of float32 NumPy (the reference algorithm run
in float32) against the same oracle step, per outer iteration.  Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np
import torch

import nenmf_oracle as orc
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads

outer = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = workloads.make_workload(5, n=10000, m=10000)
X = torch.from_numpy(w.X.astype(np.float32)).to("cuda")
sk = nm.subspace_iteration_pair(X, w.nu, w.q, seed=w.sketch_seed)
init = nm.FactorPair(G=torch.from_numpy(w.G0.astype(np.float32)).to("cuda"),
                     F=torch.from_numpy(w.F0.astype(np.float32)).to("cuda"), p=w.p)
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                     max_outer_iterations=outer)
rec, facs = nm.TraceRecorder(), []


def observe(r, G, F):
    rec(r, G, F)
    facs.append((np.array(G, dtype=np.float64), np.array(F, dtype=np.float64)))


nm.factorize_compressed(X, sk, init, cfg, observer=observe, clock=nm.IterationClock())
L, R = np.asarray(sk.L, dtype=np.float64), np.asarray(sk.R, dtype=np.float64)
rre = [r.rre for r in rec.records]
for t in range(1, len(facs)):
    ref = orc.nenmf(w.X, facs[t - 1][0], facs[t - 1][1], L=L, R=R, max_outer=1, max_iter=w.inner)
    G, F = facs[t]
    print(f"outer {t}: rre gpu {rre[t]:.6e} oracle {ref.records[-1][1]:.6e}  "
          f"G rel {np.linalg.norm(G - ref.G) / np.linalg.norm(ref.G):.3e}  "
          f"F rel {np.linalg.norm(F - ref.F) / np.linalg.norm(ref.F):.3e}  "
          f"inner iters {[(i.iterations, i.returned) for i in ref.solves] if hasattr(ref, 'solves') else ''}",
          flush=True)
