"""One-step parity of the FP32 mode (development aid): every outer iteration
of the device path against the oracle's outer iteration from the same
factors, relative Frobenius deviation of G and F.
  python tools/onestep_fp32.py [n] [ranks (0: 1-GPU path, R: emulated R-rank group)] [outer]"""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import nenmf_oracle as orc
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, _lib, sharded
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
ranks = int(sys.argv[2]) if len(sys.argv) > 2 else 0
outer = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = workloads.make_workload(2, n=n, m=n, dtype="fp32")
Xd = torch.from_numpy(w.X.astype(np.float32)).cuda()
sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
L, R = _lib.to_host(sk.L), _lib.to_host(sk.R)
facs = []
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=500), time_budget_seconds=0.0, max_outer_iterations=outer)
init = nm.FactorPair(G=torch.from_numpy(w.G0.astype(np.float32)).cuda(), F=torch.from_numpy(w.F0.astype(np.float32)).cuda(), p=w.p)
obs = lambda r, G, F: facs.append((G.copy(), F.copy()))
if ranks:
    sharded.factorize_compressed_emulated(Xd, sk, init, cfg, observer=obs, clock=nm.IterationClock(), ranks=ranks)
else:
    nm.factorize_compressed(Xd, sk, init, cfg, observer=obs, clock=nm.IterationClock())
for t in range(1, len(facs)):
    ref = orc.nenmf(w.X, facs[t-1][0], facs[t-1][1], L=L, R=R, max_outer=1, max_iter=500)
    print(n, ranks, t, "Gdiff", np.linalg.norm(facs[t][0]-ref.G)/np.linalg.norm(ref.G), "Fdiff", np.linalg.norm(facs[t][1]-ref.F)/np.linalg.norm(ref.F), flush=True)
