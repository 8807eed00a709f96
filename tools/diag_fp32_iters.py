import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import nenmf_oracle as orc
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, _lib, _ops
w = workloads.make_workload(2, n=4000, m=4000, dtype="fp32")
Xd = torch.from_numpy(w.X.astype(np.float32)).cuda()
sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
L, R = _lib.to_host(sk.L), _lib.to_host(sk.R)
facs = []
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=500), time_budget_seconds=0.0, max_outer_iterations=2)
init = nm.FactorPair(G=torch.from_numpy(w.G0.astype(np.float32)).cuda(), F=torch.from_numpy(w.F0.astype(np.float32)).cuda(), p=w.p)
nm.factorize_compressed(Xd, sk, init, cfg, observer=lambda r, G, F: facs.append((G.copy(), F.copy())), clock=nm.IterationClock())
XL, XR = orc.compress(w.X, L, R)
for t in (1, 2):
    G0, F0 = facs[t-1]
    # oracle G-half then F-half with info
    A = np.ascontiguousarray((F0 @ R).T); ig = orc.SolveInfo()
    Gn = orc.nesterov_nnls(A, np.ascontiguousarray(XR.T), np.ascontiguousarray(G0.T), 500, 1e-4, 1.0, ig).T
    A2 = L @ Gn; ifo = orc.SolveInfo()
    Fn = orc.nesterov_nnls(A2, XL, F0, 500, 1e-4, 1.0, ifo)
    # GPU F-half from the ORACLE's G (isolates the F solve)
    At = _lib.to_device(np.ascontiguousarray(A2.T), "fp32"); B = _lib.to_device(XL, "fp32"); Fd = _lib.to_device(F0, "fp32")
    Fo = torch.empty_like(Fd); st = _lib.new_status()
    _ops.solve(At, B, Fd, Fo, trans_b=False, max_iter=500, grad_tol=1e-4, lipschitz_safety=1.0, status=st)
    s = _lib.read_status(st)[0]
    Fg = _lib.to_host(Fo)
    print(t, "oracle G iters", ig.iterations, ig.returned, "F iters", ifo.iterations, ifo.returned, "| gpu F iters", int(s["inner_iters"]), int(s["returned_best"]),
          "Fdiff(same inputs)", np.linalg.norm(Fg-Fn)/np.linalg.norm(Fn), flush=True)
