import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import nenmf_oracle as orc
from paper_1812_04315_b200 import workloads
w = workloads.make_workload(2, dtype="fp32")
L, R = orc.rsi(w.X, w.nu, w.q, w.sketch_seed)
ref = orc.nenmf(w.X, w.G0, w.F0, L=L, R=R, max_outer=3, max_iter=500)
print("fp64", [r for _, r, _ in ref.records], flush=True)
# the same algorithm in float32 arithmetic: run the oracle's solver on float32 arrays
import nenmf_oracle
orig = np.ascontiguousarray
def nn32(A, B, F0, max_iter=500, grad_tol=1e-4, lipschitz_safety=1.0, info=None):
    A = A.astype(np.float32); B = B.astype(np.float32); F0 = F0.astype(np.float32)
    W = A.T @ A; V = A.T @ B
    lip = np.float32(orc.sigma_max_sq(A.astype(np.float64)))
    start = F0.copy(); g = W @ start - V
    best, best_part = None, 0.5*(float(np.vdot(start, g)) - float(np.vdot(start, V)))
    pg_ref = orc.kkt_norm(start.astype(np.float64), g.astype(np.float64))
    f_old, g_old = start.copy(), g.copy(); y, gy = start.copy(), g.copy(); alpha = 1.0
    for k in range(max_iter):
        f = np.maximum(y + gy / (-lip), np.float32(0)); gn = W @ f - V
        pg = orc.kkt_norm(f.astype(np.float64), gn.astype(np.float64))
        part = 0.5*(float(np.vdot(f.astype(np.float64), gn.astype(np.float64))) - float(np.vdot(f.astype(np.float64), V.astype(np.float64))))
        if part < best_part: best_part, best = part, f.copy()
        if pg <= grad_tol * pg_ref: break
        a1 = orc.next_alpha(alpha); ww = np.float32((alpha - 1.0) / a1)
        y = (f - f_old) * ww + f; gy = (gn - g_old) * ww + gn; f_old, g_old = f, gn; alpha = a1
    if best is None: return start.astype(np.float64)
    rb = orc.half_sq_residual(A.astype(np.float64), B.astype(np.float64), best.astype(np.float64))
    rs = orc.half_sq_residual(A.astype(np.float64), B.astype(np.float64), start.astype(np.float64))
    return (best if rb <= rs else start).astype(np.float64)
orc.nesterov_nnls = nn32
r32 = orc.nenmf(w.X, w.G0, w.F0, L=L, R=R, max_outer=3, max_iter=500)
print("fp32-numpy", [r for _, r, _ in r32.records], flush=True)
print("Gdiff", np.linalg.norm(r32.G-ref.G)/np.linalg.norm(ref.G), "Fdiff", np.linalg.norm(r32.F-ref.F)/np.linalg.norm(ref.F))
