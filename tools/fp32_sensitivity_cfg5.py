"""cfg5 proxy (10^4 x 10^4, noiseless rank 16, p' = 26): how far the reference algorithm run in
float32 NumPy leaves its float64 run in ONE outer iteration, iteration by iteration (each float32
step starts from the float64 factors of the iteration before).  CPU only."""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO)); sys.path.insert(0, str(REPO / "oracle"))
import nenmf_oracle as orc
from paper_1812_04315_b200 import workloads

w = workloads.make_workload(5, n=10000, m=10000)
L, R = orc.rsi(w.X, w.nu, w.q, w.sketch_seed)
f64 = orc.nesterov_nnls


def nn32(A, B, F0, max_iter=500, grad_tol=1e-4, lipschitz_safety=1.0, info=None):
    A = A.astype(np.float32); B = B.astype(np.float32); F0 = F0.astype(np.float32)
    W = A.T @ A; V = A.T @ B
    lip = np.float32(orc.sigma_max_sq(A.astype(np.float64)))
    start = F0.copy(); g = W @ start - V
    best, best_part = None, 0.5 * (float(np.vdot(start, g)) - float(np.vdot(start, V)))
    pg_ref = orc.kkt_norm(start.astype(np.float64), g.astype(np.float64))
    f_old, g_old = start.copy(), g.copy(); y, gy = start.copy(), g.copy(); alpha = 1.0
    for k in range(max_iter):
        f = np.maximum(y + gy / (-lip), np.float32(0)); gn = W @ f - V
        pg = orc.kkt_norm(f.astype(np.float64), gn.astype(np.float64))
        part = 0.5 * (float(np.vdot(f.astype(np.float64), gn.astype(np.float64)))
                      - float(np.vdot(f.astype(np.float64), V.astype(np.float64))))
        if part < best_part: best_part, best = part, f.copy()
        if pg <= grad_tol * pg_ref: break
        a1 = orc.next_alpha(alpha); ww = np.float32((alpha - 1.0) / a1)
        y = (f - f_old) * ww + f; gy = (gn - g_old) * ww + gn; f_old, g_old = f, gn; alpha = a1
    if best is None: return start.astype(np.float64)
    rb = orc.half_sq_residual(A.astype(np.float64), B.astype(np.float64), best.astype(np.float64))
    rs = orc.half_sq_residual(A.astype(np.float64), B.astype(np.float64), start.astype(np.float64))
    return (best if rb <= rs else start).astype(np.float64)


G, F = w.G0.copy(), w.F0.copy()
for t in range(1, 4):
    orc.nesterov_nnls = f64
    r64 = orc.nenmf(w.X, G, F, L=L, R=R, max_outer=1, max_iter=w.inner)
    orc.nesterov_nnls = nn32
    r32 = orc.nenmf(w.X, G, F, L=L, R=R, max_outer=1, max_iter=w.inner)
    print(f"outer {t}: float32 NumPy vs float64, one step: G rel "
          f"{np.linalg.norm(r32.G - r64.G) / np.linalg.norm(r64.G):.3e}  F rel "
          f"{np.linalg.norm(r32.F - r64.F) / np.linalg.norm(r64.F):.3e}  rre {r32.records[-1][1]:.6e} vs {r64.records[-1][1]:.6e}",
          flush=True)
    G, F = r64.G, r64.F
