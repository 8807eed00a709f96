import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np, math
import paper_1812_04315_b200 as nm
import nenmf_oracle as orc
d = dict(np.load("tests/golden/nnls.npz"))
i = int(sys.argv[1]) if len(sys.argv) > 1 else 5
A, B, F0 = d[f"A{i}"], d[f"B{i}"], d[f"F0_{i}"]
max_iter, tol, saf, calls = d["meta"][i]
# oracle iterates
W = A.T @ A; V = A.T @ B; L = saf * orc.sigma_max_sq(A)
f_old = F0.copy(); g_old = W @ F0 - V; y, gy = F0.copy(), g_old.copy(); alpha = 1.0
its = []
for k in range(int(max_iter)):
    f = np.maximum(y + gy / (-L), 0.0); g = W @ f - V
    its.append(f.copy())
    a1 = orc.next_alpha(alpha); w = (alpha - 1) / a1
    y = (f - f_old) * w + f; gy = (g - g_old) * w + g; f_old, g_old = f, g; alpha = a1
rep = []
F = nm.solve_nnls(A, B, F0, nm.InnerSolverConfig(max_iter=int(max_iter), grad_tol=tol, lipschitz_safety=saf), report=rep)
print("report", rep)
print("diff to golden", np.abs(F - d[f"F{i}"]).max())
print("diff to F0", np.abs(F - F0).max())
for k, f in enumerate(its):
    print("diff to iterate", k, np.abs(F - f).max())
