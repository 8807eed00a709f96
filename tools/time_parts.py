"""Warm CUDA-event timings of the pieces of one cfg2 step (fp32)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1812_04315_b200 import _lib, _ops, workloads
from paper_1812_04315_b200.compression import rsi_device, compress_device, sketch_draws

w = workloads.make_workload(2, dtype="fp32")
X = torch.from_numpy(w.X.astype(np.float32)).cuda()
n, m, p, nu = w.n, w.m, w.p, w.nu
F = torch.rand((p, m), device="cuda"); Gt = torch.rand((p, n), device="cuda")
L, Rt, st = rsi_device(X, nu, w.q, w.sketch_seed)
XL, XRt = compress_device(X, L, Rt)
FR = torch.empty((p, nu), device="cuda")
out = torch.zeros(4, dtype=torch.float64, device="cuda")
status = _lib.new_status()
Yt = torch.empty((nu, n), device="cuda"); Zt = torch.empty((nu, m), device="cuda")
P = torch.randn((nu, n), device="cuda")

def ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

def solve(mi):
    def f():
        status.zero_()
        _ops.solve(FR, XRt, Gt, Gt, trans_b=False, max_iter=mi, grad_tol=1e-12, lipschitz_safety=1.0, status=status)
    return f
res = {
    "abt F.R^T (K=m)": ev(lambda: _ops.abt(F, Rt, FR)),
    "solve max_iter=1": ev(solve(1)),
    "solve max_iter=500": ev(solve(500), 5),
    "dual pass": ev(lambda: _ops.dual_pass(X, Rt, L, Yt, Zt)),
    "orthonormalize nu x n": ev(lambda: _ops.orthonormalize(P, status)),
    "residual_sumsq (emit)": ev(lambda: _ops.residual_sumsq(X, Gt, F, out[0:1]), 5),
    "sumsq X": ev(lambda: _ops.sumsq(X, out[1:2])),
    "rsi_device total": ev(lambda: rsi_device(X, nu, w.q, w.sketch_seed), 3),
    "X != 0 any": ev(lambda: (X != 0).any()),
}
t = time.perf_counter()
for _ in range(5): sketch_draws(n, m, nu, w.sketch_seed)
res["host omega draws"] = (time.perf_counter() - t) / 5 * 1e6
for k, v in res.items(): print(f"{k:28s} {v:9.1f} us")
