"""Time the explicit residual ||X - G F||^2 (RRE emit) and the two-candidate
tie-break forms at cfg2 shape."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _ops, _lib
n, m, p = 10000, 10000, 20
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.rand((n, m), device="cuda", generator=g)
Gt = torch.rand((p, n), device="cuda", generator=g)
F = torch.rand((p, m), device="cuda", generator=g)
out = torch.zeros(1, dtype=torch.float64, device="cuda")
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 10
ms = t(lambda: _ops.residual_sumsq(X, Gt, F, out))
ref = float(((X.double() - Gt.double().T @ F.double()) ** 2).sum())
print(f"residual_sumsq {ms*1e3:.1f} us ({n*m*4/ms/1e6:.0f} GB/s), rel err {abs(float(out[0]) - ref) / ref:.2e}")
