"""Time V = A^T B at cfg2 vanilla shapes (both orientations) against fp64 torch."""
import os, sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _ops, _lib
n = m = 10000; p = 20
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.rand((n, m), device="cuda", generator=g)
Gt = torch.rand((p, n), device="cuda", generator=g)
F = torch.rand((p, m), device="cuda", generator=g)
out_m = torch.empty((p, m), device="cuda"); out_n = torch.empty((p, n), device="cuda")
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 10
# gradient(A, B, F) = A^T (A F - B) uses V = A^T B; time via nenmf_gradient with F = 0 -> -V
zF_m = torch.zeros((p, m), device="cuda"); zF_n = torch.zeros((p, n), device="cuda")
At_G = Gt  # A = G (n x p): At = Gt
ms = t(lambda: _ops.gradient(At_G, X, zF_m, out_m))
ref = -(Gt.double() @ X.double())
print(f"V = G^T X   (Z side) {ms*1e3:.1f} us ({n*m*4/ms/1e6:.0f} GB/s) rel err {float((out_m.double()-ref).abs().max()/ref.abs().max()):.2e}")
ms = t(lambda: _ops.gradient(F, X, zF_n, out_n, trans_b=True))
ref = -(F.double() @ X.double().T)
print(f"V = F X^T   (Y side) {ms*1e3:.1f} us ({n*m*4/ms/1e6:.0f} GB/s) rel err {float((out_n.double()-ref).abs().max()/ref.abs().max()):.2e}")
