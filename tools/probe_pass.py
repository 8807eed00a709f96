"""Time the FP32 RSI pieces at cfg2 (development aid, not the bench)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1812_04315_b200 import _lib, _ops, workloads
from paper_1812_04315_b200.compression import rsi_device

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
m = int(sys.argv[2]) if len(sys.argv) > 2 else n
nu = int(sys.argv[3]) if len(sys.argv) > 3 else 30
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.rand((n, m), device="cuda", generator=g)
L = torch.randn((nu, n), device="cuda", generator=g)
Rt = torch.randn((nu, m), device="cuda", generator=g)
Yt = torch.empty((nu, n), device="cuda"); Zt = torch.empty((nu, m), device="cuda")
Xp = _ops.prepare_x(X, nu)
ms = timeit(lambda: _ops.prepare_x(X, nu), 5)
print(f"prepare_x {ms:.4f} ms  ({2*n*m*4/ms/1e6:.0f} GB/s r+w)")
ms = timeit(lambda: _ops.dual_pass_prepared(Xp, n, m, Rt, L, Yt, Zt), 20)
print(f"dual_pass_prepared {ms:.4f} ms  ({n*m*4/ms/1e6:.0f} GB/s)")
Y64 = (Rt.double() @ X.double().T); Z64 = (L.double() @ X.double())
print("rel err Y", float((Yt.double() - Y64).abs().max() / Y64.abs().max()),
      "Z", float((Zt.double() - Z64).abs().max() / Z64.abs().max()))
ms = timeit(lambda: _ops.dual_pass(X, Rt, L, Yt, Zt), 5)
print(f"dual_pass (prepare+pass) {ms:.4f} ms")
om_l = torch.randn((nu, m), device="cuda", generator=g); om_r = torch.randn((nu, n), device="cuda", generator=g)
st = _lib.new_status()
ms = timeit(lambda: _ops.rsi(X, om_l, om_r, 4, L, Rt, st, Xp=Xp), 5)
print(f"rsi q=4 prepared {ms:.4f} ms")
ms = timeit(lambda: _ops.orthonormalize(Yt, st), 5)
print(f"orthonormalize {nu}x{n} {ms:.4f} ms")
