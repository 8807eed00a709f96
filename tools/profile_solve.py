"""One compressed G-half solve at cfg2 size (for ncu launch lists / full captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1812_04315_b200 import workloads, _lib, _ops
from paper_1812_04315_b200.compression import rsi_device, compress_device

dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = workloads.make_workload(2, dtype=dtype)
Xd = _lib.to_device(w.X, dtype)
L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
XL, XRt = compress_device(Xd, L, Rt)
Fd = _lib.to_device(w.F0, dtype)
FR = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
_ops.abt(Fd, Rt, FR)
Gt = _lib.to_device(w.G0.T.copy(), dtype)
Gout = torch.empty_like(Gt)
status = _lib.new_status()
for _ in range(reps):
    status.zero_()
    _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0, status=status)
torch.cuda.synchronize()
s = _lib.read_status(status)[0]
print("inner", s["inner_iters"], "L", s["lipschitz"], "best", s["returned_best"])
