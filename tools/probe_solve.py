"""Inner-solver timing experiments at cfg2 (NENMF_NNLS_DBG variants; development aid)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1812_04315_b200 import workloads, _lib, _ops
from paper_1812_04315_b200.compression import rsi_device, compress_device

dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
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
def solve():
    status.zero_()
    _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0, status=status)
for dbg in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "4", "3", "7"]):
    os.environ["NENMF_NNLS_DBG"] = dbg
    solve(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        solve()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"dbg {dbg}: {ms*1e3:.1f} us per solve, {ms*1e3/w.inner:.3f} us/iter", flush=True)
