"""Back-to-back fused solves at cfg2 (G-half, next product) timed with events,
with and without the records memset (development aid for the launch gap)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import workloads, _lib, _ops
from paper_1812_04315_b200.compression import rsi_device, compress_device
w = workloads.make_workload(2, dtype="fp32")
Xd = _lib.to_device(w.X, "fp32")
L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
XL, XRt = compress_device(Xd, L, Rt)
Fd = _lib.to_device(w.F0, "fp32")
FR = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
_ops.abt(Fd, Rt, FR)
Gt = _lib.to_device(w.G0.T.copy(), "fp32")
Gout = torch.empty_like(Gt)
GLt = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
status = _lib.new_status(64)
def run(n, nxt):
    for i in range(n):
        if nxt:
            _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                       status=status, status_index=i % 64, next_bt=L, next_out=GLt)
        else:
            _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                       status=status, status_index=i % 64)
Fo = torch.empty_like(Fd)
_ops.abt(Gt, L, GLt)
def runF(n):
    for i in range(n):
        _ops.solve(GLt, XL, Fd, Fo, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                   status=status, status_index=i % 64, next_bt=Rt, next_out=FR)
runF(3); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); runF(20); b.record(); torch.cuda.synchronize()
print(f"F-half next n=20: {1e3 * a.elapsed_time(b) / 20:.1f} us per solve", flush=True)
for nxt in (False, True):
    run(3, nxt); torch.cuda.synchronize()
    for n in (1, 20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(n, nxt); b.record(); torch.cuda.synchronize()
        print(f"next={nxt} n={n}: {1e3 * a.elapsed_time(b) / n:.1f} us per solve", flush=True)
