import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1812_04315_b200 import workloads, _lib, _ops
from paper_1812_04315_b200.compression import rsi_device, sketch_draws
w = workloads.make_workload(2, dtype="fp32")
Xd = _lib.to_device(w.X, "fp32")
om_l, om_r = sketch_draws(w.n, w.m, w.nu, w.sketch_seed)
olt = _lib.to_device(np.ascontiguousarray(om_l.T), "fp32"); orr = _lib.to_device(om_r, "fp32")
L = torch.empty((w.nu, w.n), device="cuda"); Rt = torch.empty((w.nu, w.m), device="cuda"); st = _lib.new_status()
for _ in range(3):
    _ops.rsi(Xd, olt, orr, w.q, L, Rt, st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); t0 = time.perf_counter()
_ops.rsi(Xd, olt, orr, w.q, L, Rt, st)
t1 = time.perf_counter(); b.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0):.2f} ms, gpu {a.elapsed_time(b):.2f} ms, wall {1e3*(t2-t0):.2f} ms")
# QR alone
Yt = L.clone()
torch.cuda.synchronize(); a.record(); t0 = time.perf_counter()
for _ in range(10): _ops.orthonormalize(Yt, st)
t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
print(f"10 QR: host {1e3*(t1-t0):.2f} ms gpu {a.elapsed_time(b):.2f} ms")
Zt = torch.empty((w.nu, w.m), device="cuda")
torch.cuda.synchronize(); a.record(); t0 = time.perf_counter()
for _ in range(10): _ops.dual_pass(Xd, Rt, L, Yt, Zt)
t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
print(f"10 dual: host {1e3*(t1-t0):.2f} ms gpu {a.elapsed_time(b):.2f} ms")
