import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1812_04315_b200 import workloads, _lib
from paper_1812_04315_b200.compression import rsi_device
dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
w = workloads.make_workload(2, dtype=dtype)
Xd = _lib.to_device(w.X, dtype)
for _ in range(2):
    L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
b.record(); torch.cuda.synchronize()
print("rsi ms", a.elapsed_time(b))
