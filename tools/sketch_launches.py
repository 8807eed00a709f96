"""One device-resident cfg2 sketch + compression (the RSI part of bench.py's
step) inside cudaProfilerStart/Stop, after a warm-up, for an ncu launch list:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      python tools/sketch_launches.py [fp32|fp64]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import compression, workloads

dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
w = workloads.make_workload(2, dtype=dtype)
X = torch.from_numpy(w.X.astype(np.float32 if dtype == "fp32" else np.float64)).cuda()


def once():
    sk = nm.subspace_iteration_pair(X, w.nu, w.q, w.sketch_seed)
    L, Rt = sk.device[dtype]
    compression.compress_device(X, L, Rt, prepared=compression.prepared_for(sk, X))


once()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    once()
e.record()
torch.cuda.synchronize()
print(f"sketch+compress {dtype}: {s.elapsed_time(e) / 3:.3f} ms", flush=True)
torch.cuda.cudart().cudaProfilerStart()
once()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
