"""Prologue time and power-iteration count of the solves inside the compressed
outer loop at cfg2 (NENMF_NNLS_TRACE; the trace holds the last solve)."""
import os, sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["NENMF_NNLS_TRACE"] = "1"
import numpy as np
import torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, _lib
w = workloads.make_workload(2, dtype="fp32")
Xd = torch.from_numpy(w.X.astype(np.float32)).cuda()
G0 = torch.from_numpy(w.G0.astype(np.float32)).cuda()
F0 = torch.from_numpy(w.F0.astype(np.float32)).cuda()
sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
lib = _lib.load_library()
N = 4 * 4096
buf = (ctypes.c_ulonglong * N)()
for outer in (1, 2, 5, 20, 60, 100):
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                         max_outer_iterations=outer, trace_every=outer)
    nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True)
    torch.cuda.synchronize()
    lib.nenmf_debug_nnls_trace(ctypes.addressof(buf), N)
    t = np.array(buf[:], dtype=np.int64).reshape(4, 4096)
    base = t[1, 60]
    print(f"after {outer} outer: last solve prologue {(t[1, 63] - base) / 1e3:.1f} us, power iterations {t[1, 75]}, "
          f"end {(t[1, 70] - base) / 1e3:.1f} us; power done {(t[1,71]-base)/1e3:.1f}", flush=True)
