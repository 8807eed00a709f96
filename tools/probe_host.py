"""Host issue rate vs device time of the compressed outer loop at cfg2 (development aid):
is the step bound by the GPU or by the Python/C-ABI issue path?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, factorize

w = workloads.make_workload(2, dtype="fp32")
Xd = torch.from_numpy(w.X.astype(np.float32)).cuda()
G0 = torch.from_numpy(w.G0.astype(np.float32)).cuda()
F0 = torch.from_numpy(w.F0.astype(np.float32)).cuda()
OUT = 100
cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                     max_outer_iterations=OUT, trace_every=OUT)
stamps = []
orig = factorize._DeviceLoop.half_steps
def hs(self, t, icfg):
    orig(self, t, icfg)
    stamps.append(time.perf_counter())
factorize._DeviceLoop.half_steps = hs
sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
for rep in range(3):
    stamps.clear()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg, return_device=True)
    b.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d = np.diff(np.array(stamps)) * 1e6
    print(f"rep {rep}: device {a.elapsed_time(b):.2f} ms, host {1e3*(t1-t0):.2f} ms, "
          f"issue interval per outer iter: median {np.median(d):.1f} us, first {d[:3].round(1)}, "
          f"host done issuing at {1e3*(stamps[-1]-t0):.2f} ms; first stamp at {1e3*(stamps[0]-t0):.2f} ms; "
          f"max interval {d.max():.1f} us at {int(d.argmax())}", flush=True)
# inner iterations of the loop's solves (status slots read by drain())
from paper_1812_04315_b200 import _lib
seen = []
orig_rs = _lib.read_status
def rs(buf):
    out = orig_rs(buf)
    seen.append(out)
    return out
_lib.read_status = rs
factorize._lib.read_status = rs
cfg1 = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                      max_outer_iterations=20, trace_every=1)
nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg1, return_device=True)
its = [int(s["inner_iters"]) for arr in seen for s in arr if int(s["inner_iters"]) > 0]
print("inner iters per solve (first 20 outer, G/F alternating):", its[:40])
for outer in (1, 2, 10):
    cfg0 = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                          max_outer_iterations=outer, trace_every=max(outer, 1))
    nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg0, return_device=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    nm.factorize_compressed(Xd, sk, nm.FactorPair(G=G0, F=F0, p=w.p), cfg0, return_device=True)
    b.record(); torch.cuda.synchronize()
    print(f"outer={outer}: {a.elapsed_time(b):.2f} ms", flush=True)
