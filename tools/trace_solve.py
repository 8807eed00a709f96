"""Timeline of one compressed G-half solve at cfg2 (NENMF_NNLS_TRACE, CTA 0)."""
import os, sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["NENMF_NNLS_TRACE"] = "1"
import numpy as np
import torch
from paper_1812_04315_b200 import workloads, _lib, _ops
from paper_1812_04315_b200.compression import rsi_device, compress_device
DT = "fp64" if "fp64" in sys.argv else "fp32"
w = workloads.make_workload(2, dtype=DT)
Xd = _lib.to_device(w.X, DT)
L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
XL, XRt = compress_device(Xd, L, Rt)
Fd = _lib.to_device(w.F0, DT)
FR = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
_ops.abt(Fd, Rt, FR)
Gt = _lib.to_device(w.G0.T.copy(), DT)
Gout = torch.empty_like(Gt)
status = _lib.new_status()
lib = _lib.load_library()
N = 4 * 4096
buf = (ctypes.c_ulonglong * N)()
for rep in range(3):
    status.zero_()
    if "next" in sys.argv:
        GLt = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
        _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                   status=status, next_bt=L, next_out=GLt)
    else:
        _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0,
                   status=status)
    torch.cuda.synchronize()
lib.nenmf_debug_nnls_trace(ctypes.addressof(buf), N)
t = np.array(buf[:], dtype=np.int64).reshape(4, 4096)
T = 4096
base = t[1, 60 + 0]
def us(x): return (int(x) - int(base)) / 1e3
print("start->prologue done %.1f us" % us(t[1, 60 + 3]))
print("loop start %.1f, loop end %.1f (k=%d)" % (us(t[1, 53]), us(t[1, 51]), t[1, 54]))
print("after output barrier %.1f; tie-break done %.1f; end %.1f" % (us(t[1, 60 + 6]), us(t[1, 60 + 8]), us(t[1, 60 + 10])))
print("resolver done %.1f" % us(t[1, 60 + 14]))
for wdw in range(0, 16):
    a, b2, c = t[1, 100 + 4 * wdw], t[1, 100 + 4 * wdw + 1], t[1, 100 + 4 * wdw + 2]
    pub = t[1, wdw + 1] if wdw + 1 < T else 0   # row 1 = publish times of CTA 0
    res = t[2, min(32 * wdw + 31 + 1, T - 1)]   # resolve time of the window's last iteration
    sm = t[3, 3072 + wdw + 1]
    print("win %2d: start %.1f waited %.1f | published %.1f | summarized(j0) %.1f | resolved %.1f" %
          (wdw, us(a), (int(b2) - int(a)) / 1e3, us(pub) if pub else -1, us(sm) if sm else -1, us(res) if res else -1))
G = 148
def stats(name, v):
    v = np.array([us(x) for x in v])
    print("%-28s min %.1f  med %.1f  max %.1f  (argmax CTA %d)" % (name, v.min(), np.median(v), v.max(), int(v.argmax())))
stats("CTA start", t[0, :G])
stats("loop start (warp 0)", t[3, :G])
for wd in range(5):
    stats("loop end warp %d" % wd, t[3, 512 * (1 + wd): 512 * (1 + wd) + G])
stats("last window published", t[0, 512:512 + G])
stats("resolver exit", t[0, 1024:1024 + G])
for wd in range(5):
    stats("past output barrier warp %d" % wd, t[0, 512 * (3 + wd): 512 * (3 + wd) + G])
fin = t[2, 3072:3072 + G].astype(np.int64) - 1
for wd in range(5):
    seen = t[2, 512 * (1 + wd): 512 * (1 + wd) + G].astype(np.int64) - 1
    print("warp %d: best_j seen past the barrier != final in %d CTAs (final %s)" % (wd, int((seen != fin).sum()), np.unique(fin)))
print("spec path (CTA 0 warp 0): start %.1f resid %.1f partials %.1f" % tuple(us(t[1, 90 + i]) for i in range(3)))
