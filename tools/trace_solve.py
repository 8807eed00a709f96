import ctypes, os, sys
from pathlib import Path
os.environ["NENMF_NNLS_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1812_04315_b200 import _lib, _ops
lib = _lib.load_library()
dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
tdt = _lib.torch_dtype(dtype)
torch.manual_seed(0)
p, nu, c = 20, 30, 10000
FR = torch.rand((p, nu), dtype=tdt, device="cuda"); XRt = torch.rand((nu, c), dtype=tdt, device="cuda")
Gt = torch.rand((p, c), dtype=tdt, device="cuda"); Gout = torch.empty_like(Gt); st = _lib.new_status()
for _ in range(2):
    st.zero_()
    _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=500, grad_tol=1e-12, lipschitz_safety=1.0, status=st)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 4096))()
lib.nenmf_debug_nnls_trace(ctypes.addressof(buf), 4 * 4096)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4, 4096).astype(np.int64)
n = 501
t0 = t[0, 0]
for name, row in zip(["post0", "publish0", "resolve0", "postLast"], t):
    r = (row[:n] - t0) / 1e3
    d = np.diff(r)
    print(f"{name:9s} start {r[0]:8.2f} us  end {r[n-1]:8.2f}  median step {np.median(d):6.2f} us  p90 {np.percentile(d,90):6.2f}")
print("lag post->publish (us) median", np.median((t[1,:n]-t[0,:n])/1e3), " publish->resolve", np.median((t[2,:n]-t[1,:n])/1e3))
for k in range(0, 60, 3):
    print(k-1, [round((t[i,k]-t0)/1e3,2) for i in range(4)])
