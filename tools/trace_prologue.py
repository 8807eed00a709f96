import ctypes, os, sys
from pathlib import Path
os.environ["NENMF_NNLS_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1812_04315_b200 import _lib, _ops
lib = _lib.load_library()
mi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p, nu, c = 20, 30, 10000
torch.manual_seed(0)
FR = torch.rand((p, nu), device="cuda"); XRt = torch.rand((nu, c), device="cuda")
Gt = torch.rand((p, c), device="cuda"); Go = torch.empty_like(Gt); st = _lib.new_status()
for _ in range(3):
    st.zero_()
    _ops.solve(FR, XRt, Gt, Go, trans_b=False, max_iter=mi, grad_tol=1e-12, lipschitz_safety=1.0, status=st)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 4096))()
lib.nenmf_debug_nnls_trace(ctypes.addressof(buf), 4 * 4096)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4, 4096).astype(np.int64)[1, 60:75]
names = ["start", "At/Bs", "W", "prologue", "recomputed", "-", "bar1", "resid", "sync", "gridbar", "end", "power", "bj read", "kd read", "resolver done"]
for i, nme in enumerate(names):
    if t[i]: print(f"{nme:10s} {(t[i]-t[0])/1e3:8.2f} us")
print(_lib.read_status(st)[0])
raw = np.frombuffer(buf, dtype=np.uint64).reshape(4, 4096).astype(np.int64)[1]
print('best_j', raw[80], 'kdone', raw[81])
