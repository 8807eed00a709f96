"""One cfg4 G-half solve (400000 columns, streamed SIMT solver) for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
n, p, nu = 400000, 30, 40
g = torch.Generator(device="cuda").manual_seed(0)
FR = torch.rand((p, nu), device="cuda", generator=g)
XRt = torch.rand((nu, n), device="cuda", generator=g) * 10
Gt = torch.rand((p, n), device="cuda", generator=g)
Gout = torch.empty_like(Gt)
st = _lib.new_status()
for _ in range(2):
    st.zero_()
    _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 500,
               grad_tol=1e-4, lipschitz_safety=1.0, status=st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); st.zero_()
_ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=500, grad_tol=1e-4, lipschitz_safety=1.0, status=st)
b.record(); torch.cuda.synchronize()
print(f"cfg4 G-half solve {a.elapsed_time(b):.2f} ms, inner {int(_lib.read_status(st)[0]['inner_iters'])}")
