import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
dtype = sys.argv[1]
torch.manual_seed(0)
tdt = _lib.torch_dtype(dtype)
p, nu, c = 20, 30, 10000
FR = torch.rand((p, nu), dtype=tdt, device="cuda")
XRt = torch.rand((nu, c), dtype=tdt, device="cuda")
Gt = torch.rand((p, c), dtype=tdt, device="cuda")
Gout = torch.empty_like(Gt)
st = _lib.new_status()
def run():
    st.zero_()
    _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=500, grad_tol=1e-12, lipschitz_safety=1.0, status=st)
run(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): run()
b.record(); torch.cuda.synchronize()
s = _lib.read_status(st)[0]
print(f"{a.elapsed_time(b)/3:.3f} ms iters {s['inner_iters']} -> {a.elapsed_time(b)/3*1e3/max(1,s['inner_iters']):.2f} us/iter")
