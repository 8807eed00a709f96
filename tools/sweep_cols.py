"""us per inner iteration of the persistent solver vs number of columns (fp32, p=20)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tdt = _lib.torch_dtype(dtype)
for c in [148, 1184, 2368, 4736, 7104, 10000, 13000]:
    torch.manual_seed(0)
    nu = 30
    FR = torch.rand((p, nu), dtype=tdt, device="cuda"); XRt = torch.rand((nu, c), dtype=tdt, device="cuda")
    Gt = torch.rand((p, c), dtype=tdt, device="cuda"); Gout = torch.empty_like(Gt); st = _lib.new_status()
    def run(mi):
        st.zero_()
        _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=mi, grad_tol=1e-12, lipschitz_safety=1.0, status=st)
    res = []
    for mi in (100, 500):
        run(mi); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): run(mi)
        b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 5)
    it = _lib.read_status(st)[0]["inner_iters"]
    print(f"c={c:6d} t100={res[0]:.3f} ms t500={res[1]:.3f} ms  marginal {(res[1]-res[0])/400*1e3:.3f} us/iter  fixed {(res[0] - (res[1]-res[0])/4):.3f} ms  iters {it}")
