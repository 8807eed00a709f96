import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
mi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p, nu, c = 20, 30, 10000
torch.manual_seed(0)
FR = torch.rand((p, nu), device="cuda"); XRt = torch.rand((nu, c), device="cuda")
Gt = torch.rand((p, c), device="cuda"); Go = torch.empty_like(Gt); st = _lib.new_status()
for _ in range(3):
    st.zero_()
    _ops.solve(FR, XRt, Gt, Go, trans_b=False, max_iter=mi, grad_tol=1e-12, lipschitz_safety=1.0, status=st)
torch.cuda.synchronize()
print(_lib.read_status(st)[0])
