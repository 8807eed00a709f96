"""Time the device orthonormalisation (CholeskyQR2) of a k x rows panel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
k = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
P = torch.randn((k, rows), device="cuda")
st = _lib.new_status()
for _ in range(3): _ops.orthonormalize(P, st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): _ops.orthonormalize(P, st)
b.record(); torch.cuda.synchronize()
Q = P.double()
err = (Q @ Q.T - torch.eye(k, device="cuda", dtype=torch.float64)).abs().max().item()
print(f"QR k={k} rows={rows}: {a.elapsed_time(b)/20*1e3:.1f} us  |QQ^T-I|={err:.2e}")
