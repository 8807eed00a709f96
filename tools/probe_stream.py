"""Streamed solver at cfg5 shape (p=16, r=26, c=1e5): resident vs HBM ring (development aid)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
torch.manual_seed(0)
p, r, c, it = 16, 26, 100000, 500
At = torch.rand(p, r, device="cuda")
B = torch.rand(r, c, device="cuda")
F0 = torch.rand(p, c, device="cuda")
Fo = torch.empty_like(F0)
st = _lib.new_status()
def solve():
    st.zero_()
    _ops.solve(At, B, F0, Fo, trans_b=False, max_iter=it, grad_tol=0.0, lipschitz_safety=1.0, status=st)
for mode in ("resident", "ring"):
    if mode == "ring":
        os.environ["NENMF_STREAM_RING"] = "1"
    solve(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        solve()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"{mode}: {ms:.3f} ms per solve, {ms * 1e3 / it:.2f} us/iter", flush=True)
