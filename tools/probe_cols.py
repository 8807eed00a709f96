"""Inner-solver us/iter vs column count (warps per CTA / SMSP sharing); development aid."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops

torch.manual_seed(0)
p, r, it = 20, 30, 500
for c in [int(x) for x in (sys.argv[1:] or ["9472", "10000", "10064", "7400", "5000", "2368"])]:
    At = torch.rand(p, r, device="cuda")
    B = torch.rand(r, c, device="cuda")
    F0 = torch.rand(p, c, device="cuda")
    Fo = torch.empty_like(F0)
    st = _lib.new_status()
    def solve():
        st.zero_()
        _ops.solve(At, B, F0, Fo, trans_b=False, max_iter=it, grad_tol=0.0, lipschitz_safety=1.0, status=st)
    solve(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        solve()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"c={c}: {ms*1e3:.1f} us/solve {ms*1e3/it:.3f} us/iter", flush=True)
