"""Per-window timeline of one persistent solve (NENMF_NNLS_TRACE=1):
compute post of the window's last iteration (CTA 0 warp 0), publish of CTA 0's
record, resolve of the window's last iteration in CTA 0."""
import ctypes, os, sys
from pathlib import Path
os.environ["NENMF_NNLS_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1812_04315_b200 import _lib, _ops
lib = _lib.load_library()
dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
c = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
tdt = _lib.torch_dtype(dtype)
torch.manual_seed(0)
p, nu = 20, 30
FR = torch.rand((p, nu), dtype=tdt, device="cuda"); XRt = torch.rand((nu, c), dtype=tdt, device="cuda")
Gt = torch.rand((p, c), dtype=tdt, device="cuda"); Gout = torch.empty_like(Gt); st = _lib.new_status()
for _ in range(2):
    st.zero_()
    _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=500, grad_tol=1e-12, lipschitz_safety=1.0, status=st)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 4096))()
lib.nenmf_debug_nnls_trace(ctypes.addressof(buf), 4 * 4096)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4, 4096).astype(np.int64)
post, pub, res, summ = t[0, :501], t[1, :17], t[2, :501], t[3, 3072:3072 + 17]
r1 = t[1]
cyc, ns, its = r1[50] - r1[52], r1[51] - r1[53], r1[54]
print(f"warp0/CTA0 loop: {its} iters, {cyc/its:.0f} cycles/iter, {ns/its:.1f} ns/iter -> {cyc/ns*1e3:.0f} MHz")
t0 = post[post > 0].min() if (post > 0).any() else 0
us = lambda x: (x - t0) / 1e3
d = np.diff(post[1:])
print(f"c={c}: compute step median {np.median(d)/1e3:.3f} us, mean {d.mean()/1e3:.3f} us, max {d.max()/1e3:.2f} us")
print(" win  post_last   publish   summed    resolved   pub-post  sum-pub  res-sum  step-gap-at-start")
for w in range(4):
    j = 32 * w + 31
    if j + 1 >= 501: break
    gap = (post[32 * w + 1] - post[32 * w]) / 1e3 if w > 0 else float("nan")
    print(f"{w:4d} {us(post[j+1]):9.2f} {us(pub[w+1]):9.2f} {us(summ[w+1]):9.2f} {us(res[j+1]):9.2f} {(pub[w+1]-post[j+1])/1e3:9.2f} {(summ[w+1]-pub[w+1])/1e3:8.2f} {(res[j+1]-summ[w+1])/1e3:8.2f} {gap:9.2f}")

ws = t[1, 100:100 + 4 * 16].reshape(16, 4)
print("window start: prev post -> enter, enter -> after wait, wait -> after snapshot, snapshot -> first post (us)")
for w in range(1, 15):
    print(w, round((ws[w,0]-post[32*w])/1e3,2), round((ws[w,1]-ws[w,0])/1e3,2), round((ws[w,2]-ws[w,1])/1e3,2), round((post[32*w+1]-ws[w,2])/1e3,2))
