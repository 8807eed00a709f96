"""Quick device timing probe (development aid, not the bench)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import workloads, _lib, _ops
from paper_1812_04315_b200.compression import rsi_device

def ev():
    return torch.cuda.Event(enable_timing=True)

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for dtype in ("fp32", "fp64"):
    t0 = time.time()
    w = workloads.make_workload(cfg, dtype=dtype)
    print(f"gen {time.time()-t0:.1f}s", flush=True)
    Xd = _lib.to_device(w.X, dtype)
    ms = timeit(lambda: rsi_device(Xd, w.nu, w.q, w.sketch_seed))
    nbytes = workloads.rsi_bytes(w.n, w.m, w.q, Xd.element_size())
    print(f"cfg{cfg} {dtype} RSI {ms:.3f} ms  -> {nbytes/ms/1e6:.1f} GB/s", flush=True)
    L, Rt, st = rsi_device(Xd, w.nu, w.q, w.sketch_seed)
    At = Rt  # any k x m operand
    Yt = torch.empty((w.nu, w.n), dtype=Xd.dtype, device="cuda")
    Zt = torch.empty((w.nu, w.m), dtype=Xd.dtype, device="cuda")
    ms = timeit(lambda: _ops.dual_pass(Xd, Rt, L, Yt, Zt))
    print(f"  dual pass {ms:.3f} ms -> {w.n*w.m*Xd.element_size()/ms/1e6:.1f} GB/s", flush=True)
    st = _lib.new_status()
    ms = timeit(lambda: _ops.orthonormalize(Yt, st))
    print(f"  QR n x nu {ms:.3f} ms", flush=True)
    sk = nm.SketchPair(_lib.to_host(L), _lib.to_host(Rt).T.copy(), w.nu, nm.SUBSPACE_ITERATION, w.q, w.sketch_seed)
    init = nm.FactorPair(G=w.G0, F=w.F0, p=w.p)
    for outer in (1, 5):
        cfgo = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=w.inner), time_budget_seconds=0.0,
                              max_outer_iterations=outer, trace_every=outer)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        nm.factorize_compressed(Xd, sk, init, cfgo, return_device=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"  compressed {outer} outer: {dt*1e3:.1f} ms ({outer/dt:.1f} it/s)", flush=True)
    # one solve timing
    rep = []
    status = _lib.new_status()
    FR = torch.empty((w.p, w.nu), dtype=Xd.dtype, device="cuda")
    Fd = _lib.to_device(w.F0, dtype)
    _ops.abt(Fd, Rt, FR)
    XL = torch.empty((w.nu, w.m), dtype=Xd.dtype, device="cuda"); XRt = torch.empty((w.nu, w.n), dtype=Xd.dtype, device="cuda")
    _ops.compress(Xd, L, Rt, XL, XRt)
    Gt = _lib.to_device(w.G0.T.copy(), dtype); Gout = torch.empty_like(Gt)
    def solve():
        status.zero_()
        _ops.solve(FR, XRt, Gt, Gout, trans_b=False, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0, status=status)
    ms = timeit(solve)
    s = _lib.read_status(status)[0]
    print(f"  G-half solve {ms:.3f} ms, inner iters {s['inner_iters']}, {ms*1e3/max(1,s['inner_iters']):.2f} us/iter", flush=True)
    def vsolve():
        status.zero_()
        _ops.solve(Fd, Xd, Gt, Gout, trans_b=True, max_iter=w.inner, grad_tol=1e-4, lipschitz_safety=1.0, status=status)
    ms = timeit(vsolve, reps=1)
    s = _lib.read_status(status)[0]
    print(f"  vanilla G-half solve {ms:.3f} ms, inner iters {s['inner_iters']}", flush=True)
