"""Time the FP64 X-pass (Yt = At X^T, Zt = Bt X on the DMMA pipe) alone, L2 flushed between
launches; NENMF_DUAL64=off selects the two one-product kernels, =v1 the first fused kernel.

  python tools/probe_dual64.py [n m nu]
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1812_04315_b200 import _ops


def run(n, m, nu, reps=10):
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.rand((n, m), device="cuda", generator=g, dtype=torch.float64)
    L = torch.randn((nu, n), device="cuda", generator=g, dtype=torch.float64)
    Rt = torch.randn((nu, m), device="cuda", generator=g, dtype=torch.float64)
    Yt = torch.empty((nu, n), device="cuda", dtype=torch.float64)
    Zt = torch.empty((nu, m), device="cuda", dtype=torch.float64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        _ops.dual_pass(X, Rt, L, Yt, Zt)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _ops.dual_pass(X, Rt, L, Yt, Zt)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    Y64 = Rt @ X.T
    Z64 = L @ X
    print(json.dumps({"n": n, "m": m, "nu": nu, "mode": os.environ.get("NENMF_DUAL64", "default"),
                      "us": round(us, 1), "tflops": round(4.0 * n * m * nu / us / 1e6, 2),
                      "gbps": round(8.0 * n * m / us / 1e3, 1),
                      "rel_err_Y": float((Yt - Y64).abs().max() / Y64.abs().max()),
                      "rel_err_Z": float((Zt - Z64).abs().max() / Z64.abs().max())}), flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    if a:
        run(int(a[0]), int(a[1]), int(a[2]))
    else:
        run(10000, 10000, 30)
        run(10000, 10000, 20)
        run(5002, 7014, 30)
