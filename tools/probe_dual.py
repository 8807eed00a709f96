"""Time the FP32 tensor-core X-pass (k_dual_bulk over the prepared X) alone, L2 flushed between
launches, at the BASELINE shapes; with NENMF_DUAL_DBG=1 (no MMAs) / 2 (no X copies) the same
launch shows the copy-only / MMA-only time (results invalid).  Development aid.

  python tools/probe_dual.py [cfg2|cfg3|cfg4|n m nu] ...
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1812_04315_b200 import _ops

SHAPES = {"cfg2": (10000, 10000, 30), "cfg3": (50000, 20000, 60), "cfg4": (400000, 2000, 40),
          "cfg5s": (25000, 100000, 30), "k16": (10000, 10000, 16)}


def run(n, m, nu, reps=20, check=True):
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.rand((n, m), device="cuda", generator=g)
    L = torch.randn((nu, n), device="cuda", generator=g)
    Rt = torch.randn((nu, m), device="cuda", generator=g)
    Yt = torch.empty((nu, n), device="cuda")
    Zt = torch.empty((nu, m), device="cuda")
    Xp = _ops.prepare_x(X, nu)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        _ops.dual_pass_prepared(Xp, n, m, Rt, L, Yt, Zt)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _ops.dual_pass_prepared(Xp, n, m, Rt, L, Yt, Zt)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    out = {"n": n, "m": m, "nu": nu, "dbg": os.environ.get("NENMF_DUAL_DBG", "0"),
           "k32": os.environ.get("NENMF_DUAL_K32") is not None,
           "us_split+pass+slabs": round(us, 1), "gbps": round(4.0 * n * m / us / 1e3, 1)}
    if check and os.environ.get("NENMF_DUAL_DBG") is None:
        rows = min(n, 4096)
        Y64 = Rt.double() @ X[:rows].double().T
        out["rel_err_Y"] = float((Yt[:, :rows].double() - Y64).abs().max() / Y64.abs().max())
        Z64 = torch.zeros((nu, m), dtype=torch.float64, device="cuda")
        for r0 in range(0, n, 8192):
            Z64 += L[:, r0:r0 + 8192].double() @ X[r0:r0 + 8192].double()
        out["rel_err_Z"] = float((Zt.double() - Z64).abs().max() / Z64.abs().max())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:] or ["cfg2"]
    if args[0] in SHAPES:
        for a in args:
            run(*SHAPES[a])
    else:
        run(int(args[0]), int(args[1]), int(args[2]))
