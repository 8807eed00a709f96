"""Time ||X - G F||^2 on the GPU: the tensor-core pass over the prepared X
(k_resid_bulk) against the CUDA-core pass over the raw X (k_resid_pipe), and
the tie-break pair, with CUDA events; prints one JSON line per variant with
the achieved X bandwidth (algorithmic bytes: 4 per X element, the prepared
copy being the same size).

  python tools/time_resid.py --n 10000 --m 10000 --p 20
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--m", type=int, default=10000)
    ap.add_argument("--p", type=int, default=20)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_1812_04315_b200 import _lib, _ops

    torch.manual_seed(0)
    n, m, p = a.n, a.m, a.p
    G = torch.rand(p, n, device="cuda")
    F = torch.rand(p, m, device="cuda")
    X = (G.t() @ F + 0.01 * torch.rand(n, m, device="cuda")).contiguous()
    Xp = _ops.prepare_x(X, p)
    out = _lib.zeros(2, torch.float64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = float(((X.double() - G.double().t() @ F.double()) ** 2).sum())

    def timed(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        return ts[len(ts) // 2]

    xbytes = 4.0 * n * m
    for name, fn in (("prepared", lambda: _ops.residual_sumsq(X, G, F, out, Xp=Xp)),
                     ("raw", lambda: _ops.residual_sumsq(X, G, F, out))):
        us = timed(fn)
        val = float(out[0].item())
        print(json.dumps({"variant": name, "n": n, "m": m, "p": p, "us": round(us, 2),
                          "x_gbps": round(xbytes / us / 1e3, 1), "rel_err_vs_fp64": abs(val - ref) / ref}))


if __name__ == "__main__":
    main()
