"""The host logic of the multi-GPU compressed loop (factorize._GroupDeviceLoop
in its real, one-process-per-rank mode) at world size 2 on CPU with gloo.

On the GPU every rank's half-step is one nenmf_solve_nnls_group launch that
exchanges the per-iteration decision sums with its peers inside the kernel.
Here that launch is replaced by a NumPy stand-in with the SAME contract: each
rank runs the reference's Nesterov iteration (oracle/nenmf_oracle.py) on its
own columns, and the global quantities of nnls.py:177-227 (the start point's
partial objective and PG norm, every iteration's PG norm and partial
objective, the tie-break residuals) are all-reduced every time, so both ranks
take the same decisions; the partial next product is returned per rank.
Everything else -- the row/column partition, the replicated F R, the
all-reduces of L G and F R, the all-gathers of F at emits and of G at the
end, the all-reduced RRE -- is the product code.  World 2 must reproduce the
oracle's single-process trajectory and factors (fp64, 1e-10)."""
import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _group_solve_numpy(dist, At, B, F0, Fout, *, max_iter, grad_tol, lipschitz_safety, status, group,
                       status_index=0, next_bt=None, next_out=None):
    """nenmf_solve_nnls_group's contract on CPU: this rank's columns, global
    decisions through all-reduces (nnls.py:119-227 restated by the oracle)."""
    import torch

    import nenmf_oracle as orc

    A = At.numpy().T                      # r x p
    Bl, Fl = B.numpy(), F0.numpy()
    W, V = A.T @ A, A.T @ Bl
    lip = lipschitz_safety * orc.sigma_max_sq(A)

    def allsum(*vals):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t)
        return t.tolist()

    start = Fl.copy()
    g0 = W @ start - V
    pg2, fg, fv = allsum(float((np.where(start > 0, g0, np.minimum(g0, 0)) ** 2).sum()),
                         float(np.vdot(start, g0)), float(np.vdot(start, V)))
    pg_ref, best_part = np.sqrt(pg2), 0.5 * (fg - fv)
    f_old, g_old, y, gy = start.copy(), g0.copy(), start.copy(), g0.copy()
    best, alpha = None, 1.0
    for _ in range(max_iter):
        f = np.maximum(y + gy / (-lip), 0.0)
        g = W @ f - V
        pg2, fg, fv = allsum(float((np.where(f > 0, g, np.minimum(g, 0)) ** 2).sum()),
                             float(np.vdot(f, g)), float(np.vdot(f, V)))
        part = 0.5 * (fg - fv)
        if part < best_part:
            best_part, best = part, f.copy()
        if np.sqrt(pg2) <= grad_tol * pg_ref:
            break
        a1 = orc.next_alpha(alpha)
        w = (alpha - 1.0) / a1
        y, gy = (f - f_old) * w + f, (g - g_old) * w + g
        f_old, g_old, alpha = f, g, a1
    out = start
    if best is not None:
        rb, rs = allsum(float(np.linalg.norm(A @ best - Bl) ** 2), float(np.linalg.norm(A @ start - Bl) ** 2))
        out = best if 0.5 * rb <= 0.5 * rs else start
    Fout.copy_(torch.from_numpy(out))
    if next_bt is not None:
        next_out[0].copy_(torch.from_numpy(out @ next_bt.numpy().T))


def _worker(rank, world, port, X, Lfull, Rfull, G0, F0, outer, inner, out_dir):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "oracle"))
    import torch
    import torch.distributed as dist

    from paper_1812_04315_b200 import _lib, _ops, factorize, sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = sharded.Comm()

    # --- CPU stand-ins for the device layer (the product's host logic is unchanged)
    class _Stream:
        def synchronize(self):
            pass

    class _TorchShim:
        float64 = torch.float64
        float32 = torch.float32

        class cuda:  # noqa: N801
            @staticmethod
            def current_stream():
                return _Stream()

        empty = staticmethod(lambda *a, **k: torch.empty(*a, **{kk: v for kk, v in k.items() if kk != "device"}))
        empty_like = staticmethod(torch.empty_like)
        sum = staticmethod(torch.sum)

    _lib.require_device = lambda: (None, _TorchShim)
    _lib.zeros = lambda shape, dtype: torch.zeros(shape, dtype=dtype)
    _lib.zero_ = lambda t: t.zero_() if isinstance(t, torch.Tensor) else t.fill(0)
    _lib.new_status = lambda count=1: np.zeros(count, dtype=_lib.STATUS_FIELDS)
    _lib.read_status = lambda buf: buf
    _lib.to_device = lambda a, dtype: (a.clone() if isinstance(a, torch.Tensor)
                                       else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)))
    _lib.to_host = lambda t: t.detach().double().numpy()
    _ops.abt = lambda A, B, out: out.copy_(A @ B.T)
    _ops.sumsq = lambda M, out, g=None: out.add_(float((M.double() ** 2).sum()))
    _ops.residual_sumsq = lambda X, Gt, F, out, Xp=None: out.add_(float(((X - Gt.T @ F) ** 2).sum()))
    _ops.solve_group = lambda *a, **k: _group_solve_numpy(dist, *a, **k)
    factorize._panel_t = lambda G, dtype: torch.from_numpy(np.ascontiguousarray(np.asarray(G).T))

    class _Group:
        def __init__(self):
            self.ranks, self.rank, self.nvr = world, rank, 1

        def struct(self, col0):
            return col0

    n, m = X.shape
    r0, nr = sharded.row_block(n, world, rank)
    Xl = torch.from_numpy(np.ascontiguousarray(X[r0:r0 + nr]))
    L_l = torch.from_numpy(np.ascontiguousarray(Lfull[:, r0:r0 + nr]))
    Rt = torch.from_numpy(np.ascontiguousarray(Rfull.T))
    XL = torch.from_numpy(Lfull @ X)
    XRt_l = torch.from_numpy(np.ascontiguousarray((X @ Rfull).T[:, r0:r0 + nr]))
    init = factorize.FactorPair(G=G0, F=F0, p=G0.shape[1])
    run = factorize._GroupDeviceLoop(Xl, n, r0, init, L_l, Rt, XL, XRt_l, _Group(), comm)
    run.torch = _TorchShim
    cfg = factorize.OuterConfig(inner=factorize.InnerSolverConfig(max_iter=inner), time_budget_seconds=0.0,
                                max_outer_iterations=outer)
    recs = []
    out = factorize._run_outer(None, init, cfg, lambda r, G, F: recs.append(r.rre), None, None, "fp64",
                               run=run)
    if rank == 0:
        np.savez(Path(out_dir) / "w.npz", G=np.asarray(out.G), F=np.asarray(out.F), rre=np.array(recs))
    dist.barrier()
    dist.destroy_process_group()


def test_group_loop_world2_matches_oracle():
    import torch.multiprocessing as mp

    sys.path.insert(0, str(REPO / "oracle"))
    import nenmf_oracle as orc

    rng = np.random.default_rng(8)
    n, m, p, nu = 61, 47, 4, 8
    X = rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))
    Lr, Rr = orc.rsi(X, nu, 2, 5)
    G0, F0 = rng.random((n, p)) + 0.05, rng.random((p, m)) + 0.05
    outer, inner = 4, 60
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), X, Lr, Rr, G0, F0, outer, inner, d), nprocs=2, join=True)
        got = dict(np.load(Path(d) / "w.npz"))
    ref = orc.nenmf(X, G0, F0, L=Lr, R=Rr, max_outer=outer, max_iter=inner)
    exp = np.array([r for _, r, _ in ref.records])
    np.testing.assert_allclose(got["rre"], exp, rtol=1e-10)
    np.testing.assert_allclose(got["G"], ref.G, rtol=1e-9, atol=1e-10 * np.abs(ref.G).max())
    np.testing.assert_allclose(got["F"], ref.F, rtol=1e-9, atol=1e-10 * np.abs(ref.F).max())
