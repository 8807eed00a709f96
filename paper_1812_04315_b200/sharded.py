"""Row-sharded compressed NeNMF across GPUs.

One process per GPU (``torchrun``), X split into row blocks: rank r holds
rows [row0_r, row0_r + n_r) of X (``row_block``).  The exchange steps, all
through ``torch.distributed`` (NCCL over NVLink on GPUs), carry only the small
sketch-sized partials named by the north star:

* RSI pass (compression.py:134-139): Y = X_r A is local (this rank's rows of
  the n-panel); Z = sum_r X_r^T B_r is ONE all-reduce of the nu x m partial
  per pass (2q + 2 per sketch).
* n-panel orthonormalisation: CholeskyQR2 whose two nu x nu Gram matrices are
  all-reduced (fp64); the factorisation is replicated and identical on every
  rank; random completion columns are keyed by the global row index, so the
  shards reproduce the 1-GPU panel.
* m-panel orthonormalisation: replicated (identical input, deterministic
  kernel -> bit-identical on every rank).
* compression (compression.py:179-188): X_L = sum_r L_r X_r, one nu x m
  all-reduce; X_R stays row-local.
* factorization (factorize.py:197-213): X_R^T and L are all-gathered once
  (nu x n each) and the outer loop then runs replicated (every rank holds the
  same G and F; no per-step traffic); the reported RRE uses the sharded
  ||X_r - G_r F||^2 and ||X_r||^2, one all-reduced scalar each.

The local arithmetic goes through an ops backend: ``DeviceOps`` (the C-ABI
kernels; the product path) by default.  The CPU tests substitute a NumPy
backend to check this exchange logic with ``gloo`` at world size 2.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib, _ops
from .compression import SketchPair, SUBSPACE_ITERATION, _check_iteration_inputs, sketch_draws, sketch_draws_device
from .errors import DimensionError, raise_for_status


def row_block(n: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of rank ``rank`` in a balanced split of n rows."""
    r0 = rank * n // world
    r1 = (rank + 1) * n // world
    return r0, r1 - r0


def load_row_shard(path, world: int, rank: int, *, dtype: str = "fp32"):
    """This rank's row block of an NMFB file as a CUDA tensor, streamed from
    disk through pinned chunks; returns (X_local, n, row0)."""
    from pathlib import Path

    from .matrix import _nmfb_header, read_nmfb_device

    n, _ = _nmfb_header(path, Path(path).stat().st_size)
    row0, rows = row_block(n, world, rank)
    return read_nmfb_device(path, dtype=dtype, row0=row0, rows=rows), n, row0


class Comm:
    """The collectives of the sharded path over a torch.distributed group."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_reduce(self, t):
        if self.size > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def any(self, flag: bool) -> bool:
        """True on every rank if ``flag`` is True on any rank (MAX all-reduce)."""
        if self.size == 1:
            return bool(flag)
        torch = _lib.torch_mod()
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def all_gather_cols(self, local, n: int):
        """(k x n_r) blocks in rank order -> (k x n); ragged blocks are padded."""
        torch = _lib.torch_mod()
        if self.size == 1:
            return local
        counts = [row_block(n, self.size, r)[1] for r in range(self.size)]
        w = max(counts)
        k = local.shape[0]
        pad = torch.zeros((k, w), dtype=local.dtype, device=local.device)
        pad[:, : local.shape[1]] = local
        parts = [torch.empty_like(pad) for _ in range(self.size)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:, :c] for p, c in zip(parts, counts)], dim=1).contiguous()


class DeviceOps:
    """Local arithmetic of a shard on its GPU (libnenmf_b200 kernels)."""

    def __init__(self):
        _, self.torch = _lib.require_device()

    def tensor(self, a, like):
        return _lib.to_device(np.ascontiguousarray(a), "fp64" if like.dtype == self.torch.float64 else "fp32")

    def empty(self, shape, like, dtype=None):
        return self.torch.empty(shape, dtype=dtype or like.dtype, device=like.device)

    def prepare(self, X, k):
        return _ops.prepare_x(X, k)

    def draws(self, n, m, nu, seed, like):
        dtype = "fp64" if like.dtype == self.torch.float64 else "fp32"
        dev = sketch_draws_device(n, m, nu, seed, dtype)
        if dev is not None:
            return dev
        omega_l, omega_r = sketch_draws(n, m, nu, seed)
        return self.tensor(omega_l.T, like), self.tensor(omega_r, like), None

    def draws_ok(self, ok):
        return ok is None or bool(ok.item())

    def dual_pass(self, X, Xp, At, Bt):
        """(At X^T, Bt X): this shard's rows of X A and its partial of X^T B."""
        n, m = X.shape
        k = At.shape[0]
        Yt = self.empty((k, n), X)
        Zt = self.empty((k, m), X)
        if Xp is not None:
            _ops.dual_pass_prepared(Xp, n, m, At, Bt, Yt, Zt)
        else:
            _ops.dual_pass(X, At, Bt, Yt, Zt)
        return Yt, Zt

    def gram(self, Pt):
        k = Pt.shape[0]
        G = self.torch.empty((k, k), dtype=self.torch.float64, device=Pt.device)
        _ops.panel_gram(Pt, G)
        return G

    def factor(self, G, pivot, status):
        k = G.shape[0]
        R = self.torch.empty((k, k), dtype=self.torch.float64, device=G.device)
        meta = self.torch.empty(k + 4, dtype=self.torch.int32, device=G.device)
        _ops.panel_factor(G, pivot, R, meta, status)
        return R, meta

    def trsm(self, Pin, R, meta, Pout, row0, full_rank_only):
        _ops.panel_trsm(Pin, R, meta, Pout, row0, full_rank_only)

    def qr(self, Pt, status):
        _ops.orthonormalize(Pt, status)

    def new_status(self):
        return _lib.new_status()

    def check_status(self, status, what):
        st = _lib.read_status(status)[0]
        if st["code"] != 0:
            raise_for_status(int(st["code"]), int(st["iteration"]), what)

    def sumsq(self, X):
        out = _lib.zeros(1, self.torch.float64)
        _ops.sumsq(X, out)
        return out

    def residual_sumsq(self, X, Gt, F):
        out = _lib.zeros(1, self.torch.float64)
        _ops.residual_sumsq(X, Gt, F, out)
        return out


def _qr_rows(ops, comm: Comm, Pt, row0: int, status):
    """CholeskyQR2 of a row-sharded panel (this rank's columns Pt, k x n_r),
    in place: two Gram all-reduces, replicated factorisations."""
    Q1 = ops.empty(Pt.shape, Pt)
    G = comm.all_reduce(ops.gram(Pt))
    R, meta = ops.factor(G, True, status)
    ops.trsm(Pt, R, meta, Q1, row0, False)
    G2 = comm.all_reduce(ops.gram(Q1))
    R2, meta2 = ops.factor(G2, False, status)
    ops.trsm(Q1, R2, meta2, Pt, row0, True)
    return Pt


def _rsi_loop(X_local, q, comm, ops, row0, Olt, Orl, Xp):
    status = ops.new_status()
    # start: L = (X Omega_L)^T (local columns), R^T = Omega_R X (all-reduced)
    L, Rt = ops.dual_pass(X_local, Xp, Olt, Orl)
    comm.all_reduce(Rt)
    _qr_rows(ops, comm, L, row0, status)
    ops.qr(Rt, status)
    for _ in range(q):
        trow, tcol = ops.dual_pass(X_local, Xp, Rt, L)   # X Q_row (local), X^T Q_col (partial)
        comm.all_reduce(tcol)
        ops.qr(tcol, status)
        _qr_rows(ops, comm, trow, row0, status)
        L, Rt = ops.dual_pass(X_local, Xp, tcol, trow)
        comm.all_reduce(Rt)
        _qr_rows(ops, comm, L, row0, status)
        ops.qr(Rt, status)
    return L, Rt, status


def _rsi_with(X_local, n, nu, q, seed, comm, ops, row0, Olt, Orl, Xp):
    L, Rt, status = _rsi_loop(X_local, q, comm, ops, row0, Olt, Orl, Xp)
    ops.check_status(status, "subspace iteration")
    return ShardedSketch(L_local=L, Rt=Rt, n=n, row0=row0, nu=nu, q=q, seed=seed, prepared=Xp)


@dataclass
class ShardedSketch:
    """This rank's part of a sketch: L_r (nu x n_r, its columns of L) and the
    replicated R^T (nu x m)."""

    L_local: object
    Rt: object
    n: int
    row0: int
    nu: int
    q: int
    seed: int
    prepared: object = None  # the prepared copy of X_r (FP32), reused by compress


def subspace_iteration_pair_sharded(X_local, n: int, nu: int, q: int, seed: int, *, comm: Comm | None = None,
                                    ops=None) -> ShardedSketch:
    """Algorithm 2 (compression.py:120-141) on a row-sharded X: the same
    sequence of products and orthonormalisations as the 1-GPU
    ``subspace_iteration_pair``, with the exchanges listed in the module doc."""
    comm = comm or Comm()
    ops = ops or DeviceOps()
    n_r, m = X_local.shape
    row0, expect = row_block(n, comm.size, comm.rank)
    if expect != n_r:
        raise DimensionError(f"rank {comm.rank} holds {n_r} rows, row_block gives {expect}")
    nz = ops.sumsq(X_local)
    comm.all_reduce(nz)
    _check_iteration_inputs(n, m, nu, q, bool(float(nz[0]) > 0.0))
    # every rank draws the full stream (compression.py:130-132), on the device when it can
    Olt, Or, ok = ops.draws(n, m, nu, seed, X_local)
    Orl = Or[:, row0:row0 + n_r].contiguous()                 # this rank's columns of Omega_R
    Xp = ops.prepare(X_local, nu)
    L, Rt, status = _rsi_loop(X_local, q, comm, ops, row0, Olt, Orl, Xp)
    if not ops.draws_ok(ok):  # device stream not stitched (never observed): host draws, same sketch
        omega_l, omega_r = sketch_draws(n, m, nu, seed)
        return _rsi_with(X_local, n, nu, q, seed, comm, ops, row0, ops.tensor(omega_l.T, X_local),
                         ops.tensor(omega_r[:, row0:row0 + n_r], X_local), Xp)
    ops.check_status(status, "subspace iteration")
    return ShardedSketch(L_local=L, Rt=Rt, n=n, row0=row0, nu=nu, q=q, seed=seed, prepared=Xp)


def compress_problem_sharded(X_local, sketch: ShardedSketch, *, comm: Comm | None = None, ops=None):
    """(X_L (nu x m, all-reduced), X_R^T local columns (nu x n_r))."""
    comm = comm or Comm()
    ops = ops or DeviceOps()
    XRt, XL = ops.dual_pass(X_local, sketch.prepared, sketch.Rt, sketch.L_local)
    comm.all_reduce(XL)
    return XL, XRt


def gather_sketch(sketch: ShardedSketch, *, comm: Comm | None = None) -> SketchPair:
    """The full SketchPair (host NumPy, like the 1-GPU API) from the shards."""
    comm = comm or Comm()
    L = comm.all_gather_cols(sketch.L_local, sketch.n)
    pair = SketchPair(L=_lib.to_host(L), R=np.ascontiguousarray(_lib.to_host(sketch.Rt).T), nu=sketch.nu,
                      scheme=SUBSPACE_ITERATION, q=sketch.q, seed=sketch.seed)
    return pair


def _group_for(comm: Comm):
    """The SolveGroup of this communicator (created once: IPC-mapped buffers),
    or None when two ranks share a GPU: group solves wait on each other
    inside the kernel, so every rank needs its own device."""
    from .group import SolveGroup

    g = getattr(comm, "_solve_group", False)
    if g is False:
        torch = _lib.torch_mod()
        uuid = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
        uuids = [None] * comm.size
        comm.dist.all_gather_object(uuids, uuid, group=comm.group)
        g = SolveGroup.over(comm) if len(set(uuids)) == comm.size else None
        if g is not None and not g.self_test(comm):
            g.close()
            g = None
        comm._solve_group = g
    return g


def factorize_compressed_sharded(X_local, n: int, sketch: ShardedSketch, init, cfg=None, observer=None, clock=None,
                                 *, comm: Comm | None = None, return_device: bool = False,
                                 split_solves: bool | None = None):
    """Compressed NeNMF (factorize.py:197-213) on a row-sharded X.  ``init``
    holds the FULL initial factors (the same on every rank).

    With more than one rank the inner solves are split by columns over the
    ranks (group.py: this rank's rows of G, a slice of F's columns; the
    decision sums exchanged inside the solver over NVLink; two p x p'
    all-reduces per outer iteration) whenever every rank's share fits the
    register-resident solver -- the ranks agree on that first.  Otherwise
    (or with split_solves=False) X_R^T and L are all-gathered once and the
    outer loop is replicated on every rank.  The RRE always comes from
    all-reduced shard residuals."""
    from .factorize import OuterConfig, _GroupDeviceLoop, _run_outer, _ShardedDeviceLoop

    comm = comm or Comm()
    cfg = cfg or OuterConfig()
    XL, XRt_local = compress_problem_sharded(X_local, sketch, comm=comm)
    if split_solves is None:
        split_solves = comm.size > 1
    if split_solves and comm.size > 1:
        dt = "fp64" if str(X_local.dtype).endswith("float64") else "fp32"
        group = _group_for(comm)
        m = int(X_local.shape[1])
        _, n_r = row_block(n, comm.size, comm.rank)
        _, m_r = row_block(m, comm.size, comm.rank)
        ok = group is not None and (group.supported(dt, sketch.nu, init.p, n_r, sketch.nu, cfg.inner.max_iter) and
                                    group.supported(dt, sketch.nu, init.p, m_r, sketch.nu, cfg.inner.max_iter))
        if not comm.any(not ok):
            run = _GroupDeviceLoop(X_local, n, sketch.row0, init, sketch.L_local, sketch.Rt, XL, XRt_local, group,
                                   comm)
            return _run_outer(X_local, init, cfg, observer, clock, None, run.dtype, return_device, run=run)
    XRt = comm.all_gather_cols(XRt_local, n)
    L = comm.all_gather_cols(sketch.L_local, n)
    run = _ShardedDeviceLoop(X_local, n, sketch.row0, init, L, sketch.Rt, XL, XRt, comm)
    return _run_outer(X_local, init, cfg, observer, clock, None, run.dtype, return_device, run=run)


def factorize_compressed_emulated(X, sketch, init, cfg=None, observer=None, clock=None, *, ranks: int = 2,
                                  return_device: bool = False):
    """factorize_compressed with every inner solve run as an R-rank group
    EMULATED on the current GPU (group.SolveGroup.emulated: one launch whose
    CTAs form R virtual ranks over the same column split and exchange
    protocol as R GPUs).  X, the sketch and the factors as in the 1-GPU API;
    used to test the group solver on one device."""
    from .compression import compress_device, sketch_on_device
    from .factorize import OuterConfig, _GroupDeviceLoop, _run_outer
    from .group import SolveGroup

    cfg = cfg or OuterConfig()
    if hasattr(X, "is_cuda") and X.is_cuda:
        Xd = X
        dt = "fp64" if str(X.dtype).endswith("float64") else "fp32"
    else:
        dt = "fp64"
        Xd = _lib.to_device(np.asarray(X, dtype=np.float64), dt)
    L, Rt = sketch_on_device(sketch, dt)
    XL, XRt = compress_device(Xd, L, Rt)
    group = SolveGroup.emulated(ranks)
    run = _GroupDeviceLoop(Xd, Xd.shape[0], 0, init, L, Rt, XL, XRt, group)
    return _run_outer(Xd, init, cfg, observer, clock, None, dt, return_device, run=run)
