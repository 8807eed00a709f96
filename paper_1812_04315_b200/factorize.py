"""Outer alternating loops of vanilla and compressed NeNMF (reference
``factorize.py``), driving the GPU kernels.

The loop keeps the reference's control flow, stopping rules, trace cadence,
clock protocol and exceptions (``factorize.py:116-183``).  All arithmetic runs
on the device: X, the sketch, X_L / X_R^T and both factors stay resident in
HBM for the whole run; each half-step is one ``nenmf_solve_nnls`` call (plus
one skinny product for the compressed A-operand); ``emit`` evaluates the full
||X - G F||_F on the GPU with the clock paused.  The host synchronises only
where the reference's semantics need a value: ``emit``, time-budget checks
and status checks (status words of queued half-steps are drained at those
points, so a failure still surfaces with its outer and inner indices).

Layout in HBM: X row-major n x m; G held transposed (G^T, p x n) so that both
half-steps solve the same column-parallel problem; F p x m; L nu x n and R^T
nu x m; X_L nu x m and X_R^T nu x n.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib, _ops
from .compression import SketchPair, compress_device, prepared_for, sketch_on_device
from .errors import DimensionError, NumericalFailureError, ZeroMatrixError, raise_for_status
from .matrix import DenseMatrix, as_matrix, check_seed, open_uniform
from .nnls import InnerSolverConfig
from .tracing import MonotonicClock, SolverClock, TraceRecord

Observer = Callable[[TraceRecord, np.ndarray, np.ndarray], None]


def _on_device(M) -> bool:
    return bool(getattr(M, "is_cuda", False))


@dataclass(frozen=True, eq=False)
class FactorPair:
    """Factors G (n x p) and F (p x m), entrywise nonnegative (factorize.py:32-48)."""

    G: DenseMatrix
    F: DenseMatrix
    p: int

    def __post_init__(self):
        if self.G.ndim != 2 or self.F.ndim != 2:
            raise DimensionError("factors must be 2-D")
        if self.G.shape[1] != self.p or self.F.shape[0] != self.p:
            raise DimensionError(
                f"factor shapes {tuple(self.G.shape)}, {tuple(self.F.shape)} do not match rank {self.p}")
        # host arrays are checked here (the reference's point); factors already
        # on the device are checked by a flag scan when a factorization starts
        # (_run_outer), so building a pair never synchronises the device
        for M in (self.G, self.F):
            if not _on_device(M) and M.min() < 0.0:
                raise ValueError("factors must be entrywise nonnegative")


@dataclass(frozen=True)
class OuterConfig:
    """Stopping rules and trace cadence (factorize.py:51-74)."""

    inner: InnerSolverConfig = InnerSolverConfig()
    time_budget_seconds: float = 15.0
    max_outer_iterations: int = 0
    rre_target: float = 0.0
    trace_every: int = 1

    def __post_init__(self):
        if self.time_budget_seconds < 0 or self.max_outer_iterations < 0:
            raise ValueError("stopping limits must be nonnegative")
        if not (self.time_budget_seconds > 0 or self.max_outer_iterations >= 1):
            raise ValueError("need a positive time budget or an iteration cap")
        if self.rre_target < 0:
            raise ValueError(f"rre_target must be >= 0, got {self.rre_target}")
        if self.trace_every < 1:
            raise ValueError(f"trace_every must be >= 1, got {self.trace_every}")


def init_factors(n: int, m: int, p: int, seed: int) -> FactorPair:
    """Seeded open-uniform G then F from one stream (factorize.py:77-86)."""
    if p < 1:
        raise DimensionError(f"rank must be >= 1, got {p}")
    if p > min(n, m):
        raise DimensionError(f"rank {p} exceeds min(n, m) = {min(n, m)}")
    gen = np.random.default_rng(check_seed(seed))
    G = open_uniform(gen, n, p)
    F = open_uniform(gen, p, m)
    return FactorPair(G=G, F=F, p=p)


_STATUS_CAP = 128  # queued half-steps between status drains


def _panel_t(G, dtype: str):
    """G (n x p) as a fresh contiguous G^T (p x n) on the device: a transpose
    kernel (nenmf_transpose) for device factors, one upload for host ones."""
    if not _on_device(G):
        return _lib.to_device(np.ascontiguousarray(np.asarray(G, dtype=np.float64).T), dtype)
    G = _lib.to_device(G, dtype) if G.dtype != _lib.torch_dtype(dtype) else G
    if G.t().is_contiguous():
        return G.t().clone()
    return _ops.transpose(G)


class _DeviceLoop:
    """Device state of one factorization run."""

    def __init__(self, X, init: FactorPair, sketch: SketchPair | None, dtype: str):
        _, torch = _lib.require_device()
        self.torch = torch
        if hasattr(X, "is_cuda") and X.is_cuda:
            self.X = X if X.is_contiguous() else X.contiguous()
            dtype = "fp64" if X.dtype == torch.float64 else "fp32"
        else:
            self.X = _lib.to_device(as_matrix(X, "X"), dtype)
        self.dtype = dtype
        self.n, self.m = self.X.shape
        self.p = init.p
        self.sketch = sketch
        self.scal = _lib.zeros(4, torch.float64)
        self.status = _lib.new_status(_STATUS_CAP)
        self.pending: list[tuple[int, str, int]] = []
        self.tensor_v = False

    def norm_x(self) -> float:
        _ops.sumsq(self.X, self.scal[0:1])
        return math.sqrt(self.scal[0].item())

    def prepare(self, init: FactorPair) -> None:
        torch = self.torch
        G = init.G
        self.Gt = _panel_t(G, self.dtype)
        self.F = _lib.to_device(init.F, self.dtype)
        if self.F is init.F:  # never write into the caller's tensor
            self.F = self.F.clone()
        self.Gt_alt = torch.empty_like(self.Gt)
        self.F_alt = torch.empty_like(self.F)
        if self.sketch is not None:
            L, Rt = sketch_on_device(self.sketch, self.dtype)
            self.L, self.Rt = L, Rt
            # the compressed preamble stays on the solver clock (factorize.py:130)
            self.Xp = prepared_for(self.sketch, self.X)  # also read by the emit's residual (objective)
            self.XL, self.XRt = compress_device(self.X, L, Rt, prepared=self.Xp)
            nu = L.shape[0]
            self.FR = torch.empty((self.p, nu), dtype=self.X.dtype, device="cuda")
            self.fr_ready = False
            self.GLt = torch.empty((self.p, nu), dtype=self.X.dtype, device="cuda")

    def _slot(self, t: int, half: str) -> int:
        if len(self.pending) >= _STATUS_CAP:
            self.drain()
        idx = len(self.pending)
        self.pending.append((t, half, idx))
        return idx

    def half_steps(self, t: int, icfg: InnerSolverConfig) -> None:
        kw = dict(max_iter=icfg.max_iter, grad_tol=icfg.grad_tol, lipschitz_safety=icfg.lipschitz_safety,
                  status=self.status)
        if self.sketch is not None:
            # G-half: A = (F R)^T, B = X_R^T (factorize.py:109-110); F R comes
            # from the previous F-half's launch (or once, before the first)
            if not self.fr_ready:
                _ops.abt(self.F, self.Rt, self.FR)
            # ... and L G for the F-half is formed by this G-half's launch
            _ops.solve(self.FR, self.XRt, self.Gt, self.Gt_alt, trans_b=False,
                       status_index=self._slot(t, "G"), next_bt=self.L, next_out=self.GLt, **kw)
            self.Gt, self.Gt_alt = self.Gt_alt, self.Gt
            # F-half: A = L G, B = X_L (factorize.py:112-113); it also forms the
            # next G-half's F R
            _ops.solve(self.GLt, self.XL, self.F, self.F_alt, trans_b=False,
                       status_index=self._slot(t, "F"), next_bt=self.Rt, next_out=self.FR, **kw)
            self.fr_ready = True
        else:
            # FP32 with tensor_v: V = A^T B from one tensor-core pass over the
            # prepared X (BF16x3: ~2x faster half-steps, V to ~1e-5 relative,
            # factors to ~1e-3 of the fp64 reference); default: CUDA-core V
            if not hasattr(self, "Xp"):
                self.Xp = _ops.prepare_x(self.X, self.p) if self.tensor_v else None
            # G-half: A = F^T, B = X^T read in place (factorize.py:94-95)
            _ops.solve(self.F, self.X, self.Gt, self.Gt_alt, trans_b=True,
                       status_index=self._slot(t, "G"), Xp=self.Xp, **kw)
            self.Gt, self.Gt_alt = self.Gt_alt, self.Gt
            # F-half: A = G, B = X (factorize.py:97-98)
            _ops.solve(self.Gt, self.X, self.F, self.F_alt, trans_b=False,
                       status_index=self._slot(t, "F"), Xp=self.Xp, **kw)
        self.F, self.F_alt = self.F_alt, self.F

    def drain(self) -> None:
        """Synchronise and surface the first failure among queued half-steps."""
        if not self.pending:
            return
        sts = _lib.read_status(self.status)
        pending, self.pending = self.pending, []
        _lib.zero_(self.status)
        for t, half, idx in pending:
            st = sts[idx]
            code = int(st["code"])
            if code == 0:
                continue
            try:
                raise_for_status(code, int(st["iteration"]), f"{half} update")
            except NumericalFailureError as exc:
                raise NumericalFailureError(
                    f"outer iteration {t} ({half} update): {exc}",
                    iteration=exc.iteration, outer_iteration=t) from exc

    def stop_vote(self, stop: bool) -> bool:
        return stop

    def resid_xp(self):
        """The prepared copy of this rank's X read by the emit's residual (FP32:
        one tensor-core pass, k_resid_bulk): the solver's / sketch's copy when
        there is one, else made once on first use; None for FP64."""
        if self.dtype != "fp32":
            return None
        xp = getattr(self, "Xp", None)
        if xp is None:
            xp = getattr(self, "_resid_xp", None)
            if xp is None:
                xp = self._resid_xp = _ops.prepare_x(self.X, self.p)
        return xp

    def objective(self) -> float:
        _ops.residual_sumsq(self.X, self.Gt, self.F, self.scal[1:2], Xp=self.resid_xp())
        return math.sqrt(self.scal[1].item())

    def host_factors(self):
        return _lib.to_host(self.Gt).T.copy(), _lib.to_host(self.F)


class _ShardedDeviceLoop(_DeviceLoop):
    """Device state of a row-sharded run (sharded.py): this rank holds rows
    [row0, row0 + n_r) of X; the compressed operands are replicated, so the
    half-steps are the 1-GPU ones and every rank computes the same G and F.
    ||X|| and the objective are all-reduced over the shards."""

    def __init__(self, X_local, n: int, row0: int, init: FactorPair, L, Rt, XL, XRt, comm):
        _, torch = _lib.require_device()
        self.torch = torch
        self.X = X_local if X_local.is_contiguous() else X_local.contiguous()
        self.dtype = "fp64" if X_local.dtype == torch.float64 else "fp32"
        self.n, self.m = int(n), int(X_local.shape[1])
        self.row0, self.n_r = int(row0), int(X_local.shape[0])
        self.p = init.p
        self.sketch = "sharded"  # compressed half-steps
        self.scal = _lib.zeros(4, torch.float64)
        self.status = _lib.new_status(_STATUS_CAP)
        self.pending = []
        self.comm = comm
        self._ops_in = (L, Rt, XL, XRt)

    def norm_x(self) -> float:
        _lib.zero_(self.scal[0:1])
        _ops.sumsq(self.X, self.scal[0:1])
        self.comm.all_reduce(self.scal[0:1])
        return math.sqrt(self.scal[0].item())

    def prepare(self, init: FactorPair) -> None:
        torch = self.torch
        G = init.G
        self.Gt = _panel_t(G, self.dtype)
        self.F = _lib.to_device(init.F, self.dtype)
        if self.F is init.F:  # never write into the caller's tensor
            self.F = self.F.clone()
        self.Gt_alt = torch.empty_like(self.Gt)
        self.F_alt = torch.empty_like(self.F)
        self.L, self.Rt, self.XL, self.XRt = self._ops_in
        nu = self.L.shape[0]
        self.FR = torch.empty((self.p, nu), dtype=self.X.dtype, device="cuda")
        self.fr_ready = False
        self.GLt = torch.empty((self.p, nu), dtype=self.X.dtype, device="cuda")

    def stop_vote(self, stop: bool) -> bool:
        """The time-budget stop is decided collectively: every rank leaves the
        loop after the same outer iteration if ANY rank's clock ran out, so the
        all-reduces of emit always have all partners."""
        return self.comm.any(stop)

    def objective(self) -> float:
        Gl = self.Gt[:, self.row0:self.row0 + self.n_r].contiguous()
        _lib.zero_(self.scal[1:2])
        _ops.residual_sumsq(self.X, Gl, self.F, self.scal[1:2], Xp=self.resid_xp())
        self.comm.all_reduce(self.scal[1:2])
        return math.sqrt(self.scal[1].item())


class _GroupDeviceLoop(_DeviceLoop):
    """Compressed NeNMF with every inner solve split by columns over the ranks
    of a SolveGroup (group.py).

    Real group (one process per GPU, group.nvr == 1): this rank holds rows
    [row0, row0 + n_r) of X, its columns of X_R^T and L (from the sharded
    compression), the replicated X_L and R^T; it solves its n_r columns of
    G^T and its slice [m0, m0 + m_r) of F's columns; the partial next products
    (L_r G_r and F_r R_r) are all-reduced, F is all-gathered at emits.

    Emulated group (group.nvr == R, one GPU): the whole problem in this
    process, each solve ONE launch whose CTAs form R virtual ranks over the
    same column split; the per-rank partial next products are summed here."""

    def __init__(self, X_local, n: int, row0: int, init: FactorPair, L_local, Rt, XL, XRt_local, group, comm=None):
        _, torch = _lib.require_device()
        self.torch = torch
        self.X = X_local if X_local.is_contiguous() else X_local.contiguous()
        self.dtype = "fp64" if X_local.dtype == torch.float64 else "fp32"
        self.n, self.m = int(n), int(X_local.shape[1])
        self.row0, self.n_r = int(row0), int(X_local.shape[0])
        self.p = init.p
        self.sketch = "group"
        self.scal = _lib.zeros(4, torch.float64)
        self.status = _lib.new_status(_STATUS_CAP)
        self.pending = []
        self.group, self.comm = group, comm
        self.emulated = group.nvr > 1
        self._ops_in = (L_local, Rt, XL, XRt_local)

    def norm_x(self) -> float:
        _lib.zero_(self.scal[0:1])
        _ops.sumsq(self.X, self.scal[0:1])
        if not self.emulated:
            self.comm.all_reduce(self.scal[0:1])
        return math.sqrt(self.scal[0].item())

    def prepare(self, init: FactorPair) -> None:
        from .group import partition
        from .sharded import row_block

        torch = self.torch
        L, Rt, XL, XRt = self._ops_in
        nu = Rt.shape[0]
        G = init.G
        Gt_full = _panel_t(G, self.dtype)
        F_full = _lib.to_device(init.F, self.dtype)
        R = self.group.ranks
        # the first G-half's F R from the (replicated) initial F
        self.FR = torch.empty((self.p, nu), dtype=self.X.dtype, device="cuda")
        _ops.abt(F_full, Rt, self.FR)
        self.GLt = torch.empty((self.p, nu), dtype=self.X.dtype, device="cuda")
        self.L, self.Rt_full = L, Rt
        if self.emulated:
            self.Gt = Gt_full
            self.F = F_full if F_full is not init.F else F_full.clone()
            self.XRt, self.XL_s, self.Rt_s = XRt, XL, Rt
            self.g_cols, self.f_cols = partition(self.n, R), partition(self.m, R)
        else:
            self.Gt = Gt_full[:, self.row0:self.row0 + self.n_r].contiguous()
            self.m0, self.m_r = row_block(self.m, R, self.group.rank)
            self.F = F_full[:, self.m0:self.m0 + self.m_r].contiguous()
            self.XRt = XRt
            self.XL_s = XL[:, self.m0:self.m0 + self.m_r].contiguous()
            self.Rt_s = Rt[:, self.m0:self.m0 + self.m_r].contiguous()
            self.g_cols, self.f_cols = [0, self.n_r], [0, self.m_r]
        self.Gt_alt = torch.empty_like(self.Gt)
        self.F_alt = torch.empty_like(self.F)
        self.part = torch.empty((self.group.nvr, self.p, nu), dtype=self.X.dtype, device="cuda")

    def _reduce_next(self, out) -> None:
        if self.emulated:
            self.torch.sum(self.part, dim=0, out=out)
        else:
            out.copy_(self.part[0])
            self.comm.all_reduce(out)

    def half_steps(self, t: int, icfg: InnerSolverConfig) -> None:
        kw = dict(max_iter=icfg.max_iter, grad_tol=icfg.grad_tol, lipschitz_safety=icfg.lipschitz_safety,
                  status=self.status)
        # G-half: A = (F R)^T, B = X_R^T (factorize.py:109-110), columns = G's rows
        _ops.solve_group(self.FR, self.XRt, self.Gt, self.Gt_alt, group=self.group.struct(self.g_cols),
                         status_index=self._slot(t, "G"), next_bt=self.L, next_out=self.part, **kw)
        self.Gt, self.Gt_alt = self.Gt_alt, self.Gt
        self._reduce_next(self.GLt)
        # F-half: A = L G, B = X_L (factorize.py:112-113), columns = F's columns
        _ops.solve_group(self.GLt, self.XL_s, self.F, self.F_alt, group=self.group.struct(self.f_cols),
                         status_index=self._slot(t, "F"), next_bt=self.Rt_s, next_out=self.part, **kw)
        self.F, self.F_alt = self.F_alt, self.F
        self._reduce_next(self.FR)

    def stop_vote(self, stop: bool) -> bool:
        return stop if self.emulated else self.comm.any(stop)

    def full_F(self):
        return self.F if self.emulated else self.comm.all_gather_cols(self.F, self.m)

    def objective(self) -> float:
        _lib.zero_(self.scal[1:2])
        _ops.residual_sumsq(self.X, self.Gt, self.full_F(), self.scal[1:2], Xp=self.resid_xp())
        if not self.emulated:
            self.comm.all_reduce(self.scal[1:2])
        return math.sqrt(self.scal[1].item())

    def full_Gt(self):
        return self.Gt if self.emulated else self.comm.all_gather_cols(self.Gt, self.n)

    def host_factors(self):
        return _lib.to_host(self.full_Gt()).T.copy(), _lib.to_host(self.full_F())

    def device_factors(self):
        return self.full_Gt().t(), self.full_F()


def _run_outer(X, init: FactorPair, cfg: OuterConfig, observer, clock, sketch, dtype: str,
               return_device: bool = False, run: _DeviceLoop | None = None) -> FactorPair:
    if run is not None:
        n, m = run.n, run.m
    elif hasattr(X, "is_cuda") and X.is_cuda:
        n, m = X.shape
    else:
        X = as_matrix(X, "X")
        n, m = X.shape
    if tuple(init.G.shape) != (n, init.p) or tuple(init.F.shape) != (init.p, m):
        raise DimensionError(
            f"init shapes {tuple(init.G.shape)}, {tuple(init.F.shape)} do not match data {n}x{m}")
    if sketch is not None and (np.shape(sketch.L) != (sketch.nu, n) or np.shape(sketch.R) != (m, sketch.nu)):
        raise DimensionError(
            f"sketch shapes L {np.shape(sketch.L)}, R {np.shape(sketch.R)} do not match "
            f"data {n}x{m} at target rank {sketch.nu}")
    if run is None:
        run = _DeviceLoop(X, init, sketch, dtype)
    neg = None
    if _on_device(init.G) or _on_device(init.F):
        # FactorPair's sign check for device factors, read with ||X||'s sync
        neg = _lib.zeros(2, run.torch.int32)
        for i, M in enumerate((init.G, init.F)):
            if _on_device(M):
                _ops.scan_flags(M, negative_ptr=neg.data_ptr() + 4 * i)
    norm_x = run.norm_x()
    if neg is not None and bool(neg.cpu().any()):
        raise ValueError("factors must be entrywise nonnegative")
    if norm_x == 0.0:
        raise ZeroMatrixError("cannot factorize the zero matrix")
    if clock is None:
        clock = MonotonicClock()
    run.prepare(init)
    stream = run.torch.cuda.current_stream()
    last_traced = -1

    def emit(t: int) -> float:
        nonlocal last_traced
        stream.synchronize()  # charge queued device work to the solver clock
        run.drain()
        clock.pause()
        objective = run.objective()
        value = objective / norm_x
        record = TraceRecord(outer_iter=t, solver_elapsed_s=clock.elapsed(),
                             wall_elapsed_s=clock.wall_elapsed(), rre=value, objective=objective)
        if observer is not None:
            G, F = run.host_factors()
            observer(record, G, F)
        last_traced = t
        clock.resume()
        return value

    current = emit(0)
    t = 0
    done = cfg.rre_target > 0 and current <= cfg.rre_target
    while not done:
        if cfg.max_outer_iterations > 0 and t >= cfg.max_outer_iterations:
            break
        if cfg.time_budget_seconds > 0:
            stream.synchronize()
            run.drain()
            # one decision for all shards of a sharded run (each rank has its own clock)
            if run.stop_vote(clock.elapsed() >= cfg.time_budget_seconds):
                break
        t += 1
        run.half_steps(t, cfg.inner)
        clock.tick()
        if t % cfg.trace_every == 0:
            current = emit(t)
            if cfg.rre_target > 0 and current <= cfg.rre_target:
                break
    if last_traced != t:
        emit(t)
    run.drain()
    if return_device:
        if hasattr(run, "device_factors"):
            G, F = run.device_factors()
            return FactorPair(G=G, F=F, p=init.p)
        return FactorPair(G=run.Gt.t(), F=run.F, p=init.p)
    G, F = run.host_factors()
    return FactorPair(G=G, F=F, p=init.p)


def factorize_vanilla(X, init: FactorPair, cfg: OuterConfig = OuterConfig(),
                      observer: Observer | None = None, clock: SolverClock | None = None, *,
                      dtype: str = "fp64", return_device: bool = False, tensor_v: bool = True) -> FactorPair:
    """Alternating NeNMF on the full data (factorize.py:186-194), on the GPU.
    ``tensor_v`` (FP32 only, default): form V = A^T B with the tcgen05 BF16x3
    pass over a prepared copy of X (the RSI X-pass kernel); False: the
    CUDA-core/mma.sync 3xTF32 products over the raw X.  An fp64 X has no
    prepared form (the flag is then a no-op)."""
    if tensor_v and (dtype == "fp32" or str(getattr(X, "dtype", "")).endswith("float32")):
        if not (hasattr(X, "is_cuda") and X.is_cuda):
            X = as_matrix(X, "X")
        run = _DeviceLoop(X, init, None, dtype)
        run.tensor_v = True
        return _run_outer(X, init, cfg, observer, clock, None, dtype, return_device, run=run)
    return _run_outer(X, init, cfg, observer, clock, None, dtype, return_device)


def factorize_compressed(X, sketch: SketchPair, init: FactorPair, cfg: OuterConfig = OuterConfig(),
                         observer: Observer | None = None, clock: SolverClock | None = None, *,
                         dtype: str = "fp64", return_device: bool = False) -> FactorPair:
    """Alternating NeNMF on the sketch-compressed surrogates (factorize.py:197-213);
    RRE and objective are still reported against the full X."""
    return _run_outer(X, init, cfg, observer, clock, sketch, dtype, return_device)
