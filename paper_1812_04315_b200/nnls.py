"""Nesterov-accelerated NNLS inner solver (reference ``nnls.py``), on the GPU.

``solve_nnls`` keeps the reference signature and semantics (nnls.py:119-227):
Gram-form gradients, the affine extrapolated-gradient trick, the KKT
projected-gradient stop relative to the start point, best-iterate tracking
and the explicit-residual tie-break.  The whole solve is one call into
``libnenmf_b200`` (``nenmf_solve_nnls``): W and V products, the Lipschitz
power iteration, a single persistent kernel for the inner loop, and the
tie-break, with no host round trip per inner iteration.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib, _ops
from .errors import DimensionError, ZeroMatrixError, raise_for_status
from .matrix import DenseMatrix, as_matrix


@dataclass(frozen=True)
class InnerSolverConfig:
    """Stop/step parameters (nnls.py:25-46): iteration cap, relative
    projected-gradient tolerance, Lipschitz safety factor."""

    max_iter: int = 500
    grad_tol: float = 1e-4
    lipschitz_safety: float = 1.0

    def __post_init__(self):
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if not (self.grad_tol > 0 and math.isfinite(self.grad_tol)):
            raise ValueError(f"grad_tol must be positive and finite, got {self.grad_tol}")
        if not self.lipschitz_safety >= 1.0:
            raise ValueError(f"lipschitz_safety must be >= 1, got {self.lipschitz_safety}")


@dataclass
class InnerSolverState:
    """Loop state of the reference solver (nnls.py:49-58); exported for API
    parity.  The device solver keeps the equivalent state on the GPU."""

    k: int
    alpha: float
    Y: DenseMatrix
    F_prev: DenseMatrix
    F_curr: DenseMatrix
    lipschitz: float


def alpha_next(alpha: float) -> float:
    """alpha_{k+1} = (1 + sqrt(4 alpha_k^2 + 1)) / 2 (nnls.py:61-69)."""
    if not alpha >= 1.0:
        raise ValueError(f"alpha must be >= 1, got {alpha}")
    return (1.0 + math.sqrt(4.0 * alpha * alpha + 1.0)) / 2.0


def _check_abf(A, B, F):
    r, p = A.shape
    if F.shape[0] != p or B.shape != (r, F.shape[1]):
        raise DimensionError(f"incompatible shapes: A {A.shape}, F {F.shape}, B {B.shape}")


def gradient(A, B, F, *, dtype: str = "fp64") -> DenseMatrix:
    """A^T (A F - B), evaluated on the GPU in Gram form (nnls.py:72-86)."""
    A = as_matrix(A, "A")
    B = as_matrix(B, "B")
    F = as_matrix(F, "F")
    _check_abf(A, B, F)
    _, torch = _lib.require_device()
    At = _lib.to_device(np.ascontiguousarray(A.T), dtype)
    Bd = _lib.to_device(B, dtype)
    Fd = _lib.to_device(F, dtype)
    out = torch.empty_like(Fd)
    _ops.gradient(At, Bd, Fd, out)
    return _lib.to_host(out)


def projected_gradient_norm(F, grad, *, dtype: str = "fp64") -> float:
    """||g where F > 0 else min(g, 0)||_F (nnls.py:89-100), on the GPU."""
    F = as_matrix(F, "F")
    grad = as_matrix(grad, "grad")
    if F.shape != grad.shape:
        raise DimensionError(f"shape mismatch: F {F.shape} vs grad {grad.shape}")
    _, torch = _lib.require_device()
    if F.size == 0:
        return 0.0
    out = _lib.zeros(1, torch.float64)
    _ops.sumsq(_lib.to_device(F, dtype), out, g=_lib.to_device(grad, dtype))
    return math.sqrt(out.item())


@dataclass
class SolveReport:
    """Device status of one solve (extension, not in the reference API)."""

    inner_iters: int
    returned_best: bool
    lipschitz: float


def _raise_solve_status(st) -> None:
    code = int(st["code"])
    if code != 0:
        raise_for_status(code, int(st["iteration"]), "solve_nnls")


def solve_nnls(A, B, F0, cfg: InnerSolverConfig = InnerSolverConfig(), *, dtype: str = "fp64",
               report: list | None = None) -> DenseMatrix:
    """min_{F >= 0} 1/2 ||B - A F||_F^2 from F0 (nnls.py:119-227), on the GPU.

    Same checks in the same order as the reference: shapes (DimensionError),
    A all zero (ZeroMatrixError), F0 negative (ValueError); non-finite
    iterates raise NumericalFailureError carrying the inner iteration.
    ``dtype`` (keyword-only extension) selects FP64 (parity) or FP32
    arithmetic; ``report`` (extension) receives a SolveReport.
    """
    A = np.ascontiguousarray(as_matrix(A, "A"))
    B = np.ascontiguousarray(as_matrix(B, "B"))
    F0 = np.ascontiguousarray(as_matrix(F0, "F0"))
    r, p = A.shape
    c = B.shape[1]
    if B.shape[0] != r or F0.shape != (p, c):
        raise DimensionError(f"incompatible shapes: A {A.shape}, B {B.shape}, F0 {F0.shape}")
    if not A.any():
        raise ZeroMatrixError("A is all zero; the subproblem has no useful gradient")
    if F0.min() < 0.0:
        raise ValueError("F0 must be entrywise nonnegative")
    _, torch = _lib.require_device()
    At = _lib.to_device(np.ascontiguousarray(A.T), dtype)
    Bd = _lib.to_device(B, dtype)
    F0d = _lib.to_device(F0, dtype)
    Fout = torch.empty_like(F0d)
    status = _lib.new_status()
    _ops.solve(At, Bd, F0d, Fout, trans_b=False, max_iter=cfg.max_iter, grad_tol=cfg.grad_tol,
               lipschitz_safety=cfg.lipschitz_safety, status=status)
    st = _lib.read_status(status)[0]
    _raise_solve_status(st)
    if report is not None:
        report.append(SolveReport(int(st["inner_iters"]), bool(st["returned_best"]), float(st["lipschitz"])))
    return _lib.to_host(Fout)
