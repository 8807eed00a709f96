"""Matrix primitives of the drop-in API (reference ``matrix.py``).

Host-side: input coercion and the seeded draws, which must reproduce the
reference's NumPy PCG64 streams bit for bit (``matrix.py:31-87``).
Device-side: ``spectral_norm_sq`` and ``frobenius_norm`` run on the B200
through ``libnenmf_b200`` (no CPU fallback).
"""

from __future__ import annotations

import numpy as np

from . import _lib, _ops
from .errors import DimensionError, ZeroMatrixError

DenseMatrix = np.ndarray


def as_matrix(value, name: str = "matrix") -> DenseMatrix:
    """2-D float64 view/copy of ``value`` (matrix.py:31-36)."""
    if hasattr(value, "detach") and hasattr(value, "cpu"):  # torch tensor
        value = value.detach().cpu().numpy()
    M = np.asarray(value, dtype=np.float64)
    if M.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {M.shape}")
    return M


def check_seed(seed: int) -> int:
    """Seeds are unsigned 64-bit integers (matrix.py:45-49)."""
    seed = int(seed)
    if seed < 0 or seed >= 1 << 64:
        raise ValueError(f"seed must be an unsigned 64-bit integer, got {seed}")
    return seed


def gaussian_matrix(rows: int, cols: int, seed: int) -> DenseMatrix:
    """Seeded i.i.d. N(0,1) draws (matrix.py:52-70)."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"dimensions must be positive, got {rows}x{cols}")
    return np.random.default_rng(check_seed(seed)).standard_normal((rows, cols))


def open_uniform(rng: np.random.Generator, rows: int, cols: int) -> DenseMatrix:
    """U(0,1) draws with exact zeros re-drawn (matrix.py:73-82)."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"dimensions must be positive, got {rows}x{cols}")
    out = rng.random((rows, cols))
    hit = out == 0.0
    while hit.any():
        out[hit] = rng.random(int(hit.sum()))
        hit = out == 0.0
    return out


def uniform_matrix(rows: int, cols: int, seed: int) -> DenseMatrix:
    """Seeded open-uniform matrix (matrix.py:85-87)."""
    return open_uniform(np.random.default_rng(check_seed(seed)), rows, cols)


def _device_scalar():
    torch = _lib.torch_mod()
    return torch.zeros(4, dtype=torch.float64, device="cuda")


def spectral_norm_sq(G, tol: float = 1e-9, max_iters: int = 100, *, dtype: str = "fp64") -> float:
    """sigma_max(G)^2 by power iteration on the smaller Gram from the fixed
    seeded start vector, x1.01 when ``max_iters`` runs out (matrix.py:158-174).
    Runs on the GPU."""
    G = as_matrix(G, "G")
    if not G.any():
        raise ZeroMatrixError("spectral norm of the zero matrix is not useful here")
    _lib.require_device()
    r, p = G.shape
    At = _lib.to_device(np.ascontiguousarray(G.T), dtype)
    out = _device_scalar()
    status = _lib.new_status()
    _ops.spectral_norm_sq(At, tol, max_iters, out, status)
    st = _lib.read_status(status)[0]
    if st["code"] != 0:
        from .errors import raise_for_status

        raise_for_status(int(st["code"]), int(st["iteration"]), "spectral_norm_sq")
    return float(out[0].item())


def frobenius_norm(M, *, dtype: str = "fp64") -> float:
    """sqrt(sum of squares) (matrix.py:177-179), reduced on the GPU."""
    M = as_matrix(M)
    if M.size == 0:
        return 0.0
    _lib.require_device()
    Md = _lib.to_device(M, dtype)
    out = _device_scalar()
    _ops.sumsq(Md, out)
    return float(np.sqrt(out[0].item()))
