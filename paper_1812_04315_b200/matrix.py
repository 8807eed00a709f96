"""Matrix primitives of the drop-in API (reference ``matrix.py``).

Host-side: input coercion and the seeded draws, which must reproduce the
reference's NumPy PCG64 streams bit for bit (``matrix.py:31-87``).
Device-side: ``spectral_norm_sq`` and ``frobenius_norm`` run on the B200
through ``libnenmf_b200`` (no CPU fallback).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _lib, _ops
from .errors import DimensionError, ZeroMatrixError

DenseMatrix = np.ndarray

# NMFB binary format (matrix.py:26-28): magic, u32 version, u64 rows, u64 cols,
# then rows*cols little-endian float64, row-major
NMFB_MAGIC = b"NMFB"
NMFB_VERSION = 1
_NMFB_HEADER = struct.Struct("<4sIQQ")


def as_matrix(value, name: str = "matrix") -> DenseMatrix:
    """2-D float64 view/copy of ``value`` (matrix.py:31-36)."""
    if hasattr(value, "detach") and hasattr(value, "cpu"):  # torch tensor
        value = value.detach().cpu().numpy()
    M = np.asarray(value, dtype=np.float64)
    if M.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {M.shape}")
    return M


def require_finite(M: DenseMatrix, source: str) -> None:
    """Reject NaN/Inf entries of matrices read from files (matrix.py:39-42)."""
    if not np.isfinite(M).all():
        raise ValueError(f"non-finite entries in matrix from {source}")


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


# ------------------------------------------------------------------ NMFB IO
def write_nmfb(path, M) -> None:
    """Write ``M`` in the NMFB format (matrix.py:180-191)."""
    M = as_matrix(M)
    require_finite(M, f"write_nmfb({path})")
    rows, cols = M.shape
    header = _NMFB_HEADER.pack(NMFB_MAGIC, NMFB_VERSION, rows, cols)
    Path(path).write_bytes(header + np.ascontiguousarray(M, dtype="<f8").tobytes())


def _nmfb_header(path, size: int):
    """Validated (rows, cols) of an NMFB file of ``size`` bytes (matrix.py:196-208)."""
    with open(path, "rb") as fh:
        head = fh.read(_NMFB_HEADER.size)
    if len(head) < _NMFB_HEADER.size:
        raise ValueError(f"{path}: truncated NMFB file ({size} bytes)")
    magic, version, rows, cols = _NMFB_HEADER.unpack(head)
    if magic != NMFB_MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}, expected {NMFB_MAGIC!r}")
    if version != NMFB_VERSION:
        raise ValueError(f"{path}: unsupported NMFB version {version}")
    if rows < 1 or cols < 1:
        raise DimensionError(f"{path}: degenerate dimensions {rows}x{cols}")
    expected = _NMFB_HEADER.size + 8 * rows * cols
    if size != expected:
        raise ValueError(f"{path}: expected {expected} bytes, found {size}")
    return int(rows), int(cols)


def read_nmfb(path) -> DenseMatrix:
    """Read a matrix written by :func:`write_nmfb`; bit-exact (matrix.py:194-214)."""
    size = Path(path).stat().st_size
    rows, cols = _nmfb_header(path, size)
    data = np.fromfile(path, dtype="<f8", offset=_NMFB_HEADER.size, count=rows * cols)
    M = np.array(data, dtype=np.float64).reshape(rows, cols)
    require_finite(M, str(path))
    return M


def read_nmfb_device(path, *, dtype: str = "fp32", row0: int = 0, rows: int | None = None,
                     chunk_bytes: int = 64 << 20):
    """Rows [row0, row0 + rows) of an NMFB file straight into a CUDA tensor of
    ``dtype`` (feeding large X, e.g. one rank's row shard).

    The payload is read in chunks into two pinned host buffers; while one
    chunk is copied to the device and converted there (``nenmf_convert_f64``,
    which also flags NaN/Inf as read_nmfb's require_finite does), the host
    reads the next.  Header validation and errors follow read_nmfb."""
    lib, torch = _lib.require_device()
    size = Path(path).stat().st_size
    n, m = _nmfb_header(path, size)
    rows = n - row0 if rows is None else int(rows)
    if row0 < 0 or rows < 1 or row0 + rows > n:
        raise DimensionError(f"{path}: rows [{row0}, {row0 + rows}) outside the file's {n} rows")
    out = torch.empty((rows, m), dtype=_lib.torch_dtype(dtype), device="cuda")
    total = rows * m
    per = max(2, (int(chunk_bytes) // 8) & ~1)  # even: the device loads pairs
    per = min(per, total + (total & 1))
    stream = torch.cuda.current_stream()
    host = [torch.empty(per, dtype=torch.float64).pin_memory() for _ in range(2)]
    dev = [torch.empty(per, dtype=torch.float64, device="cuda") for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    code = _lib.code_of(dtype)
    flat = out.view(-1)
    with open(path, "rb") as fh:
        fh.seek(_NMFB_HEADER.size + 8 * row0 * m)
        off, i = 0, 0
        while off < total:
            cnt = min(per, total - off)
            b = i & 1
            done[b].synchronize()  # the pinned buffer's previous copy has left
            hv = host[b].numpy()
            got = fh.readinto(memoryview(hv[:cnt]).cast("B"))
            if got != 8 * cnt:
                raise ValueError(f"{path}: truncated NMFB file")
            dev[b][:cnt].copy_(host[b][:cnt], non_blocking=True)
            rc = lib.nenmf_convert_f64(code, dev[b].data_ptr(), cnt, flat[off:].data_ptr(), flag.data_ptr(),
                                       stream.cuda_stream)
            _lib.check(rc, "read_nmfb_device")
            done[b].record(stream)
            off += cnt
            i += 1
    if int(flag.item()) != 0:
        raise ValueError(f"non-finite entries in matrix from {path}")
    return out
