"""Sketch operators and data compression (reference ``compression.py``).

``subspace_iteration_pair`` (Alg. 2, ``compression.py:120-141``) and
``compress_problem`` (``:179-188``) run on the GPU: the Gaussian draws are
made on the host with the reference's exact NumPy stream, then every pass
over X and every QR executes in ``libnenmf_b200`` (fused X-passes that serve
the L-chain and the R-chain from one read of X; TSQR in shared memory).
``gaussian_sketch_pair`` is host RNG only, as in the reference.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib, _ops
from .errors import DimensionError, ZeroMatrixError, raise_for_status
from .matrix import DenseMatrix, as_matrix, check_seed, read_nmfb, write_nmfb

GAUSSIAN = "gaussian"
POWER_ITERATION = "power_iteration"
SUBSPACE_ITERATION = "subspace_iteration"
SCHEMES = (GAUSSIAN, POWER_ITERATION, SUBSPACE_ITERATION)


@dataclass(frozen=True, eq=False)
class SketchPair:
    """L (nu x n) left-compresses, R (m x nu) right-compresses
    (compression.py:42-55).  ``device`` (extension) optionally caches the
    device copies (L, R^T) keyed by dtype so factorization can skip re-upload."""

    L: DenseMatrix
    R: DenseMatrix
    nu: int
    scheme: str
    q: int
    seed: int
    device: dict = field(default_factory=dict, repr=False, compare=False)


@dataclass(frozen=True, eq=False)
class CompressedProblem:
    """X_L = L X (nu x m) and X_R = X R (n x nu) (compression.py:58-63)."""

    X_L: DenseMatrix
    X_R: DenseMatrix


def _check_sketch_dims(n: int, m: int, nu: int) -> None:
    if nu < 1:
        raise DimensionError(f"target rank must be >= 1, got {nu}")
    if n < 1 or m < 1:
        raise DimensionError(f"data dimensions must be positive, got {n}x{m}")


def gaussian_sketch_pair(n: int, m: int, nu: int, seed: int) -> SketchPair:
    """L = Omega_L / sqrt(nu), R = Omega_R / sqrt(nu), L drawn first
    (compression.py:73-85).  Host RNG only."""
    _check_sketch_dims(n, m, nu)
    gen = np.random.default_rng(check_seed(seed))
    scale = 1.0 / np.sqrt(nu)
    L = gen.standard_normal((nu, n)) * scale
    R = gen.standard_normal((m, nu)) * scale
    return SketchPair(L=L, R=R, nu=nu, scheme=GAUSSIAN, q=0, seed=seed)


def _check_iteration_inputs(n: int, m: int, nu: int, q: int, nonzero: bool) -> None:
    """compression.py:109-117, same order."""
    _check_sketch_dims(n, m, nu)
    if nu > min(n, m):
        raise DimensionError(f"target rank {nu} exceeds min(n, m) = {min(n, m)}")
    if q < 1:
        raise ValueError(f"iteration count must be >= 1, got {q}")
    if not nonzero:
        raise ZeroMatrixError("cannot sketch the zero matrix")


def sketch_draws(n: int, m: int, nu: int, seed: int):
    """The reference's Gaussian start blocks, Omega_L (m x nu) then Omega_R
    (nu x n), from one PCG64 stream (compression.py:130-132)."""
    gen = np.random.default_rng(check_seed(seed))
    omega_l = gen.standard_normal((m, nu))
    omega_r = gen.standard_normal((nu, n))
    return omega_l, omega_r


_ZIG_TABLES: dict = {}
# ziggurat tail constants of NumPy's random_standard_normal
_ZIG_R = 3.6541528853610087963519472518
_ZIG_INV_R = 0.27366123732975827203338247596


def _numpy_ziggurat_tables():
    """NumPy's standard_normal ziggurat tables (fi, wi: double[256]; ki:
    uint64[256]) read from the installed NumPy build (the reference's RNG
    dependency), or None if they cannot be located and checked."""
    if "host" in _ZIG_TABLES:
        return _ZIG_TABLES["host"]
    import os
    import struct

    import numpy.random

    tabs = None
    try:
        d = os.path.dirname(numpy.random.__file__)
        for name in sorted(os.listdir(d)):
            if not (name.startswith("_generator") and name.endswith(".so")):
                continue
            blob = open(os.path.join(d, name), "rb").read()
            i = blob.find(struct.pack("<d", 8.68362706080130616677e-16))  # wi[0]
            if i < 2048:
                continue
            fi = np.frombuffer(blob[i - 2048:i], dtype="<f8")
            wi = np.frombuffer(blob[i:i + 2048], dtype="<f8")
            ki = np.frombuffer(blob[i + 2048:i + 4096], dtype="<u8")
            if fi[0] == 1.0 and 0.97 < fi[1] < 0.98 and ki[0] == 0x000EF33D8025EF6A and ki[1] == 0 \
                    and np.all(np.diff(fi) < 0):
                tabs = np.concatenate([fi.view(np.uint64), wi.view(np.uint64), ki]).copy()
                break
    except OSError:
        tabs = None
    _ZIG_TABLES["host"] = tabs
    return tabs


def sketch_draws_device(n: int, m: int, nu: int, seed: int, dtype: str, ok_ptr: int | None = None):
    """The draws of ``sketch_draws`` generated on the device (nenmf_sketch_draws,
    bit-identical to NumPy): (Omega_L^T (nu x m), Omega_R (nu x n), ok flag),
    or None when NumPy's ziggurat tables are not available.  ``ok_ptr``: a
    device int* (e.g. a status word) that receives the stitching flag instead
    of a fresh tensor (the returned flag is then None)."""
    st = np.random.PCG64(check_seed(seed)).state["state"]
    return normal_draws_device(int(st["state"]), int(st["inc"]), n, m, nu, dtype, ok_ptr=ok_ptr)


def normal_draws_device(s: int, inc: int, n: int, m: int, nu: int, dtype: str, ok_ptr: int | None = None):
    """NumPy's standard_normal stream from PCG64 state ``s`` / increment ``inc``
    on the device: m*nu draws into (nu x m) transposed, then nu*n into (nu x n)
    (the Omega_L^T / Omega_R layout of sketch_draws); see sketch_draws_device.
    Asynchronous: the ziggurat tail draws use the device restatement of the C
    library's log1p (csrc/glibc_log1p.cuh), so no value is fixed up on the host."""
    lib, torch = _lib.require_device()
    tabs = _numpy_ziggurat_tables()
    if tabs is None:
        return None
    dev = torch.cuda.current_device()
    dt = _ZIG_TABLES.get(dev)
    if dt is None:
        dt = _ZIG_TABLES[dev] = torch.from_numpy(tabs.view(np.int64).copy()).to("cuda")
    M64 = (1 << 64) - 1
    tdt = _lib.torch_dtype(dtype)
    olt = torch.empty((nu, m), dtype=tdt, device="cuda")
    orr = torch.empty((nu, n), dtype=tdt, device="cuda")
    ok = None
    if ok_ptr is None:
        ok = _lib.zeros(1, torch.int32)
        ok_ptr = ok.data_ptr()
    cap = int(lib.nenmf_sketch_tail_capacity(n, m, nu))
    ws = _lib.workspace(lib.nenmf_sketch_draws_workspace_bytes(n, m, nu) + 8 * (1 + 2 * cap) + 256)
    # the tail list (diagnostics only) lives at the end of the workspace
    off = (ws.numel() - 8 * (1 + 2 * cap)) // 256 * 256
    rc = lib.nenmf_sketch_draws(_lib.code_of(dtype), dt.data_ptr(), s & M64, s >> 64, inc & M64, inc >> 64, n, m,
                                nu, olt.data_ptr(), orr.data_ptr(), ok_ptr, ws.data_ptr() + off, ws.data_ptr(),
                                off, _lib.stream_handle())
    _lib.check(rc, "sketch_draws")
    return olt, orr, ok


# status word 1 of a sketch's status buffer carries two device flags, read
# with the sketch's own status in ONE synchronisation at its end
_OK_OFF, _NZ_OFF = 0, 4


def rsi_device(Xd, nu: int, q: int, seed: int, prepared=None, draws=None, power: bool = False, status=None,
               check: bool = True):
    """Device RSI on a resident X (CUDA tensor).  Returns (L, Rt, status)
    tensors; Rt is R transposed (nu x m).  ``prepared`` is an optional
    ``_ops.prepare_x`` copy of Xd (made once, reused by the compression pass).
    The Gaussian draws are made on the device (bit-identical to NumPy's
    stream) with no synchronisation; ``status`` (2 words, zeroed) receives the
    sketch status in word 0 and the draws' stitching flag in word 1.  With
    ``check`` the status is read once at the end, and in the never-observed
    case that the device stream could not be stitched the draws are redone on
    the host and the sketch recomputed."""
    _, torch = _lib.require_device()
    n, m = Xd.shape
    dtype = "fp64" if Xd.dtype == torch.float64 else "fp32"
    if status is None:
        status = _lib.new_status(2)
    L = torch.empty((nu, n), dtype=Xd.dtype, device="cuda")
    Rt = torch.empty((nu, m), dtype=Xd.dtype, device="cuda")
    run = _ops.power_iteration if power else _ops.rsi  # compression.py:144-176 / :120-141
    if draws is not None:
        dev, own = draws, False
    else:
        dev, own = sketch_draws_device(n, m, nu, seed, dtype, ok_ptr=_lib.status_ptr(status, 1) + _OK_OFF), True
    if dev is not None:
        om_lt, om_r, ok = dev
        run(Xd, om_lt, om_r, q, L, Rt, status, Xp=prepared)
        if not check:
            return L, Rt, status
        stitched = int(_lib.read_status(status)[1]["code"]) == 1 if own else bool(ok.item())
        if stitched:
            return L, Rt, status
    omega_l, omega_r = sketch_draws(n, m, nu, seed)
    om_lt = _lib.to_device(np.ascontiguousarray(omega_l.T), dtype)
    om_r = _lib.to_device(omega_r, dtype)
    _lib.zero_(status[:_lib.STATUS_BYTES])
    run(Xd, om_lt, om_r, q, L, Rt, status, Xp=prepared)
    return L, Rt, status


def _x_key(Xd):
    return (Xd.data_ptr(), tuple(Xd.shape), tuple(Xd.stride()), Xd.dtype, Xd._version)


def prepared_for(sketch: "SketchPair", Xd):
    """The prepared copy of Xd cached on ``sketch`` by subspace_iteration_pair
    when it was computed from this very tensor (same storage, unmodified)."""
    hit = sketch.device.get("prepared")
    if hit is not None and hit[0] == _x_key(Xd):
        return hit[1]
    return None


def _is_device_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def subspace_iteration_pair(X, nu: int, q: int, seed: int, *, dtype: str = "fp64") -> SketchPair:
    """Randomized subspace iteration with a QR after every product
    (compression.py:120-141), on the GPU.  Returns NumPy L = Q_col^T and
    R = Q_row like the reference; the device copies are cached on the pair.
    Extension: for X given as a CUDA tensor the pair holds CUDA tensors (L,
    and R as a view of R^T) and the sketch never leaves the device."""
    return _iterated_pair(X, nu, q, seed, dtype, SUBSPACE_ITERATION)


def power_iteration_pair(X, nu: int, q: int, seed: int, *, dtype: str = "fp64") -> SketchPair:
    """Randomized power iteration: the same draws and alternating products as
    subspace_iteration_pair, orthonormalised only once at the end
    (compression.py:144-176), on the GPU.  An iterate that overflows at step k
    raises NumericalCollapseError(iteration=k) (FP32 tracks power-of-two scale
    factors so that the reference's fp64 overflow step is reproduced); a zero
    column after the last step raises it with iteration=q."""
    return _iterated_pair(X, nu, q, seed, dtype, POWER_ITERATION)


def _iterated_pair(X, nu: int, q: int, seed: int, dtype: str, scheme: str) -> SketchPair:
    power = scheme == POWER_ITERATION
    what = "power iteration" if power else "subspace iteration"
    if not _is_device_tensor(X):
        Xh = as_matrix(X, "X")
        n, m = Xh.shape
        _check_iteration_inputs(n, m, nu, q, bool(Xh.any()))
        _lib.require_device()
        Xd = _lib.to_device(Xh, dtype)
        L, Rt, status = rsi_device(Xd, nu, q, seed, power=power)
        st = _lib.read_status(status)[0]
        if st["code"] != 0:
            raise_for_status(int(st["code"]), int(st["iteration"]), what)
        pair = SketchPair(L=_lib.to_host(L), R=np.ascontiguousarray(_lib.to_host(Rt).T), nu=nu,
                          scheme=scheme, q=q, seed=seed)
        pair.device[dtype] = (L, Rt)
        return pair
    # device-resident X (extension): no host round trip inside the sketch.  The
    # X != 0 check (compression.py:116-117) is a device flag raised by the one
    # read of X that prepares it (FP32) or by a flag scan (FP64), read together
    # with the sketch status in the single synchronisation at the end; the
    # host-side checks keep the reference's order before any launch.
    Xd = X
    dtype = "fp64" if str(X.dtype).endswith("float64") else "fp32"
    n, m = X.shape
    _check_iteration_inputs(n, m, nu, q, True)
    _lib.require_device()
    status = _lib.new_status(2)
    nz_ptr = _lib.status_ptr(status, 1) + _NZ_OFF
    Xp = _ops.prepare_x(Xd, nu, nonzero_ptr=nz_ptr)
    if Xp is None:
        _ops.scan_flags(Xd, nonzero_ptr=nz_ptr)
    L, Rt, status = rsi_device(Xd, nu, q, seed, prepared=Xp, power=power, status=status, check=False)
    sts = _lib.read_status(status)
    if int(sts[1]["iteration"]) == 0:
        raise ZeroMatrixError("cannot sketch the zero matrix")
    if int(sts[1]["code"]) != 1:  # device draws not stitched (never observed): host draws, same sketch
        _lib.zero_(status[:_lib.STATUS_BYTES])
        L, Rt, status = rsi_device(Xd, nu, q, seed, prepared=Xp, power=power, status=status,
                                   draws=_host_draws(n, m, nu, seed, dtype))
        sts = _lib.read_status(status)
    if sts[0]["code"] != 0:
        raise_for_status(int(sts[0]["code"]), int(sts[0]["iteration"]), what)
    # the pair keeps device tensors (L: nu x n, R: an m x nu view of R^T)
    pair = SketchPair(L=L, R=Rt.t(), nu=nu, scheme=scheme, q=q, seed=seed)
    pair.device[dtype] = (L, Rt)
    if Xp is not None:
        pair.device["prepared"] = (_x_key(Xd), Xp)
    return pair


def _host_draws(n, m, nu, seed, dtype):
    omega_l, omega_r = sketch_draws(n, m, nu, seed)
    return (_lib.to_device(np.ascontiguousarray(omega_l.T), dtype), _lib.to_device(omega_r, dtype),
            _lib.torch_mod().ones(1, dtype=_lib.torch_mod().int32, device="cuda"))


def sketch_on_device(sketch: SketchPair, dtype: str):
    """(L, R^T) of a sketch as CUDA tensors of ``dtype`` (cached)."""
    hit = sketch.device.get(dtype)
    if hit is not None:
        return hit
    L = _lib.to_device(np.ascontiguousarray(sketch.L), dtype)
    Rt = _lib.to_device(np.ascontiguousarray(np.asarray(sketch.R, dtype=np.float64).T), dtype)
    sketch.device[dtype] = (L, Rt)
    return L, Rt


def compress_device(Xd, L, Rt, prepared=None):
    """(X_L, X_R^T) on the device from one fused pass over X."""
    torch = _lib.torch_mod()
    nu = L.shape[0]
    n, m = Xd.shape
    XL = torch.empty((nu, m), dtype=Xd.dtype, device="cuda")
    XRt = torch.empty((nu, n), dtype=Xd.dtype, device="cuda")
    _ops.compress(Xd, L, Rt, XL, XRt, Xp=prepared)
    return XL, XRt


def compress_problem(X, sketch: SketchPair, *, dtype: str = "fp64") -> CompressedProblem:
    """X_L = L X and X_R = X R (compression.py:179-188), one pass on the GPU."""
    X = as_matrix(X, "X")
    n, m = X.shape
    if np.shape(sketch.L) != (sketch.nu, n) or np.shape(sketch.R) != (m, sketch.nu):
        raise DimensionError(
            f"sketch shapes L {np.shape(sketch.L)}, R {np.shape(sketch.R)} do not match "
            f"data {n}x{m} at target rank {sketch.nu}")
    _lib.require_device()
    Xd = _lib.to_device(X, dtype)
    L, Rt = sketch_on_device(sketch, dtype)
    XL, XRt = compress_device(Xd, L, Rt)
    return CompressedProblem(X_L=_lib.to_host(XL), X_R=np.ascontiguousarray(_lib.to_host(XRt).T))


def _host(M):
    return _lib.to_host(M) if _is_device_tensor(M) else M


def save_sketch(sketch: SketchPair, directory) -> None:
    """L and R as NMFB matrices plus a JSON provenance header (compression.py:191-198)."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    write_nmfb(directory / "L.nmfb", _host(sketch.L))
    write_nmfb(directory / "R.nmfb", _host(sketch.R))
    meta = {"nu": sketch.nu, "scheme": sketch.scheme, "q": sketch.q, "seed": sketch.seed}
    (directory / "sketch.json").write_text(json.dumps(meta, sort_keys=True, indent=2) + "\n")


def load_sketch(directory) -> SketchPair:
    """Inverse of :func:`save_sketch` (compression.py:201-210)."""
    directory = Path(directory)
    meta = json.loads((directory / "sketch.json").read_text())
    return SketchPair(L=read_nmfb(directory / "L.nmfb"), R=read_nmfb(directory / "R.nmfb"), nu=int(meta["nu"]),
                      scheme=str(meta["scheme"]), q=int(meta["q"]), seed=int(meta["seed"]))
