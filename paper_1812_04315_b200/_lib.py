"""ctypes binding of libnenmf_b200.so plus the device plumbing around it.

PyTorch is used only as the container: CUDA memory, the current stream and
pinned host staging.  Every computation is a call into the C ABI declared in
``include/nenmf_b200.h``.  There is no CPU fallback: when the library or a
CUDA device is missing, every compute entry point raises ``BackendError``.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

from .errors import BackendError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libnenmf_b200.so"

F64, F32 = 0, 1
DTYPES = {"fp64": F64, "fp32": F32}

_vp, _i64, _i32, _dbl, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_size_t

# name -> (restype, argtypes); mirrors include/nenmf_b200.h
_SIGS = {
    "nenmf_abi_version": (_i32, []),
    "nenmf_status_string": (C.c_char_p, [_i32]),
    "nenmf_device_sm_count": (_i32, []),
    "nenmf_launch_count": (C.c_ulonglong, []),
    "nenmf_debug_nnls_trace": (_i32, [_vp, _i32]),
    "nenmf_solve_nnls_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_solve_nnls": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _i32, _dbl, _dbl,
                                _vp, _i32, _i32, _dbl, _vp, _vp, _sz, _vp]),
    "nenmf_solve_nnls_next_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64, _i64]),
    "nenmf_solve_nnls_next": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _i32, _dbl, _dbl,
                                     _vp, _i32, _i32, _dbl, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_solve_nnls_prepared_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_group_xch_bytes": (_sz, []),
    "nenmf_generate_workspace_bytes": (_sz, []),
    "nenmf_generate_norms": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_generate_write": (_i32, [_i32, _vp, _vp, _vp, _i64, _i64, _i64, _dbl, _vp, _vp]),
    "nenmf_solve_nnls_group_check": (_i32, [_i32, _i64, _i64, _i64, _i64, _i32, _i32, _i32]),
    "nenmf_solve_nnls_group": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _i32, _dbl, _dbl,
                                      _vp, _i32, _i32, _dbl, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_ipc_handle": (_i32, [_vp, _vp]),
    "nenmf_ipc_open": (_i32, [_vp, _vp]),
    "nenmf_ipc_close": (_i32, [_vp]),
    "nenmf_solve_nnls_prepared": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _dbl,
                                         _dbl, _vp, _i32, _i32, _dbl, _vp, _vp, _sz, _vp]),
    "nenmf_spectral_norm_sq_workspace_bytes": (_sz, [_i32, _i64, _i64]),
    "nenmf_spectral_norm_sq": (_i32, [_i32, _vp, _i64, _i64, _vp, _i32, _i32, _dbl, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_gradient_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_gradient": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_reduce_workspace_bytes": (_sz, [_i64]),
    "nenmf_pg_norm_sq": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_sumsq": (_i32, [_i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_scan_flags": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "nenmf_transpose": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp]),
    "nenmf_zero": (_i32, [_vp, _sz, _vp]),
    "nenmf_convert_f64": (_i32, [_i32, _vp, _i64, _vp, _vp, _vp]),
    "nenmf_uniform_draws": (_i32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _i64, _vp, _vp, _vp]),
    "nenmf_residual_sumsq_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_residual_sumsq": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_residual_sumsq_prepared_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_residual_sumsq_prepared": (_i32, [_i32, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_abt_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_abt": (_i32, [_i32, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_dual_pass_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_dual_pass": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_orthonormalize_workspace_bytes": (_sz, [_i64, _i64]),
    "nenmf_orthonormalize": (_i32, [_i32, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_rsi_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_rsi": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_compress": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_sketch_draws_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "nenmf_sketch_tail_capacity": (_i64, [_i64, _i64, _i64]),
    "nenmf_sketch_draws": (_i32, [_i32, _vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _i64, _i64, _i64,
                                  _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_panel_gram_workspace_bytes": (_sz, [_i32, _i64, _i64]),
    "nenmf_panel_gram": (_i32, [_i32, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "nenmf_panel_factor": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "nenmf_panel_trsm": (_i32, [_i32, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _i32, _vp]),
    "nenmf_debug_xpass_timing": (None, [_i32]),
    "nenmf_debug_xpass_ms": (_i32, [C.POINTER(C.c_double)]),
    "nenmf_prepared_x_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_prepare_x": (_i32, [_i32, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "nenmf_prepare_x_checked": (_i32, [_i32, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "nenmf_dual_pass_prepared_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_dual_pass_prepared": (_i32, [_i32, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "nenmf_rsi_prepared_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "nenmf_rsi_prepared": (_i32, [_i32, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz,
                                  _vp]),
    "nenmf_power_iteration": (_i32, [_i32, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp,
                                     _sz, _vp]),
    "nenmf_compress_prepared": (_i32, [_i32, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: Path | str | None = None):
    """Load libnenmf_b200.so (no device needed) and declare its signatures."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise BackendError(
                f"{p} is missing: build it with `python -m paper_1812_04315_b200._build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.nenmf_abi_version() != 1:
            raise BackendError("libnenmf_b200 ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def torch_mod():
    import torch  # deferred: importing torch is slow on a cold box

    return torch


def require_device():
    """The CUDA library and a CUDA device, or BackendError (no CPU fallback)."""
    lib = load_library()
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise BackendError("no CUDA device: the NeNMF hot path runs only on the GPU (no CPU fallback)")
    return lib, torch


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise_for_status(rc, what=f"{what}: {load_library().nenmf_status_string(rc).decode()}")


def torch_dtype(dtype: str):
    torch = torch_mod()
    if dtype == "fp64":
        return torch.float64
    if dtype == "fp32":
        return torch.float32
    raise ValueError(f"dtype must be 'fp64' or 'fp32', got {dtype!r}")


def code_of(dtype: str) -> int:
    try:
        return DTYPES[dtype]
    except KeyError:
        raise ValueError(f"dtype must be 'fp64' or 'fp32', got {dtype!r}") from None


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle() -> int:
    torch = torch_mod()
    return torch.cuda.current_stream().cuda_stream


# ----------------------------------------------------------------- workspace
_tls = threading.local()


def workspace(nbytes: int):
    """Thread-local, growable device scratch (calls from different host threads
    never share scratch, cli.py:324-331 runs seeds concurrently)."""
    torch = torch_mod()
    dev = torch.cuda.current_device()
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    buf = cache.get(dev)
    nbytes = max(int(nbytes), 256)
    if buf is None or buf.numel() < nbytes:
        # the stream may still use the old buffer; torch's caching allocator
        # keeps it alive until the stream's work that used it has completed
        buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device="cuda")
        cache[dev] = buf
    return buf


# ------------------------------------------------------------- rank groups
class GroupStruct(C.Structure):
    """nenmf_group (include/nenmf_b200.h): one solve split over R ranks."""

    _fields_ = [("ranks", C.c_int), ("rank0", C.c_int), ("nvr", C.c_int), ("watchdog_s", C.c_int),
                ("col0", C.c_int64 * 9), ("xch", C.c_void_p * 8), ("epoch", C.c_uint64)]


# -------------------------------------------------------------- status words
STATUS_BYTES = 64
STATUS_FIELDS = np.dtype([("code", "<i4"), ("iteration", "<i4"), ("inner_iters", "<i4"),
                          ("returned_best", "<i4"), ("lipschitz", "<f8"), ("best_partial", "<f8"),
                          ("pg_ref", "<f8"), ("resid", "<f8", (2,)), ("pad", "<f8")])
assert STATUS_FIELDS.itemsize == STATUS_BYTES


def zeros(shape, dtype):
    """A zeroed CUDA tensor by cudaMemsetAsync (nenmf_zero): no fill kernel."""
    torch = torch_mod()
    t = torch.empty(shape, dtype=dtype, device="cuda")
    check(load_library().nenmf_zero(t.data_ptr(), t.numel() * t.element_size(), stream_handle()), "zero")
    return t


def zero_(t):
    check(load_library().nenmf_zero(t.data_ptr(), t.numel() * t.element_size(), stream_handle()), "zero")
    return t


def new_status(count: int = 1):
    return zeros(count * STATUS_BYTES, torch_mod().uint8)


def status_ptr(buf, index: int = 0) -> int:
    return buf.data_ptr() + index * STATUS_BYTES


def read_status(buf) -> np.ndarray:
    """Synchronising read of status words (structured numpy array)."""
    host = buf.cpu().numpy()
    return host.view(STATUS_FIELDS)


# ------------------------------------------------- seeded power start vectors
_POWER_SEED = 0x9E3779B97F4A7C15  # matrix.py:24
_power_cache: dict = {}
_power_lock = threading.Lock()
POWER_DRAWS = 4  # start vector + re-draws shipped to the device (see header)


def power_vectors(k: int, count: int = POWER_DRAWS):
    """Device float64 (count x k): the reference's start vector and re-draws,
    each normalised exactly as matrix.py:139-140,148-149 does."""
    torch = torch_mod()
    key = (int(k), int(count), torch.cuda.current_device())
    with _power_lock:
        hit = _power_cache.get(key)
        if hit is not None:
            return hit
        gen = np.random.default_rng(_POWER_SEED)
        rows = []
        for _ in range(count):
            v = gen.standard_normal(k)
            v /= np.linalg.norm(v)
            rows.append(v)
        dev = torch.from_numpy(np.ascontiguousarray(np.array(rows))).to("cuda")
        _power_cache[key] = dev
        return dev


# --------------------------------------------------------- host <-> device
def to_device(a, dtype: str):
    """numpy (or torch) 2-D array -> contiguous CUDA tensor of ``dtype``."""
    torch = torch_mod()
    tdt = torch_dtype(dtype)
    if isinstance(a, torch.Tensor):
        t = a.to(device="cuda", dtype=tdt)
        return t.contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64 if dtype == "fp64" else np.float32)
    return torch.from_numpy(arr).to("cuda", non_blocking=False)


def to_host(t) -> np.ndarray:
    return t.detach().to("cpu", dtype=torch_mod().float64).numpy()
