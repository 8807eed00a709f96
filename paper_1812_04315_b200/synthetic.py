"""Problem generator of the reference (synthetic.py:47-95) on the device
(exact-SNR instances at n = 10^4 and beyond without a
host round trip).

``generate_problem_device`` consumes the reference's NumPy stream exactly:
G then F by ``Generator.random`` (open_uniform, matrix.py:73-82) and the
noise by ``standard_normal`` from the same PCG64 stream, all drawn on the
B200 bit-identical to NumPy (``nenmf_uniform_draws``; the ziggurat kernels of
the sketch).  X = G F + s N with s = ||G F|| 10^(-snr/20) / ||N|| (the
reference's exact-SNR rescale): G F is a plain library GEMM (cuBLAS through
torch), the norms and the update are this package's kernels, so X agrees
with the reference's to rounding (summation order of the GEMM and norms).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib, _ops
from .compression import normal_draws_device
from .errors import DimensionError
from .matrix import check_seed

_M64 = (1 << 64) - 1


@dataclass(frozen=True, eq=False)
class DeviceProblemInstance:
    """ProblemInstance (synthetic.py:35-44) with CUDA tensors."""

    X: object
    G_true: object
    F_true: object
    snr_db_target: float
    snr_db_realized: float
    seed: int


def _uniform(lib, torch, bitgen, count: int):
    st = bitgen.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    zero = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = lib.nenmf_uniform_draws(s & _M64, s >> 64, inc & _M64, inc >> 64, count, out.data_ptr(), zero.data_ptr(),
                                 _lib.stream_handle())
    _lib.check(rc, "uniform_draws")
    bitgen.advance(count)
    return out, zero


def _sumsq(t) -> float:
    out = _lib.torch_mod().zeros(1, dtype=_lib.torch_mod().float64, device="cuda")
    _ops.sumsq(t, out)
    return float(out.item())


def generate_problem_device(n: int, m: int, p: int, snr_db: float, seed: int, *,
                            dtype: str = "fp64") -> DeviceProblemInstance:
    """generate_problem (synthetic.py:47-95) with X, G_true, F_true on the GPU
    in ``dtype`` (the draws and the rescale run in float64, X is rounded last)."""
    if p < 1:
        raise DimensionError(f"rank must be >= 1, got {p}")
    if p > min(n, m):
        raise DimensionError(f"rank {p} exceeds min(n, m) = {min(n, m)}")
    if math.isnan(snr_db) or snr_db == -math.inf:
        raise ValueError(f"snr_db must be finite or +inf, got {snr_db}")
    lib, torch = _lib.require_device()
    bitgen = np.random.PCG64(check_seed(seed))
    G, zg = _uniform(lib, torch, bitgen, n * p)
    F, zf = _uniform(lib, torch, bitgen, p * m)
    if int(zg.item()) or int(zf.item()):
        # an exact zero (probability 2^-53 per draw): open_uniform's redraws
        # shift the stream, so take the reference's host path for this seed
        rng = np.random.default_rng(check_seed(seed))
        from .matrix import open_uniform
        Gh, Fh = open_uniform(rng, n, p), open_uniform(rng, p, m)
        G, F = torch.from_numpy(Gh).cuda(), torch.from_numpy(Fh).cuda()
        bitgen = rng.bit_generator
    G = G.view(n, p).contiguous()
    F = F.view(p, m).contiguous()
    tdt = _lib.torch_dtype(dtype)
    X = torch.empty((n, m), dtype=tdt, device="cuda")
    stream = _lib.stream_handle()
    if snr_db == math.inf:
        # G F straight into X (synthetic.py:62-66, noiseless)
        _lib.check(lib.nenmf_generate_write(_lib.code_of(dtype), G.data_ptr(), F.data_ptr(), None, n, m, p, 0.0,
                                            X.data_ptr(), stream), "generate_write")
        return DeviceProblemInstance(X=X, G_true=G.to(tdt), F_true=F.to(tdt), snr_db_target=snr_db,
                                     snr_db_realized=math.inf, seed=seed)
    st = bitgen.state["state"]
    draws = normal_draws_device(int(st["state"]), int(st["inc"]), 1, n, m, "fp64")
    if draws is None or not int(draws[2].item()):
        Nh = np.random.Generator(bitgen).standard_normal((n, m))
        noise = torch.from_numpy(Nh).cuda()
    else:
        noise = draws[0].t().contiguous()  # the first n*m draws, row-major n x m (stored transposed)
    # the exact-SNR rescale (synthetic.py:77-81) in two fused passes: both
    # norms in one read of the noise (G F formed on the fly), then X = G F + s N
    ws = _lib.workspace(lib.nenmf_generate_workspace_bytes())
    norms = _lib.zeros(2, torch.float64)
    _lib.check(lib.nenmf_generate_norms(G.data_ptr(), F.data_ptr(), noise.data_ptr(), n, m, p, norms.data_ptr(),
                                        ws.data_ptr(), ws.numel(), stream), "generate_norms")
    c2, n2 = (float(v) for v in norms.cpu())
    clean_norm, noise_norm = math.sqrt(c2), math.sqrt(n2)
    scale = clean_norm * 10.0 ** (-snr_db / 20.0) / noise_norm
    _lib.check(lib.nenmf_generate_write(_lib.code_of(dtype), G.data_ptr(), F.data_ptr(), noise.data_ptr(), n, m, p,
                                        scale, X.data_ptr(), stream), "generate_write")
    # ||s N|| = s ||N|| up to rounding (the reference forms the scaled noise's norm)
    realized = 10.0 * math.log10((clean_norm / (scale * noise_norm)) ** 2)
    return DeviceProblemInstance(X=X, G_true=G.to(tdt), F_true=F.to(tdt), snr_db_target=float(snr_db),
                                 snr_db_realized=realized, seed=seed)
