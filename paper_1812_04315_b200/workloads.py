"""Seeded synthetic inputs for the five BASELINE.json configs.

The reference benchmarks on synthetic data too (``synthetic.py:47-95``,
``PAPER.md:71-72``); no public dataset is involved.  Configs 1-4 are drawn on
the host with NumPy so that the CPU oracle sees bit-identical inputs; config 5
(40 GB) is generated on the device and only its scaled proxy exists on host.

Seeds follow the reference CLI's derived streams (``cli.py:50-52,111-114``):
stream 0 = data, 1 = initial factors, 2 = sketch.  Initial factors must NOT
reuse the data seed (SURVEY §8c trap: ``init_factors(s)`` equals
``generate_problem(s)``'s ground truth).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .matrix import open_uniform

BASE_SEED = 1234


def derive_seed(base: int, stream: int) -> int:
    """Same derivation as the reference CLI (``cli.py:111-114``)."""
    seq = np.random.SeedSequence(entropy=int(base), spawn_key=(int(stream),))
    return int(seq.generate_state(1, np.uint64)[0])


@dataclass
class Workload:
    cfg: int
    n: int
    m: int
    p: int
    nu: int
    q: int
    dtype: str          # "fp64" or "fp32": the GPU arithmetic of this config
    inner: int          # InnerSolverConfig.max_iter
    outer: int          # fixed outer-iteration count
    X: np.ndarray       # float64, already rounded to ``dtype`` when fp32
    G0: np.ndarray
    F0: np.ndarray
    sketch_seed: int
    description: str


# n, m, p, nu(=p'), q, dtype, inner, outer
SPECS = {
    1: (1000, 1000, 10, 20, 4, "fp64", 10, 50),
    2: (10000, 10000, 20, 30, 4, "fp32", 500, 100),
    3: (50000, 20000, 50, 60, 4, "fp32", 500, 20),
    4: (400000, 2000, 30, 40, 4, "fp32", 500, 10),
    5: (100000, 100000, 16, 26, 4, "fp32", 500, 50),
}


def _round(M: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "fp32":
        return M.astype(np.float32).astype(np.float64)
    return M


def make_data(cfg: int, n: int | None = None, m: int | None = None,
              p: int | None = None, seed: int = BASE_SEED) -> np.ndarray:
    """X for config ``cfg`` (optionally at a scaled shape), float64."""
    n0, m0, p0 = SPECS[cfg][:3]
    n = n0 if n is None else n
    m = m0 if m is None else m
    p = p0 if p is None else p
    rng = np.random.default_rng(derive_seed(seed, 0))
    if cfg in (1, 5):
        G = open_uniform(rng, n, p)
        F = open_uniform(rng, p, m)
        return G @ F
    if cfg == 2:
        G = open_uniform(rng, n, p)
        F = open_uniform(rng, p, m)
        X = G @ F
        # BASELINE's "1% iid |N(0, sigma)|": sigma = 0.01 * mean(GF) (declared choice)
        sigma = 0.01 * float(X.mean())
        X += np.abs(rng.standard_normal((n, m))) * sigma
        return X
    if cfg == 3:
        G = rng.exponential(1.0, (n, p))
        F = open_uniform(rng, p, m)
        F[rng.random((p, m)) < 0.7] = 0.0
        return G @ F
    if cfg == 4:
        G = open_uniform(rng, n, p)
        F = open_uniform(rng, p, m)
        X = G @ F
        noise = rng.standard_normal((n, m))
        # exact 20 dB SNR as synthetic.py:77-81, then clipped at 0 (BASELINE cfg 4)
        noise *= np.linalg.norm(X) * 10.0 ** (-20.0 / 20.0) / np.linalg.norm(noise)
        X += noise
        np.maximum(X, 0.0, out=X)
        return X
    raise ValueError(f"unknown config {cfg}")


def make_workload(cfg: int, *, n: int | None = None, m: int | None = None,
                  seed: int = BASE_SEED, dtype: str | None = None) -> Workload:
    n0, m0, p, nu, q, dt, inner, outer = SPECS[cfg]
    n = n0 if n is None else n
    m = m0 if m is None else m
    dt = dt if dtype is None else dtype
    X = _round(make_data(cfg, n, m, p, seed), dt)
    rng = np.random.default_rng(derive_seed(seed, 1))
    G0 = _round(open_uniform(rng, n, p), dt)
    F0 = _round(open_uniform(rng, p, m), dt)
    desc = (f"cfg{cfg}: n={n} m={m} p={p} p'={nu} q={q} {dt} inner={inner} "
            f"outer={outer} seed=derive_seed({seed},0/1/2)")
    return Workload(cfg, n, m, p, nu, q, dt, inner, outer, X, G0, F0,
                    derive_seed(seed, 2), desc)


def rsi_bytes(n: int, m: int, q: int, itemsize: int) -> int:
    """Algorithmic HBM bytes of one RSI sketch + compress:
    X is read once per dependent stage, (2q+2) stages."""
    return (2 * q + 2) * n * m * itemsize


def rsi_flops(n: int, m: int, q: int, nu: int) -> int:
    return (4 * q + 4) * 2 * n * m * nu


def snr_db(clean: np.ndarray, noisy: np.ndarray) -> float:
    return 10.0 * math.log10((np.linalg.norm(clean) / np.linalg.norm(noisy - clean)) ** 2)


def device_shard(cfg: int, world: int, rank: int, *, n: int | None = None, m: int | None = None,
                 seed: int = BASE_SEED, dtype: str = "fp32"):
    """This rank's row block of config ``cfg``'s X = G F generated ON THE
    DEVICE (BASELINE cfg 5: 40 GB, never on the host), plus the full initial
    factors.  G (n x p) and F (p x m) are U(0,1) from a Philox generator seeded
    with derive_seed(seed, 0) on every rank (identical on all ranks); zeros
    are mapped to the smallest positive draw (the open-interval convention of
    matrix.py:73-82).  X_r = G[rows] F by one plain GEMM (data setup, not the
    hot path).  Initial factors from derive_seed(seed, 1).  Returns
    (X_local, row0, n, m, p, nu, q, inner, outer, G0, F0, sketch_seed)."""
    import torch

    from .sharded import row_block

    if cfg != 5:
        raise ValueError("device generation is defined for config 5 (noiseless U(0,1) G F)")
    n0, m0, p, nu, q, _dt, inner, outer = SPECS[cfg]
    n = n0 if n is None else n
    m = m0 if m is None else m
    tdt = torch.float32 if dtype == "fp32" else torch.float64

    def uni(gen, shape):
        u = torch.rand(shape, generator=gen, device="cuda", dtype=torch.float64)
        return u.clamp_(min=2.0 ** -53).to(tdt)

    g = torch.Generator(device="cuda")
    g.manual_seed(derive_seed(seed, 0) & ((1 << 63) - 1))
    G = uni(g, (n, p))
    F = uni(g, (p, m))
    r0, nr = row_block(n, world, rank)
    X_local = torch.mm(G[r0:r0 + nr], F).contiguous()
    del G, F
    g.manual_seed(derive_seed(seed, 1) & ((1 << 63) - 1))
    G0 = uni(g, (n, p))
    F0 = uni(g, (p, m))
    return X_local, r0, n, m, p, nu, q, inner, outer, G0, F0, derive_seed(seed, 2)
