"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture stores the reference's own inputs and outputs for one case.
Nothing from the reference's source is copied; it is imported and executed.
Inner-iteration counts are observed by wrapping ``nenmf.nnls.alpha_next``,
which ``nnls.py:204`` calls once per non-breaking inner iteration.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import nenmf  # noqa: E402  (the reference package)
import nenmf.nnls as ref_nnls  # noqa: E402
from nenmf.cli import derive_seed  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

from paper_1812_04315_b200 import workloads  # noqa: E402  (host-side generators only)


class _Counter:
    def __init__(self):
        self.calls = 0
        self._orig = ref_nnls.alpha_next

    def __enter__(self):
        def counted(a):
            self.calls += 1
            return self._orig(a)

        ref_nnls.alpha_next = counted
        return self

    def __exit__(self, *exc):
        ref_nnls.alpha_next = self._orig


def save(name, **arrays):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"wrote {path.relative_to(REPO)} ({path.stat().st_size} bytes)")


def gen_alpha():
    a = [1.0]
    for _ in range(50):
        a.append(nenmf.alpha_next(a[-1]))
    save("alpha", alpha=np.array(a))


def gen_spectral():
    mats, ests, ests_long = [], [], []
    shapes = [(50, 15), (15, 50), (30, 1), (2, 2), (60, 10), (40, 8)]
    for i, (r, c) in enumerate(shapes):
        G = nenmf.gaussian_matrix(r, c, 30 + i)
        mats.append(G)
        ests.append(nenmf.spectral_norm_sq(G))
        ests_long.append(nenmf.spectral_norm_sq(G, max_iters=5000))
    arrs = {f"G{i}": M for i, M in enumerate(mats)}
    save("spectral", count=np.array(len(mats)), est=np.array(ests),
         est_long=np.array(ests_long), **arrs)


def gen_nnls():
    cases = {}
    specs = []
    # (r, p, c, seed, max_iter, grad_tol, safety, signed_B)
    for seed in range(4):
        specs.append((30, 10, 8, 100 + seed, 500, 1e-4, 1.0, True))
    for max_iter in (1, 2, 5, 50):
        specs.append((12, 5, 7, 200, max_iter, 1e-4, 1.0, True))
    specs.append((30, 10, 8, 300, 20000, 1e-12, 1.0, True))
    specs.append((40, 7, 90, 301, 500, 1e-4, 1.0, False))
    specs.append((25, 12, 300, 302, 200, 1e-6, 1.5, False))
    specs.append((6, 9, 20, 303, 100, 1e-4, 1.0, True))      # r < p
    specs.append((1, 1, 1, 304, 10, 1e-4, 1.0, True))
    meta = []
    for i, (r, p, c, seed, max_iter, tol, saf, signed) in enumerate(specs):
        rng = np.random.default_rng(seed)
        A = rng.standard_normal((r, p))
        B = rng.standard_normal((r, c))
        if not signed:
            B = np.abs(B)
        F0 = rng.random((p, c))
        cfg = nenmf.InnerSolverConfig(max_iter=max_iter, grad_tol=tol, lipschitz_safety=saf)
        with _Counter() as cnt:
            F = nenmf.solve_nnls(A, B, F0, cfg)
        cases[f"A{i}"] = A
        cases[f"B{i}"] = B
        cases[f"F0_{i}"] = F0
        cases[f"F{i}"] = F
        meta.append([max_iter, tol, saf, cnt.calls])
    save("nnls", count=np.array(len(specs)), meta=np.array(meta, dtype=np.float64), **cases)


def gen_rsi():
    cases = {}
    specs = [
        ("noisy", nenmf.generate_problem(200, 180, 10, 30.0, seed=5).X, 20, 4, 6),
        ("noisy_q1", nenmf.generate_problem(150, 150, 10, 30.0, seed=22).X, 20, 1, 23),
        ("tall", nenmf.generate_problem(600, 40, 5, 20.0, seed=7).X, 12, 2, 8),
        ("wide", nenmf.generate_problem(40, 500, 5, 20.0, seed=9).X, 10, 3, 10),
    ]
    rng = np.random.default_rng(20)
    lowrank = rng.random((300, 15)) @ rng.random((15, 300))
    specs.append(("lowrank", lowrank, 25, 4, 21))
    for name, X, nu, q, seed in specs:
        sk = nenmf.subspace_iteration_pair(X, nu, q, seed)
        comp = nenmf.compress_problem(X, sk)
        cases[f"{name}_X"] = X
        cases[f"{name}_L"] = sk.L
        cases[f"{name}_R"] = sk.R
        cases[f"{name}_XL"] = comp.X_L
        cases[f"{name}_XR"] = comp.X_R
        cases[f"{name}_par"] = np.array([nu, q, seed], dtype=np.int64)
    save("rsi", names=np.array([s[0] for s in specs]), **cases)


def gen_power():
    """power_iteration_pair (compression.py:144-176): sketches, and the step
    at which an overflowing iterate raises NumericalCollapseError."""
    cases = {}
    specs = [
        ("noisy", nenmf.generate_problem(200, 180, 10, 30.0, seed=5).X, 20, 2, 6),
        ("tall", nenmf.generate_problem(600, 40, 5, 20.0, seed=7).X, 12, 1, 8),
        ("wide", nenmf.generate_problem(40, 500, 5, 20.0, seed=9).X, 10, 3, 10),
    ]
    for name, X, nu, q, seed in specs:
        sk = nenmf.power_iteration_pair(X, nu, q, seed)
        cases[f"{name}_X"] = X
        cases[f"{name}_L"] = sk.L
        cases[f"{name}_R"] = sk.R
        cases[f"{name}_par"] = np.array([nu, q, seed], dtype=np.int64)
    # overflow: a large-scale X makes X^T X ... leave the fp64 range at some step
    Xo = nenmf.generate_problem(120, 100, 4, 30.0, seed=3).X * 1e40
    try:
        nenmf.power_iteration_pair(Xo, 6, 8, 4)
        step = -1
    except nenmf.NumericalCollapseError as exc:
        step = exc.iteration
    cases["overflow_X"] = Xo
    cases["overflow_par"] = np.array([6, 8, 4, step], dtype=np.int64)
    save("power", names=np.array([s[0] for s in specs]), **cases)


def _trace(records):
    return np.array([[r.outer_iter, r.rre, r.objective] for r in records])


def gen_factorize():
    cases = {}
    # compressed + vanilla on a small noisy problem, fixed iteration count
    inst = nenmf.generate_problem(120, 110, 8, 30.0, seed=20)
    init = nenmf.init_factors(120, 110, 8, seed=21)
    sk = nenmf.subspace_iteration_pair(inst.X, 16, 4, seed=22)
    cfg = nenmf.OuterConfig(inner=nenmf.InnerSolverConfig(max_iter=500),
                            time_budget_seconds=0.0, max_outer_iterations=12)
    for method in ("vanilla", "compressed"):
        rec = nenmf.TraceRecorder()
        if method == "vanilla":
            out = nenmf.factorize_vanilla(inst.X, init, cfg, observer=rec,
                                          clock=nenmf.IterationClock())
        else:
            out = nenmf.factorize_compressed(inst.X, sk, init, cfg, observer=rec,
                                             clock=nenmf.IterationClock())
        cases[f"small_{method}_trace"] = _trace(rec.records)
        cases[f"small_{method}_G"] = out.G
        cases[f"small_{method}_F"] = out.F
    cases["small_X"] = inst.X
    cases["small_G0"] = init.G
    cases["small_F0"] = init.F
    cases["small_L"] = sk.L
    cases["small_R"] = sk.R

    # trace cadence (trace_every=3, 7 outer) on vanilla
    inst2 = nenmf.generate_problem(30, 30, 3, 30.0, seed=12)
    init2 = nenmf.init_factors(30, 30, 3, seed=13)
    cfg2 = nenmf.OuterConfig(time_budget_seconds=0.0, max_outer_iterations=7, trace_every=3)
    rec = nenmf.TraceRecorder()
    out = nenmf.factorize_vanilla(inst2.X, init2, cfg2, observer=rec, clock=nenmf.IterationClock())
    cases["cadence_X"] = inst2.X
    cases["cadence_G0"] = init2.G
    cases["cadence_F0"] = init2.F
    cases["cadence_trace"] = _trace(rec.records)
    cases["cadence_G"] = out.G
    cases["cadence_F"] = out.F
    save("factorize", **cases)


def gen_config1():
    """BASELINE config 1 exactly (n=m=1000, p=10, nu=20, q=4, inner 10, 50 outer)."""
    w = workloads.make_workload(1)
    X, G0, F0 = w.X, w.G0, w.F0
    sk = nenmf.subspace_iteration_pair(X, w.nu, w.q, w.sketch_seed)
    init = nenmf.FactorPair(G=G0, F=F0, p=w.p)
    cfg = nenmf.OuterConfig(inner=nenmf.InnerSolverConfig(max_iter=w.inner),
                            time_budget_seconds=0.0, max_outer_iterations=w.outer)
    rec_c, rec_v = nenmf.TraceRecorder(), nenmf.TraceRecorder()
    out_c = nenmf.factorize_compressed(X, sk, init, cfg, observer=rec_c,
                                       clock=nenmf.IterationClock())
    out_v = nenmf.factorize_vanilla(X, init, cfg, observer=rec_v,
                                    clock=nenmf.IterationClock())
    save("config1",
         L=sk.L, R=sk.R,
         compressed_trace=_trace(rec_c.records), compressed_G=out_c.G, compressed_F=out_c.F,
         vanilla_trace=_trace(rec_v.records), vanilla_G=out_v.G, vanilla_F=out_v.F,
         x_checksum=np.array([X.sum(), (X * X).sum()]))


def gen_seeds():
    base = [0, 1, 7, 1234, 2**63 + 5]
    out = np.array([[derive_seed(b, s) for s in (0, 1, 2)] for b in base], dtype=np.uint64)
    init = nenmf.init_factors(7, 9, 3, 11)
    om = np.random.default_rng(17)
    save("seeds", base=np.array(base, dtype=np.uint64), derived=out,
         init_G=init.G, init_F=init.F,
         uniform=nenmf.uniform_matrix(5, 4, 3), gauss=nenmf.gaussian_matrix(4, 5, 3))


if __name__ == "__main__":
    gen_alpha()
    gen_spectral()
    gen_nnls()
    gen_rsi()
    gen_power()
    gen_factorize()
    gen_config1()
    gen_seeds()
