"""GPU parity of the inner solver and matrix primitives against the CPU
oracle and the reference's golden fixtures (the reference's own test cases
from test_nnls.py / test_matrix.py, run through the C ABI).

Tolerances (north_star): rel 1e-5 in FP64 mode, 1e-3 in FP32 mode."""

import numpy as np
import pytest
from scipy.optimize import nnls as scipy_nnls

import nenmf_oracle as orc
import paper_1812_04315_b200 as nm

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-5
FP32_TOL = 1e-3


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def obj(A, B, F):
    return 0.5 * np.linalg.norm(B - A @ F) ** 2


def test_solve_matches_golden_fp64(golden):
    d = golden("nnls")
    for i in range(int(d["count"])):
        max_iter, tol, saf, calls = d["meta"][i]
        cfg = nm.InnerSolverConfig(max_iter=int(max_iter), grad_tol=tol, lipschitz_safety=saf)
        rep = []
        F = nm.solve_nnls(d[f"A{i}"], d[f"B{i}"], d[f"F0_{i}"], cfg, report=rep)
        ref = d[f"F{i}"]
        assert F.shape == ref.shape
        assert rel(F, ref) <= FP64_TOL, (i, rel(F, ref))
        # objective parity is the size-independent check
        A, B = d[f"A{i}"], d[f"B{i}"]
        assert obj(A, B, F) <= obj(A, B, ref) * (1 + FP64_TOL) + 1e-300


def test_solve_iteration_counts_match(golden):
    d = golden("nnls")
    for i in range(int(d["count"])):
        max_iter, tol, saf, calls = d["meta"][i]
        cfg = nm.InnerSolverConfig(max_iter=int(max_iter), grad_tol=tol, lipschitz_safety=saf)
        rep = []
        nm.solve_nnls(d[f"A{i}"], d[f"B{i}"], d[f"F0_{i}"], cfg, report=rep)
        info = orc.SolveInfo()
        orc.nesterov_nnls(d[f"A{i}"], d[f"B{i}"], d[f"F0_{i}"], int(max_iter), tol, saf, info)
        assert abs(rep[0].inner_iters - info.iterations) <= 1, (i, rep[0].inner_iters, info.iterations)


def test_solve_fp32_mode(golden):
    d = golden("nnls")
    for i in range(int(d["count"])):
        max_iter, tol, saf, _ = d["meta"][i]
        if max_iter > 1000:
            continue
        cfg = nm.InnerSolverConfig(max_iter=int(max_iter), grad_tol=tol, lipschitz_safety=saf)
        A, B = d[f"A{i}"], d[f"B{i}"]
        F = nm.solve_nnls(A, B, d[f"F0_{i}"], cfg, dtype="fp32")
        ref = d[f"F{i}"]
        assert obj(A, B, F) <= obj(A, B, ref) * (1 + FP32_TOL) + 1e-6


def test_identity_feasible_optimum():
    B = nm.uniform_matrix(6, 5, 7)
    F0 = nm.uniform_matrix(6, 5, 8)
    F = nm.solve_nnls(np.eye(6), B, F0, nm.InnerSolverConfig(max_iter=500, grad_tol=1e-12))
    assert np.abs(F - B).max() <= 1e-8


def test_negative_target_projects_to_zero():
    F = nm.solve_nnls(np.eye(1), np.array([[-1.0]]), np.array([[1.0]]))
    assert F == pytest.approx(np.zeros((1, 1)))


@pytest.mark.parametrize("seed", range(6))
def test_scipy_oracle_objective(seed):
    rng = np.random.default_rng(100 + seed)
    A = rng.standard_normal((30, 10))
    B = rng.standard_normal((30, 8))
    F0 = rng.random((10, 8))
    cfg = nm.InnerSolverConfig(max_iter=20000, grad_tol=1e-12)
    mine = obj(A, B, nm.solve_nnls(A, B, F0, cfg))
    Fo = np.column_stack([scipy_nnls(A, B[:, j])[0] for j in range(B.shape[1])])
    best = obj(A, B, Fo)
    assert mine <= best * (1 + 1e-6)
    assert mine >= best * (1 - 1e-9)


@pytest.mark.parametrize("seed", range(4))
def test_never_worse_than_start(seed):
    rng = np.random.default_rng(200 + seed)
    A = rng.standard_normal((12, 5))
    B = rng.standard_normal((12, 7))
    F0 = rng.random((5, 7))
    for max_iter in (1, 2, 5, 50):
        F = nm.solve_nnls(A, B, F0, nm.InnerSolverConfig(max_iter=max_iter))
        assert obj(A, B, F) <= obj(A, B, F0)
        assert F.min() >= 0.0


def test_max_iter_one_single_step():
    F = nm.solve_nnls(np.eye(2), np.array([[2.0, 0.0], [0.0, 2.0]]), np.zeros((2, 2)),
                      nm.InnerSolverConfig(max_iter=1, grad_tol=1e-30))
    assert np.allclose(F, [[2.0, 0.0], [0.0, 2.0]])


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_non_finite_failure():
    with pytest.raises((nm.NumericalFailureError, nm.ZeroMatrixError)):
        nm.solve_nnls(np.full((2, 2), 1e300), np.ones((2, 2)), np.ones((2, 2)))


def test_wide_column_count_multi_cta():
    """c large enough for many CTAs of the persistent solver (grid-wide
    speculative decisions), checked against the oracle."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((40, 20))
    B = np.abs(rng.standard_normal((40, 20000)))
    F0 = rng.random((20, 20000))
    cfg = nm.InnerSolverConfig(max_iter=300, grad_tol=1e-6)
    rep = []
    F = nm.solve_nnls(A, B, F0, cfg, report=rep)
    info = orc.SolveInfo()
    ref = orc.nesterov_nnls(A, B, F0, 300, 1e-6, 1.0, info)
    assert rel(F, ref) <= FP64_TOL
    assert abs(rep[0].inner_iters - info.iterations) <= 1


def test_gradient_and_pg_norm():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((7, 4))
    B = rng.standard_normal((7, 3))
    F = rng.standard_normal((4, 3))
    g = nm.gradient(A, B, F)
    assert np.allclose(g, A.T @ (A @ F - B), rtol=1e-10, atol=1e-12)
    assert nm.projected_gradient_norm(np.array([[0.0, 1.0]]), np.array([[-2.0, 3.0]])) == pytest.approx(np.sqrt(13))
    Fz = np.zeros((3, 3))
    assert nm.projected_gradient_norm(Fz, np.abs(nm.gaussian_matrix(3, 3, 6))) == 0.0


def test_spectral_norm_sq_golden(golden):
    d = golden("spectral")
    for i in range(int(d["count"])):
        G = d[f"G{i}"]
        assert nm.spectral_norm_sq(G) == pytest.approx(d["est"][i], rel=1e-9)
        assert nm.spectral_norm_sq(G, max_iters=5000) == pytest.approx(d["est_long"][i], rel=1e-9)
    assert nm.spectral_norm_sq(np.diag([3.0, 1.0])) == pytest.approx(9.0, abs=1e-8)


@pytest.mark.parametrize("seed", range(3))
def test_spectral_vs_svd(seed):
    G = nm.gaussian_matrix(50, 15, seed + 30)
    expected = np.linalg.svd(G, compute_uv=False)[0] ** 2
    assert nm.spectral_norm_sq(G, max_iters=5000) == pytest.approx(expected, rel=1e-6)
    est = nm.spectral_norm_sq(G)
    assert expected * (1 - 1e-6) <= est <= expected * 1.0101


def test_frobenius_and_rre():
    X = nm.uniform_matrix(15, 15, 4)
    assert nm.frobenius_norm(X) == pytest.approx(np.linalg.norm(X), rel=1e-14)
    G = nm.uniform_matrix(15, 4, 5)
    F = nm.uniform_matrix(4, 15, 6)
    base = nm.rre(X, G, F)
    assert base == pytest.approx(np.linalg.norm(X - G @ F) / np.linalg.norm(X), rel=1e-12)
    for c in (0.5, 3.0, 1e4):
        assert nm.rre(X, c * G, F / c) == pytest.approx(base, rel=1e-12)
    assert nm.rre(G @ F, G, F) <= 1e-15
    assert nm.rre(X, np.zeros((15, 2)), np.zeros((2, 15))) == 1.0
    with pytest.raises(nm.ZeroMatrixError):
        nm.rre(np.zeros((4, 4)), np.ones((4, 2)), np.ones((2, 4)))


@pytest.mark.parametrize("p,c,max_iter", [(20, 20000, 100), (9, 40000, 70), (30, 17000, 45), (50, 3000, 60),
                                          (61, 2500, 40)])
def test_streamed_solver_many_columns(monkeypatch, p, c, max_iter):
    """FP32 solves with more columns than the register-resident tensor-core
    solver holds, or 32 < p <= 64 (BASELINE cfg3's p = 50), use the streamed
    tensor-core solver (nnls_stream.cuh):
    within the FP32 tolerance of the fp64 oracle, and of the SIMT solver;
    same inner-iteration count and returned iterate kind."""
    rng = np.random.default_rng(c + p)
    r = max(30, p + 10)
    A = rng.random((r, p))
    B = A @ rng.random((p, c)) + 0.05 * rng.standard_normal((r, c))
    F0 = rng.random((p, c))
    cfg = nm.InnerSolverConfig(max_iter=max_iter, grad_tol=1e-9)
    rep_s, rep_simt = [], []
    Fs = nm.solve_nnls(A, B, F0, cfg, dtype="fp32", report=rep_s)
    monkeypatch.setenv("NENMF_NNLS_SIMT", "1")
    Fsimt = nm.solve_nnls(A, B, F0, cfg, dtype="fp32", report=rep_simt)
    Fr = orc.nesterov_nnls(A, B, F0, max_iter=max_iter, grad_tol=1e-9)
    assert rep_s[0].inner_iters == rep_simt[0].inner_iters
    assert np.linalg.norm(Fs - Fr) <= 1e-3 * np.linalg.norm(Fr)
    assert np.linalg.norm(Fs - Fsimt) <= 1e-3 * np.linalg.norm(Fsimt)


@pytest.mark.parametrize("p,c,max_iter", [(16, 30000, 80), (20, 20000, 64), (30, 17000, 45), (50, 3000, 40)])
def test_streamed_resident_matches_ring(monkeypatch, p, c, max_iter):
    """The streamed solver keeps a CTA's state in shared memory when its
    columns fit (BASELINE cfg5) and streams it through the cp.async ring from
    HBM otherwise: same arithmetic, bit-identical results."""
    rng = np.random.default_rng(p * 7 + c)
    r = max(30, p + 10)
    A = rng.random((r, p))
    B = A @ rng.random((p, c)) + 0.05 * rng.standard_normal((r, c))
    F0 = rng.random((p, c))
    cfg = nm.InnerSolverConfig(max_iter=max_iter, grad_tol=1e-9)
    rep_a, rep_b = [], []
    Fa = nm.solve_nnls(A, B, F0, cfg, dtype="fp32", report=rep_a)
    monkeypatch.setenv("NENMF_STREAM_RING", "1")
    Fb = nm.solve_nnls(A, B, F0, cfg, dtype="fp32", report=rep_b)
    assert rep_a[0].inner_iters == rep_b[0].inner_iters
    assert np.array_equal(Fa, Fb)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("shape", [(120, 100, 300), (40, 100, 257), (150, 112, 64), (90, 70, 1000)])
def test_solve_inner_dimension_above_64(shape, dtype):
    """The reference takes any p (nnls.py:119-159): p above 64 (FP64 up to 112,
    FP32 up to 128: W and the sum ring share the CTA's shared memory) runs the
    CUDA-core solver with 16 threads per column, chunked W / V products, the
    power iteration on the smaller Gram and the generic residual."""
    r, p, c = shape
    rng = np.random.default_rng(500 + r + p)
    A = rng.random((r, p))
    B = A @ rng.random((p, c)) + 0.05 * rng.random((r, c))
    F0 = rng.random((p, c))
    if dtype == "fp32":
        A, B, F0 = (M.astype(np.float32).astype(np.float64) for M in (A, B, F0))
    cfg = nm.InnerSolverConfig(max_iter=60, grad_tol=1e-6)
    rep = []
    F = nm.solve_nnls(A, B, F0, cfg, dtype=dtype, report=rep)
    info = orc.SolveInfo()
    ref = orc.nesterov_nnls(A, B, F0, 60, 1e-6, 1.0, info)
    tol = FP64_TOL if dtype == "fp64" else FP32_TOL
    assert F.shape == ref.shape and F.min() >= 0.0
    assert rel(F, ref) <= tol, rel(F, ref)
    assert abs(rep[0].lipschitz - info.lipschitz) <= (1e-9 if dtype == "fp64" else 1e-4) * info.lipschitz
    assert abs(rep[0].inner_iters - info.iterations) <= 1
    assert abs(nm.spectral_norm_sq(A, dtype=dtype) - orc.sigma_max_sq(A)) <= (1e-9 if dtype == "fp64" else 1e-4) * orc.sigma_max_sq(A)


def test_solve_fp32_p128_and_limits():
    rng = np.random.default_rng(9)
    A = rng.random((150, 128))
    B = A @ rng.random((128, 64))
    F0 = rng.random((128, 64))
    A, B, F0 = (M.astype(np.float32).astype(np.float64) for M in (A, B, F0))
    F = nm.solve_nnls(A, B, F0, nm.InnerSolverConfig(max_iter=40), dtype="fp32")
    ref = orc.nesterov_nnls(A, B, F0, 40, 1e-4, 1.0)
    assert rel(F, ref) <= FP32_TOL
    with pytest.raises(nm.BackendError):  # beyond the compiled range: a loud error, no fallback
        nm.solve_nnls(rng.random((300, 200)), rng.random((300, 8)), rng.random((200, 8)), dtype="fp64")


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_compressed_factorization_rank_above_64(dtype):
    """factorize_compressed with p = 80 and a 100-column sketch against the
    oracle fed the same sketch (two outer iterations)."""
    rng = np.random.default_rng(77)
    n, m, p, nu = 500, 420, 80, 100
    X = rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))
    if dtype == "fp32":
        X = X.astype(np.float32).astype(np.float64)
    sk = nm.subspace_iteration_pair(X, nu, 2, 78, dtype=dtype)
    init = nm.init_factors(n, m, p, seed=79)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=40), time_budget_seconds=0.0, max_outer_iterations=2)
    rec = nm.TraceRecorder()
    out = nm.factorize_compressed(X, sk, init, cfg, observer=rec, clock=nm.IterationClock(), dtype=dtype)
    ref = orc.nenmf(X, init.G, init.F, L=sk.L, R=sk.R, max_outer=2, max_iter=40)
    got = np.array([r.rre for r in rec.records])
    exp = np.array([r for _, r, _ in ref.records])
    tol = FP64_TOL if dtype == "fp64" else 2e-3
    assert np.abs(got - exp).max() <= tol * exp.max(), (got, exp)
    assert rel(out.F, ref.F) <= tol and rel(out.G, ref.G) <= tol


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_vanilla_factorization_rank_above_64(dtype):
    """factorize_vanilla with p = 72 (chunked V = A^T X products, generic
    explicit-residual tie-break) against the oracle, two outer iterations."""
    rng = np.random.default_rng(81)
    n, m, p = 300, 260, 72
    X = rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))
    if dtype == "fp32":
        X = X.astype(np.float32).astype(np.float64)
    init = nm.init_factors(n, m, p, seed=82)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=40), time_budget_seconds=0.0, max_outer_iterations=2)
    rec = nm.TraceRecorder()
    out = nm.factorize_vanilla(X, init, cfg, observer=rec, clock=nm.IterationClock(), dtype=dtype)
    ref = orc.nenmf(X, init.G, init.F, max_outer=2, max_iter=40)
    got = np.array([r.rre for r in rec.records])
    exp = np.array([r for _, r, _ in ref.records])
    tol = FP64_TOL if dtype == "fp64" else 2e-3
    assert np.abs(got - exp).max() <= tol * exp.max(), (got, exp)
    assert rel(out.F, ref.F) <= tol and rel(out.G, ref.G) <= tol
