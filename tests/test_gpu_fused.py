"""The fused solver launch (W = AᵀA, V = AᵀB, λmax and the explicit-residual
tie-break computed inside the persistent kernel, used when r <= 64) against
the unfused sequence of separate kernels (NENMF_NNLS_UNFUSED=1) and against
the CPU oracle.  W, V and L use the same arithmetic in both paths, so the
iterates agree to rounding of the residual sums (which only feed the
tie-break)."""

import numpy as np
import pytest

import nenmf_oracle as orc
import paper_1812_04315_b200 as nm

pytestmark = pytest.mark.gpu


def _case(r, p, c, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    A = rng.random((r, p)) * scale
    B = A @ rng.random((p, c)) + 0.05 * rng.standard_normal((r, c))
    F0 = rng.random((p, c))
    return A, B, F0


SHAPES = [(5, 3, 1), (30, 20, 37), (30, 20, 1000), (64, 32, 300), (12, 20, 100), (40, 9, 2500)]


@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
@pytest.mark.parametrize("shape", SHAPES)
def test_fused_matches_unfused(monkeypatch, dtype, tol, shape):
    r, p, c = shape
    A, B, F0 = _case(r, p, c, seed=r * 1000 + p * 10 + c)
    cfg = nm.InnerSolverConfig(max_iter=200, grad_tol=1e-6)
    rep_f, rep_u = [], []
    Ff = nm.solve_nnls(A, B, F0, cfg, dtype=dtype, report=rep_f)
    monkeypatch.setenv("NENMF_NNLS_UNFUSED", "1")
    # the fused prologue forms V on the CUDA cores in k_ab order: compare with
    # the same V kernel (the FP32 tensor-core V rounds differently)
    monkeypatch.setenv("NENMF_AB_SIMT", "1")
    Fu = nm.solve_nnls(A, B, F0, cfg, dtype=dtype, report=rep_u)
    assert rep_f[0].lipschitz == rep_u[0].lipschitz          # same power iteration
    assert rep_f[0].inner_iters == rep_u[0].inner_iters
    assert rep_f[0].returned_best == rep_u[0].returned_best
    assert np.abs(Ff - Fu).max() <= tol * max(np.abs(Fu).max(), 1.0)


@pytest.mark.parametrize("shape", SHAPES)
def test_fused_vs_oracle_fp64(shape):
    r, p, c = shape
    A, B, F0 = _case(r, p, c, seed=7 + r + p + c)
    cfg = nm.InnerSolverConfig(max_iter=150, grad_tol=1e-5)
    rep = []
    F = nm.solve_nnls(A, B, F0, cfg, report=rep)
    info = orc.SolveInfo()
    ref = orc.nesterov_nnls(A, B, F0, 150, 1e-5, 1.0, info)
    assert abs(rep[0].inner_iters - info.iterations) <= 1
    assert np.abs(F - ref).max() <= 1e-5 * np.abs(ref).max()


def test_fused_start_wins_and_no_improvement():
    """F0 already optimal: no iterate improves, the start point is returned
    unchanged (nnls.py:219-227 with best never set)."""
    rng = np.random.default_rng(3)
    A = rng.random((20, 6))
    F0 = rng.random((6, 50))
    B = A @ F0
    rep = []
    F = nm.solve_nnls(A, B, F0, nm.InnerSolverConfig(max_iter=30), report=rep)
    assert np.abs(F - F0).max() <= 1e-12
    assert rep[0].inner_iters >= 1


def test_fused_trans_view_matches(monkeypatch):
    """vanilla NeNMF with n, m <= 64: its G-half passes B = Xᵀ as a transposed
    view (r = m), so the fused kernel reads B through the trans path."""
    rng = np.random.default_rng(11)
    n, m, p = 48, 60, 7
    X = rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))
    init = nm.init_factors(n, m, p, seed=5)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=60), time_budget_seconds=0.0,
                         max_outer_iterations=4)
    a = nm.factorize_vanilla(X, init, cfg, clock=nm.IterationClock())
    monkeypatch.setenv("NENMF_NNLS_UNFUSED", "1")
    b = nm.factorize_vanilla(X, init, cfg, clock=nm.IterationClock())
    assert np.abs(a.G - b.G).max() <= 1e-12 * np.abs(b.G).max()
    assert np.abs(a.F - b.F).max() <= 1e-12 * np.abs(b.F).max()


def test_fused_zero_matrix_raises():
    A = np.zeros((10, 4))
    B = np.ones((10, 30))
    with pytest.raises(nm.ZeroMatrixError):
        nm.solve_nnls(A, B, np.ones((4, 30)))


@pytest.mark.parametrize("unfused", [False, True])
@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
@pytest.mark.parametrize("shape", [(30, 20, 10000, 30), (12, 5, 333, 7), (40, 32, 2000, 64)])
def test_next_product(monkeypatch, unfused, dtype, tol, shape):
    """nenmf_solve_nnls_next: next_out = F_out next_btᵀ formed by the solver
    launch (fused) or by a separate product (fallback) -- factorize.py:110,113."""
    import torch
    from paper_1812_04315_b200 import _lib, _ops
    if unfused:
        monkeypatch.setenv("NENMF_NNLS_UNFUSED", "1")
    r, p, c, k = shape
    A, B, F0 = _case(r, p, c, seed=c + k)
    P = np.random.default_rng(k).standard_normal((k, c))
    tdt = torch.float64 if dtype == "fp64" else torch.float32
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=tdt, device="cuda")
    At, Bd, F0d, Pd = dev(A.T), dev(B), dev(F0), dev(P)
    Fo = torch.empty_like(F0d)
    out = torch.empty((p, k), dtype=tdt, device="cuda")
    st = _lib.new_status()
    _ops.solve(At, Bd, F0d, Fo, trans_b=False, max_iter=60, grad_tol=1e-6, lipschitz_safety=1.0, status=st,
               next_bt=Pd, next_out=out)
    F = Fo.double().cpu().numpy()
    ref = F @ P.astype(np.float64 if dtype == "fp64" else np.float32).astype(np.float64).T
    got = out.double().cpu().numpy()
    assert np.abs(got - ref).max() <= tol * np.abs(ref).max()
    # the solve itself is unchanged by the extra product
    Fo2 = torch.empty_like(F0d)
    _ops.solve(At, Bd, F0d, Fo2, trans_b=False, max_iter=60, grad_tol=1e-6, lipschitz_safety=1.0,
               status=_lib.new_status())
    assert torch.equal(Fo, Fo2)


@pytest.mark.parametrize("case", ["start_wins", "early_stop", "full"])
def test_next_product_decision_paths(case):
    """The fused launch forms the next product from the final iterate before
    the stopping decision is known; check the product against F_out when that
    guess holds (full run), when the solve stops early (best != final
    iterate) and when the start point wins (second grid barrier)."""
    import torch
    from paper_1812_04315_b200 import _lib, _ops
    rng = np.random.default_rng({"start_wins": 1, "early_stop": 2, "full": 3}[case])
    r, p, c, k = 30, 20, 5000, 30
    A = rng.random((r, p))
    if case == "start_wins":
        F0 = rng.random((p, c))
        B = A @ F0
    else:
        B = A @ rng.random((p, c)) + 0.05 * rng.standard_normal((r, c))
        F0 = rng.random((p, c))
    P = rng.standard_normal((k, c))
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    At, Bd, F0d, Pd = dev(A.T), dev(B), dev(F0), dev(P)
    Fo = torch.empty_like(F0d)
    out = torch.empty((p, k), dtype=torch.float64, device="cuda")
    st = _lib.new_status()
    tol = {"start_wins": 1e-6, "early_stop": 1e-2, "full": 1e-12}[case]
    _ops.solve(At, Bd, F0d, Fo, trans_b=False, max_iter=80, grad_tol=tol, lipschitz_safety=1.0, status=st,
               next_bt=Pd, next_out=out)
    rep = _lib.read_status(st)[0]
    F = Fo.cpu().numpy()
    if case == "start_wins":
        assert np.abs(F - F0).max() <= 1e-12
    if case == "early_stop":
        assert int(rep["inner_iters"]) < 80
    ref = F @ P.T
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


def test_fp64_mma_solver_cfg2_shape():
    """FP64 at the cfg2 compressed shape (p = 20, r = 30, 10 000 columns: 68
    per CTA, 9 DMMA compute warps) against the fp64 oracle."""
    A, B, F0 = _case(30, 20, 10000, seed=2024)
    cfg = nm.InnerSolverConfig(max_iter=120, grad_tol=1e-7)
    rep = []
    F = nm.solve_nnls(A, B, F0, cfg, report=rep)
    info = orc.SolveInfo()
    ref = orc.nesterov_nnls(A, B, F0, 120, 1e-7, 1.0, info)
    assert abs(rep[0].inner_iters - info.iterations) <= 1
    assert np.abs(F - ref).max() <= 1e-9 * np.abs(ref).max()
