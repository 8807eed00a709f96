"""CPU tests: the C-ABI library loads and exports every declared symbol, and
the drop-in API validates its inputs (same exceptions, same order as the
reference) before any device work.  No GPU needed."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import _lib
from paper_1812_04315_b200.errors import BackendError

REPO = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (REPO / "include" / "nenmf_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nenmf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)
    assert lib.nenmf_abi_version() == 1
    assert lib.nenmf_status_string(3).decode().startswith("numerical failure")


def test_workspace_queries_are_pure():
    lib = _lib.load_library()
    assert lib.nenmf_solve_nnls_workspace_bytes(0, 30, 20, 10000) > 20 * 10000 * 8
    assert lib.nenmf_rsi_workspace_bytes(1, 10000, 10000, 30) > 0
    assert lib.nenmf_orthonormalize_workspace_bytes(400000, 40) > 400000 * 40 * 8
    assert lib.nenmf_dual_pass_workspace_bytes(0, 100, 100, 8) >= 0


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_status_struct_layout():
    assert _lib.STATUS_FIELDS.itemsize == 64


# ------------------------------------------------------------- validation
def test_alpha_next():
    assert nm.alpha_next(1.0) == pytest.approx(1.6180339887, abs=1e-9)
    assert nm.alpha_next(nm.alpha_next(1.0)) == pytest.approx(2.1935270853, abs=1e-9)
    with pytest.raises(ValueError):
        nm.alpha_next(0.99)


def test_configs_validate():
    with pytest.raises(ValueError):
        nm.InnerSolverConfig(max_iter=0)
    with pytest.raises(ValueError):
        nm.InnerSolverConfig(grad_tol=0.0)
    with pytest.raises(ValueError):
        nm.InnerSolverConfig(lipschitz_safety=0.5)
    with pytest.raises(ValueError):
        nm.OuterConfig(time_budget_seconds=0.0, max_outer_iterations=0)
    with pytest.raises(ValueError):
        nm.OuterConfig(time_budget_seconds=-1.0)
    with pytest.raises(ValueError):
        nm.OuterConfig(trace_every=0)
    with pytest.raises(ValueError):
        nm.OuterConfig(rre_target=-1.0)


def test_factor_pair_and_init():
    with pytest.raises(ValueError):
        nm.FactorPair(G=-np.ones((3, 2)), F=np.ones((2, 3)), p=2)
    with pytest.raises(nm.DimensionError):
        nm.FactorPair(G=np.ones((3, 2)), F=np.ones((3, 3)), p=2)
    with pytest.raises(nm.DimensionError):
        nm.init_factors(10, 5, 6, 1)
    pair = nm.init_factors(50, 60, 7, 2)
    assert pair.G.min() > 0 and pair.F.max() < 1
    a, b = nm.init_factors(20, 30, 4, 9), nm.init_factors(20, 30, 4, 9)
    assert (a.G == b.G).all() and (a.F == b.F).all()


def test_solve_nnls_validation_order():
    with pytest.raises(nm.DimensionError):
        nm.solve_nnls(np.eye(3), np.ones((3, 2)), np.ones((2, 2)))
    with pytest.raises(nm.ZeroMatrixError):
        nm.solve_nnls(np.zeros((3, 2)), np.ones((3, 2)), -np.ones((2, 2)))  # zero A wins over negative F0
    with pytest.raises(ValueError):
        nm.solve_nnls(np.eye(2), np.ones((2, 2)), -np.ones((2, 2)))


def test_helpers_validate_shapes():
    with pytest.raises(nm.DimensionError):
        nm.gradient(np.ones((3, 2)), np.ones((3, 3)), np.ones((3, 3)))
    with pytest.raises(nm.DimensionError):
        nm.projected_gradient_norm(np.zeros((2, 2)), np.zeros((2, 3)))
    with pytest.raises(nm.DimensionError):
        nm.rre(np.ones((4, 4)), np.ones((4, 2)), np.ones((3, 4)))
    with pytest.raises(nm.ZeroMatrixError):
        nm.spectral_norm_sq(np.zeros((3, 3)))


def test_sketch_validation():
    with pytest.raises(nm.DimensionError):
        nm.subspace_iteration_pair(np.ones((10, 8)), 9, 1, seed=1)
    with pytest.raises(nm.ZeroMatrixError):
        nm.subspace_iteration_pair(np.zeros((10, 10)), 2, 1, seed=1)
    with pytest.raises(ValueError):
        nm.subspace_iteration_pair(np.ones((10, 10)), 2, 0, seed=1)
    with pytest.raises(nm.DimensionError):
        nm.gaussian_sketch_pair(10, 10, 0, 1)
    sk = nm.gaussian_sketch_pair(10, 10, 3, 1)
    with pytest.raises(nm.DimensionError):
        nm.compress_problem(np.ones((10, 12)), sk)
    g = nm.gaussian_sketch_pair(500, 500, 25, 2)
    assert g.L.shape == (25, 500) and g.R.shape == (500, 25) and g.q == 0
    assert g.L.var() == pytest.approx(1 / 25, rel=0.10)


def test_factorize_validation():
    X = np.ones((20, 20))
    with pytest.raises(nm.DimensionError):
        nm.factorize_vanilla(X, nm.init_factors(20, 19, 3, 1),
                             nm.OuterConfig(time_budget_seconds=0.0, max_outer_iterations=2))
    bad = nm.SketchPair(L=np.eye(10), R=np.eye(10), nu=10, scheme=nm.SUBSPACE_ITERATION, q=0, seed=0)
    with pytest.raises(nm.DimensionError):
        nm.factorize_compressed(X, bad, nm.init_factors(20, 20, 3, 1),
                                nm.OuterConfig(time_budget_seconds=0.0, max_outer_iterations=2))


def test_no_cpu_fallback_without_device():
    from conftest import cuda_available

    if cuda_available():
        pytest.skip("device present")
    with pytest.raises(BackendError):
        nm.solve_nnls(np.eye(2), np.ones((2, 2)), np.ones((2, 2)))
    with pytest.raises(BackendError):
        nm.subspace_iteration_pair(np.ones((10, 10)), 2, 1, seed=1)
    with pytest.raises(BackendError):
        nm.frobenius_norm(np.ones((3, 3)))


def test_tracing_host_objects():
    rec = nm.TraceRecorder()
    r0 = nm.TraceRecord(0, 0.0, 0.0, 0.5, 1.0)
    rec(r0, None, None)
    with pytest.raises(ValueError):
        rec(r0, None, None)
    clock = nm.IterationClock(step=2.0, offset=1.0)
    clock.tick()
    assert clock.elapsed() == 3.0 and clock.wall_elapsed() == 3.0
    trace = nm.ConvergenceTrace(records=[nm.TraceRecord(1, 0.1, 0.2, 0.5, 1.0),
                                         nm.TraceRecord(2, 0.2, 0.3, 0.04, 1.0)])
    assert nm.time_to_target(trace, 0.05) == 0.2
    assert nm.iterations_to_target(trace, 0.01) is None
    mc = nm.MonotonicClock(offset=2.5)
    assert mc.elapsed() >= 2.5 and mc.wall_elapsed() >= 2.5
