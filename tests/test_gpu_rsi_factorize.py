"""GPU parity of randomized subspace iteration, compression and the outer
NeNMF loops against the reference's golden fixtures and the CPU oracle.

Sketch parity is a SUBSPACE comparison (QR is unique only up to column
signs; rank-deficient inputs leave the trailing directions as rounding noise,
SURVEY §8c).  Solver/trajectory parity feeds the SAME sketch to both sides."""

import math

import numpy as np
import pytest

import nenmf_oracle as orc
import paper_1812_04315_b200 as nm

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-5
FP32_TOL = 1e-3


def capped(outer, inner=500, **kw):
    return nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=inner), time_budget_seconds=0.0,
                          max_outer_iterations=outer, **kw)


def sin_max_angle(Q1, Q2, top=None):
    """largest principal-angle sine between the column spans of Q1, Q2 (orthonormal)."""
    s = np.linalg.svd(Q1.T @ Q2, compute_uv=False)
    if top is not None:
        s = s[:top]
    return math.sqrt(max(0.0, 1.0 - min(1.0, s.min()) ** 2))


def capture(X, sk):
    nx = np.linalg.norm(X)
    left = np.linalg.norm(X - sk.L.T @ (sk.L @ X)) / nx
    right = np.linalg.norm(X - (X @ sk.R) @ sk.R.T) / nx
    return left, right


def test_sketch_vs_golden(golden):
    d = golden("rsi")
    for name in d["names"]:
        nu, q, seed = (int(v) for v in d[f"{name}_par"])
        X = d[f"{name}_X"]
        sk = nm.subspace_iteration_pair(X, nu, q, seed)
        eye = np.eye(nu)
        assert np.abs(sk.L @ sk.L.T - eye).max() <= 1e-10, name
        assert np.abs(sk.R.T @ sk.R - eye).max() <= 1e-10, name
        Lr, Rr = d[f"{name}_L"], d[f"{name}_R"]
        if name == "lowrank":
            # rank 15 < nu = 25: only the top-15 directions are determined
            assert sin_max_angle(sk.L.T, Lr.T, top=15) <= 1e-6, name
            left, right = capture(X, sk)
            assert left <= 1e-8 and right <= 1e-8
        else:
            assert sin_max_angle(sk.L.T, Lr.T) <= 1e-6, name
            assert sin_max_angle(sk.R, Rr) <= 1e-6, name
            lg, rg = capture(X, nm.SketchPair(Lr, Rr, nu, nm.SUBSPACE_ITERATION, q, seed))
            lm, rm = capture(X, sk)
            assert lm <= lg * (1 + 1e-6) + 1e-12 and rm <= rg * (1 + 1e-6) + 1e-12


def test_sketch_deterministic_and_monotone():
    rng = np.random.default_rng(24)
    X = rng.random((50, 5)) @ rng.random((5, 40))
    a = nm.subspace_iteration_pair(X, 8, 2, seed=25)
    b = nm.subspace_iteration_pair(X, 8, 2, seed=25)
    assert (a.L == b.L).all() and (a.R == b.R).all()
    d = np.random.default_rng(22)
    X2 = d.random((150, 10)) @ d.random((10, 150)) + 0.01 * d.standard_normal((150, 150))
    prev = (math.inf, math.inf)
    for q in (1, 2, 3, 4):
        cur = capture(X2, nm.subspace_iteration_pair(X2, 20, q, seed=23))
        assert cur[0] <= prev[0] + 1e-12 and cur[1] <= prev[1] + 1e-12
        prev = cur


def test_compress_vs_golden(golden):
    d = golden("rsi")
    for name in d["names"]:
        nu, q, seed = (int(v) for v in d[f"{name}_par"])
        sk = nm.SketchPair(d[f"{name}_L"], d[f"{name}_R"], nu, nm.SUBSPACE_ITERATION, q, seed)
        comp = nm.compress_problem(d[f"{name}_X"], sk)
        assert np.abs(comp.X_L - d[f"{name}_XL"]).max() <= 1e-12 * np.abs(d[f"{name}_XL"]).max()
        assert np.abs(comp.X_R - d[f"{name}_XR"]).max() <= 1e-12 * np.abs(d[f"{name}_XR"]).max()


def test_compress_identity_exact():
    rng = np.random.default_rng(40)
    X = rng.random((20, 3)) @ rng.random((3, 20))
    sk = nm.SketchPair(L=np.eye(20), R=np.eye(20), nu=20, scheme=nm.GAUSSIAN, q=0, seed=0)
    comp = nm.compress_problem(X, sk)
    assert (comp.X_L == X).all() and (comp.X_R == X).all()


def _trace(recs):
    return np.array([[r.outer_iter, r.rre, r.objective] for r in recs])


@pytest.mark.parametrize("method", ["vanilla", "compressed"])
def test_factorize_small_vs_golden(golden, method):
    d = golden("factorize")
    X = d["small_X"]
    init = nm.FactorPair(G=d["small_G0"], F=d["small_F0"], p=8)
    rec = nm.TraceRecorder()
    if method == "vanilla":
        out = nm.factorize_vanilla(X, init, capped(12), observer=rec, clock=nm.IterationClock())
    else:
        sk = nm.SketchPair(d["small_L"], d["small_R"], 16, nm.SUBSPACE_ITERATION, 4, 22)
        out = nm.factorize_compressed(X, sk, init, capped(12), observer=rec, clock=nm.IterationClock())
    ref = d[f"small_{method}_trace"]
    got = _trace(rec.records)
    assert got.shape == ref.shape
    assert (got[:, 0] == ref[:, 0]).all()
    assert np.abs(got[:, 1] - ref[:, 1]).max() <= FP64_TOL * ref[:, 1].max()
    assert np.abs(out.G - d[f"small_{method}_G"]).max() <= FP64_TOL * np.abs(d[f"small_{method}_G"]).max()
    assert np.abs(out.F - d[f"small_{method}_F"]).max() <= FP64_TOL * np.abs(d[f"small_{method}_F"]).max()


def test_trace_cadence(golden):
    d = golden("factorize")
    init = nm.FactorPair(G=d["cadence_G0"], F=d["cadence_F0"], p=3)
    cfg = nm.OuterConfig(time_budget_seconds=0.0, max_outer_iterations=7, trace_every=3)
    rec = nm.TraceRecorder()
    nm.factorize_vanilla(d["cadence_X"], init, cfg, observer=rec, clock=nm.IterationClock())
    got = _trace(rec.records)
    assert list(got[:, 0]) == [0, 3, 6, 7]
    assert np.abs(got[:, 1] - d["cadence_trace"][:, 1]).max() <= FP64_TOL * got[:, 1].max()


def test_identity_sketch_reproduces_vanilla_exactly():
    """reference test_factorize.py:161-176 / acceptance criterion 6"""
    n = m = 90
    rng = np.random.default_rng(18)
    X = rng.random((n, 7)) @ rng.random((7, m)) + 0.01 * rng.standard_normal((n, m))
    init = nm.init_factors(n, m, 7, seed=19)
    cfg = capped(6)
    rv, rc = nm.TraceRecorder(), nm.TraceRecorder()
    pv = nm.factorize_vanilla(X, init, cfg, observer=rv, clock=nm.IterationClock())
    ident = nm.SketchPair(L=np.eye(n), R=np.eye(m), nu=n, scheme=nm.SUBSPACE_ITERATION, q=0, seed=0)
    pc = nm.factorize_compressed(X, ident, init, cfg, observer=rc, clock=nm.IterationClock())
    assert rv.records == rc.records
    assert (pv.G == pc.G).all() and (pv.F == pc.F).all()


def test_observer_contract_and_monotone_objective():
    rng = np.random.default_rng(6)
    X = rng.random((80, 6)) @ rng.random((6, 70)) + 0.02 * rng.standard_normal((80, 70))
    init = nm.init_factors(80, 70, 6, seed=7)
    rec = nm.TraceRecorder()
    seen = []
    nm.factorize_vanilla(X, init, capped(25), observer=lambda r, G, F: (rec(r, G, F), seen.append((G.min(), F.min(), G.shape, F.shape))))
    objs = [r.objective for r in rec.records]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(objs, objs[1:]))
    assert [r.outer_iter for r in rec.records] == list(range(26))
    assert all(gm >= 0 and fm >= 0 and gs == (80, 6) and fs == (6, 70) for gm, fm, gs, fs in seen)
    el = [r.solver_elapsed_s for r in rec.records]
    assert all(b > a for a, b in zip(el, el[1:]))
    assert all(r.solver_elapsed_s <= r.wall_elapsed_s for r in rec.records)


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_numerical_failure_carries_outer_index():
    X = np.full((8, 8), 1e160)
    init = nm.init_factors(8, 8, 2, 17)
    with pytest.raises(nm.NumericalFailureError) as err:
        nm.factorize_vanilla(X, init, capped(3))
    assert err.value.outer_iteration == 1


def test_zero_data_rejected():
    with pytest.raises(nm.ZeroMatrixError):
        nm.factorize_vanilla(np.zeros((10, 10)), nm.init_factors(10, 10, 2, 1), capped(2))


def test_fixed_point_returns_immediately():
    rng = np.random.default_rng(3)
    G, F = rng.random((40, 4)) + 0.1, rng.random((4, 40)) + 0.1
    X = G @ F
    rec = nm.TraceRecorder()
    out = nm.factorize_vanilla(X, nm.FactorPair(G=G, F=F, p=4),
                               nm.OuterConfig(time_budget_seconds=5.0, rre_target=1e-9), observer=rec)
    assert len(rec.records) == 1 and rec.records[0].rre <= 1e-12
    assert (out.G == G).all()


def test_rre_target_on_cadence():
    rng = np.random.default_rng(14)
    X = rng.random((60, 5)) @ rng.random((5, 60))
    rec = nm.TraceRecorder()
    nm.factorize_vanilla(X, nm.init_factors(60, 60, 5, seed=15),
                         nm.OuterConfig(time_budget_seconds=30.0, rre_target=5e-2, trace_every=2), observer=rec)
    assert rec.records[-1].rre <= 5e-2 and rec.records[-1].outer_iter % 2 == 0


def test_full_rre_reported_not_surrogate():
    rng = np.random.default_rng(23)
    X = rng.random((100, 6)) @ rng.random((6, 100)) + 0.02 * rng.standard_normal((100, 100))
    init = nm.init_factors(100, 100, 6, seed=24)
    sk = nm.subspace_iteration_pair(X, 12, 2, seed=25)
    rec = nm.TraceRecorder()
    pair = nm.factorize_compressed(X, sk, init, capped(5), observer=rec)
    expected = np.linalg.norm(X - pair.G @ pair.F) / np.linalg.norm(X)
    assert rec.records[-1].rre == pytest.approx(expected, rel=1e-12)


def test_config1_parity(golden):
    """BASELINE config 1 end to end in FP64: same sketch -> trajectory and
    factors within 1e-5; GPU-built sketch -> same top-p subspace."""
    from paper_1812_04315_b200 import workloads

    d = golden("config1")
    w = workloads.make_workload(1)
    init = nm.FactorPair(G=w.G0, F=w.F0, p=w.p)
    sk = nm.SketchPair(d["L"], d["R"], w.nu, nm.SUBSPACE_ITERATION, w.q, w.sketch_seed)
    for method in ("compressed", "vanilla"):
        rec = nm.TraceRecorder()
        if method == "compressed":
            out = nm.factorize_compressed(w.X, sk, init, capped(w.outer, w.inner), observer=rec,
                                          clock=nm.IterationClock())
        else:
            out = nm.factorize_vanilla(w.X, init, capped(w.outer, w.inner), observer=rec, clock=nm.IterationClock())
        ref = d[f"{method}_trace"]
        got = _trace(rec.records)
        assert np.abs(got[:, 1] - ref[:, 1]).max() <= FP64_TOL * ref[:, 1].max(), method
        assert np.abs(out.F - d[f"{method}_F"]).max() <= FP64_TOL * np.abs(d[f"{method}_F"]).max(), method
        assert np.abs(out.G - d[f"{method}_G"]).max() <= FP64_TOL * np.abs(d[f"{method}_G"]).max(), method
    gsk = nm.subspace_iteration_pair(w.X, w.nu, w.q, w.sketch_seed)
    assert sin_max_angle(gsk.L.T, d["L"].T, top=w.p) <= 1e-6
    assert sin_max_angle(gsk.R, d["R"], top=w.p) <= 1e-6


def test_fp32_mode_trajectory():
    """FP32 arithmetic on a cfg2-like noisy problem: trajectory within 1e-3 of
    the FP64 oracle fed the same (fp32-rounded) inputs and the same sketch."""
    from paper_1812_04315_b200 import workloads

    w = workloads.make_workload(2, n=1500, m=1200, dtype="fp32")
    sk64 = nm.subspace_iteration_pair(w.X, w.nu, w.q, w.sketch_seed)
    init = nm.FactorPair(G=w.G0, F=w.F0, p=w.p)
    rec = nm.TraceRecorder()
    nm.factorize_compressed(w.X, sk64, init, capped(10, 50), observer=rec, clock=nm.IterationClock(),
                            dtype="fp32")
    ref = orc.nenmf(w.X, w.G0, w.F0, L=sk64.L, R=sk64.R, max_outer=10, max_iter=50)
    got = _trace(rec.records)[:, 1]
    exp = np.array([r for _, r, _ in ref.records])
    assert np.abs(got - exp).max() <= FP32_TOL * exp.max()
    sk32 = nm.subspace_iteration_pair(w.X, w.nu, w.q, w.sketch_seed, dtype="fp32")
    assert sin_max_angle(sk32.L.T, sk64.L.T, top=w.p) <= 1e-3
    assert np.abs(sk32.L @ sk32.L.T - np.eye(w.nu)).max() <= 1e-5


def test_vanilla_fp32_tensor_v_vs_oracle():
    """FP32 vanilla NeNMF, default (CUDA-core V) and tensor_v=True (V = A^T B
    from the BF16x3 tensor-core pass over the prepared X,
    nenmf_solve_nnls_prepared), against the fp64 oracle on the fp32-rounded
    inputs: RRE trajectory and factors within 1e-3 (relative Frobenius) in
    both forms (the tensor_v form was 1.05e-3 before the FP32 solver's
    round-to-nearest accumulation)."""
    import nenmf_oracle as orc

    rng = np.random.default_rng(9)
    n, m, p = 300, 257, 6
    X = (rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))).astype(np.float32).astype(np.float64)
    init = nm.init_factors(n, m, p, seed=4)
    G0 = init.G.astype(np.float32).astype(np.float64)
    F0 = init.F.astype(np.float32).astype(np.float64)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=60), time_budget_seconds=0.0, max_outer_iterations=8)
    ref = orc.nenmf(X, G0, F0, max_outer=8, max_iter=60)
    exp = np.array([r for _, r, _ in ref.records])
    for tensor_v, ftol in ((False, 1e-3), (True, 1e-3)):
        rec = nm.TraceRecorder()
        out = nm.factorize_vanilla(X, nm.FactorPair(G=G0, F=F0, p=p), cfg, observer=rec, clock=nm.IterationClock(),
                                   dtype="fp32", tensor_v=tensor_v)
        got = np.array([r.rre for r in rec.records])
        assert np.abs(got - exp).max() <= 1e-3 * exp.max()
        assert np.linalg.norm(out.F - ref.F) <= ftol * np.linalg.norm(ref.F)
        assert np.linalg.norm(out.G - ref.G) <= ftol * np.linalg.norm(ref.G)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_power_iteration_vs_golden(golden, dtype):
    """power_iteration_pair (compression.py:144-176) against the reference's
    own outputs: the raw power iterates are ill-conditioned, so the dominant
    directions are compared (fp64: top half of the sketch at sin 1e-6; fp32:
    the leading direction at 1e-3),
    plus orthonormality and the overflow step of a large-scale X (fp32
    reproduces the fp64 overflow step through its power-of-two scale factors)."""
    d = golden("power")
    for name in d["names"]:
        nu, q, seed = (int(v) for v in d[f"{name}_par"])
        X = d[f"{name}_X"]
        if dtype == "fp32":
            X = X.astype(np.float32).astype(np.float64)
        sk = nm.power_iteration_pair(X, nu, q, seed, dtype=dtype)
        assert sk.scheme == nm.POWER_ITERATION
        tol_o = 1e-10 if dtype == "fp64" else 1e-5
        assert np.abs(sk.L @ sk.L.T - np.eye(nu)).max() <= tol_o, name
        assert np.abs(sk.R.T @ sk.R - np.eye(nu)).max() <= tol_o, name
        # fp64: the top half of the sketch; fp32: the passes carry ~1e-5 relative
        # precision, so only directions whose power-iterate weight
        # (s_i / s_1)^(2q+1) stays well above that are determined -- on these
        # nonnegative problems (s_1 >> s_2) the leading direction
        top = max(1, nu // 2) if dtype == "fp64" else 1
        tol = 1e-6 if dtype == "fp64" else 1e-3
        assert sin_max_angle(sk.L.T, d[f"{name}_L"].T, top=top) <= tol, name
        assert sin_max_angle(sk.R, d[f"{name}_R"], top=top) <= tol, name
    nu, q, seed, step = (int(v) for v in d["overflow_par"])
    X = d["overflow_X"]
    if dtype == "fp32":
        # entries ~1e40 do not fit fp32: scale into range; the expected step
        # comes from the pinned oracle on the same fp32-rounded data
        import nenmf_oracle as orc

        X = (X * 1e-10).astype(np.float32).astype(np.float64)
        with pytest.raises(orc.OracleFailure) as ref_exc:
            orc.power_pair(X, nu, q, seed)
        step = ref_exc.value.iteration
    with pytest.raises(nm.NumericalCollapseError) as exc:
        nm.power_iteration_pair(X, nu, q, seed, dtype=dtype)
    assert exc.value.iteration == step


@pytest.mark.parametrize("dtype,nu,shape", [("fp64", 100, (700, 600)), ("fp64", 70, (700, 600)),
                                            ("fp32", 100, (700, 600)), ("fp32", 150, (700, 600)),
                                            # 32 < nu <= 64: FP64 passes in row blocks of 32 (TMA + DMMA), FP32 the
                                            # 64-wide tcgen05 instance; odd sizes take the unaligned fallbacks
                                            ("fp64", 48, (900, 800)), ("fp64", 48, (901, 803)),
                                            ("fp32", 48, (900, 800)), ("fp32", 60, (901, 803))])
def test_wide_sketch_beyond_64_columns(dtype, nu, shape):
    """The reference takes any nu <= min(n, m) (compression.py:109-117): sketches
    wider than the 64 columns of the one-launch factorizations run the blocked
    orthonormalisation and the chunked X-passes; subspace, compression and
    the factorization against the oracle fed the same sketch."""
    rng = np.random.default_rng(91)
    (n, m), p, q = shape, 12, 2
    X = rng.random((n, p)) @ rng.random((p, m)) + 0.02 * rng.random((n, m))
    if dtype == "fp32":
        X = X.astype(np.float32).astype(np.float64)
    sk = nm.subspace_iteration_pair(X, nu, q, 92, dtype=dtype)
    eye = np.eye(nu)
    otol = 1e-10 if dtype == "fp64" else 2e-5
    assert sk.L.shape == (nu, n) and sk.R.shape == (m, nu)
    assert np.abs(sk.L @ sk.L.T - eye).max() <= otol
    assert np.abs(sk.R.T @ sk.R - eye).max() <= otol
    Lr, Rr = orc.rsi(X, nu, q, 92)
    stol = 1e-6 if dtype == "fp64" else 1e-3
    # full-rank noisy X: the whole nu-dimensional subspace is determined, but its trailing
    # directions (noise singular values nearly equal) are ill-conditioned: compare what the
    # sketch is for -- the dominant p directions and the captured energy
    ul = np.linalg.svd(sk.L @ X, full_matrices=False)[0][:, :p]
    ur = np.linalg.svd(Lr @ X, full_matrices=False)[0][:, :p]
    assert sin_max_angle(sk.L.T @ ul, Lr.T @ ur) <= stol
    vl = np.linalg.svd(X @ sk.R, full_matrices=False)[2][:p].T
    vr = np.linalg.svd(X @ Rr, full_matrices=False)[2][:p].T
    assert sin_max_angle(sk.R @ vl, Rr @ vr) <= stol
    lg, rg = capture(X, nm.SketchPair(Lr, Rr, nu, nm.SUBSPACE_ITERATION, q, 92))
    lm, rm = capture(X, sk)
    assert abs(lm - lg) <= 1e-3 * lg and abs(rm - rg) <= 1e-3 * rg
    # compression and three outer iterations with this sketch
    init = nm.init_factors(n, m, p, seed=93)
    rec = nm.TraceRecorder()
    out = nm.factorize_compressed(X, sk, init, capped(3, inner=100), observer=rec, clock=nm.IterationClock(),
                                  dtype=dtype)
    ref = orc.nenmf(X, init.G, init.F, L=sk.L, R=sk.R, max_outer=3, max_iter=100)
    got = np.array([r.rre for r in rec.records])
    exp = np.array([r for _, r, _ in ref.records])
    tol = FP64_TOL if dtype == "fp64" else 2e-3
    assert np.abs(got - exp).max() <= tol * exp.max()
    assert np.abs(out.F - ref.F).max() <= tol * np.abs(ref.F).max()


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_wide_sketch_of_rank_deficient_matrix(dtype):
    """nu = 100 on a noiseless rank-20 X: 80 of the sketch directions are the
    random completion of rank-deficient blocks.  They must still be
    orthonormal to the earlier blocks (the second sweep of the blocked
    orthonormalisation), and the sketch must capture X (reference
    test_compression.py: rank-deficient inputs)."""
    rng = np.random.default_rng(310)
    n, m, rank, nu = 640, 520, 20, 100
    X = rng.random((n, rank)) @ rng.random((rank, m))
    if dtype == "fp32":
        X = X.astype(np.float32).astype(np.float64)
    sk = nm.subspace_iteration_pair(X, nu, 2, 311, dtype=dtype)
    eye = np.eye(nu)
    otol = 1e-10 if dtype == "fp64" else 2e-5
    assert np.abs(sk.L @ sk.L.T - eye).max() <= otol
    assert np.abs(sk.R.T @ sk.R - eye).max() <= otol
    left, right = capture(X, sk)
    ctol = 1e-8 if dtype == "fp64" else 1e-4
    assert left <= ctol and right <= ctol, (left, right)
    Lr, Rr = orc.rsi(X, nu, 2, 311)
    assert sin_max_angle(sk.L.T @ np.linalg.svd(sk.L @ X, full_matrices=False)[0][:, :rank],
                         Lr.T @ np.linalg.svd(Lr @ X, full_matrices=False)[0][:, :rank]) <= (1e-6 if dtype == "fp64" else 1e-3)
