"""Pin the CPU oracle to the reference: every fixture in tests/golden/ was
produced by running the reference package itself (tests/golden/make_golden.py).
CPU only."""

import numpy as np
import pytest

import nenmf_oracle as orc


def test_alpha_series(golden):
    g = golden("alpha")["alpha"]
    a = [1.0]
    for _ in range(len(g) - 1):
        a.append(orc.next_alpha(a[-1]))
    assert np.array_equal(np.array(a), g)
    assert g[1] == pytest.approx(1.6180339887, abs=1e-9)
    assert g[2] == pytest.approx(2.1935270853, abs=1e-9)


def test_spectral_norm_sq(golden):
    d = golden("spectral")
    for i in range(int(d["count"])):
        G = d[f"G{i}"]
        assert orc.sigma_max_sq(G) == d["est"][i]
        assert orc.sigma_max_sq(G, max_iters=5000) == d["est_long"][i]


def test_nnls_cases(golden):
    d = golden("nnls")
    for i in range(int(d["count"])):
        max_iter, tol, saf, calls = d["meta"][i]
        info = orc.SolveInfo()
        F = orc.nesterov_nnls(d[f"A{i}"], d[f"B{i}"], d[f"F0_{i}"], int(max_iter), tol, saf, info)
        assert np.array_equal(F, d[f"F{i}"]), f"case {i}"
        assert info.iterations - (1 if info.stopped_on_tol else 0) == int(calls), f"case {i}"


def test_rsi_and_compress(golden):
    d = golden("rsi")
    for name in d["names"]:
        nu, q, seed = (int(v) for v in d[f"{name}_par"])
        X = d[f"{name}_X"]
        L, R = orc.rsi(X, nu, q, seed)
        assert np.array_equal(L, d[f"{name}_L"]), name
        assert np.array_equal(R, d[f"{name}_R"]), name
        XL, XR = orc.compress(X, L, R)
        assert np.array_equal(XL, d[f"{name}_XL"]), name
        assert np.array_equal(XR, d[f"{name}_XR"]), name


def _trace(res):
    return np.array([[t, r, o] for t, r, o in res.records])


def test_factorize_small(golden):
    d = golden("factorize")
    X, G0, F0 = d["small_X"], d["small_G0"], d["small_F0"]
    van = orc.nenmf(X, G0, F0, max_outer=12, max_iter=500)
    assert np.array_equal(_trace(van), d["small_vanilla_trace"])
    assert np.array_equal(van.G, d["small_vanilla_G"]) and np.array_equal(van.F, d["small_vanilla_F"])
    com = orc.nenmf(X, G0, F0, L=d["small_L"], R=d["small_R"], max_outer=12, max_iter=500)
    assert np.array_equal(_trace(com), d["small_compressed_trace"])
    assert np.array_equal(com.G, d["small_compressed_G"])
    assert np.array_equal(com.F, d["small_compressed_F"])


def test_factorize_cadence(golden):
    d = golden("factorize")
    res = orc.nenmf(d["cadence_X"], d["cadence_G0"], d["cadence_F0"], max_outer=7, trace_every=3)
    tr = _trace(res)
    assert list(tr[:, 0]) == [0, 3, 6, 7]
    assert np.array_equal(tr, d["cadence_trace"])


def test_config1(golden):
    from paper_1812_04315_b200 import workloads

    d = golden("config1")
    w = workloads.make_workload(1)
    assert np.array_equal(d["x_checksum"], np.array([w.X.sum(), (w.X * w.X).sum()]))
    L, R = orc.rsi(w.X, w.nu, w.q, w.sketch_seed)
    assert np.array_equal(L, d["L"]) and np.array_equal(R, d["R"])
    com = orc.nenmf(w.X, w.G0, w.F0, L=L, R=R, max_outer=w.outer, max_iter=w.inner)
    assert np.array_equal(_trace(com), d["compressed_trace"])
    van = orc.nenmf(w.X, w.G0, w.F0, max_outer=w.outer, max_iter=w.inner)
    assert np.array_equal(_trace(van), d["vanilla_trace"])
    assert np.array_equal(van.F, d["vanilla_F"])


def test_seeded_draws(golden):
    from paper_1812_04315_b200 import init_factors, uniform_matrix, gaussian_matrix, workloads

    d = golden("seeds")
    for b, row in zip(d["base"], d["derived"]):
        assert [orc.derive_seed(int(b), s) for s in (0, 1, 2)] == [int(v) for v in row]
        assert [workloads.derive_seed(int(b), s) for s in (0, 1, 2)] == [int(v) for v in row]
    G, F = orc.initial_pair(7, 9, 3, 11)
    assert np.array_equal(G, d["init_G"]) and np.array_equal(F, d["init_F"])
    pair = init_factors(7, 9, 3, 11)
    assert np.array_equal(pair.G, d["init_G"]) and np.array_equal(pair.F, d["init_F"])
    assert np.array_equal(uniform_matrix(5, 4, 3), d["uniform"])
    assert np.array_equal(gaussian_matrix(4, 5, 3), d["gauss"])


def test_power_pair(golden):
    """oracle.power_pair against the reference's power_iteration_pair
    (compression.py:144-176): sketches bit-equal, overflow step equal."""
    d = golden("power")
    for name in d["names"]:
        nu, q, seed = (int(v) for v in d[f"{name}_par"])
        L, R = orc.power_pair(d[f"{name}_X"], nu, q, seed)
        assert np.array_equal(L, d[f"{name}_L"]), name
        assert np.array_equal(R, d[f"{name}_R"]), name
    nu, q, seed, step = (int(v) for v in d["overflow_par"])
    with pytest.raises(orc.OracleFailure) as exc:
        orc.power_pair(d["overflow_X"], nu, q, seed)
    assert exc.value.kind == "NumericalCollapseError" and exc.value.iteration == step
