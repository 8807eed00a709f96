"""The FP32 residual on the tensor cores (k_resid_bulk, nenmf_residual_sumsq_prepared):
||X - G F||^2 read from the prepared X, against the fp64 oracle on the
fp32-rounded inputs (the RRE emit, tracing.py:45-57 / factorize.py:139), and
the explicit-residual pair of the vanilla tie-break (nnls.py:219-227) against
the CUDA-core pair.

Error model: the prepared X carries X to 16 significant
bits, the products carry the BF16x3 error (~2^-17 relative per operand) and
the tensor-core accumulator truncates; with e the per-entry error of R,
||R + e||^2 - ||R||^2 = 2<R, e> + ||e||^2.  The second-order term is
~(2^-17 |x| / |r|)^2; the first-order term is zero-mean for a zero-mean
residual but not for the nonnegative noise of these problems, where any bias
of e enters as 2 delta |x| / |r|.  The tolerance is therefore
2 eps ratio + 4 (eps ratio)^2 with ratio = |X| / |R| and eps = 2^-17, the
same bound for the CUDA-core pass over the raw X (3xTF32, truncating
accumulator).  Measured at cfg2 scale (ratio ~1000): 2e-4 prepared, 8e-4 raw."""

import numpy as np
import pytest

import paper_1812_04315_b200 as nm  # noqa: F401  (loads the library)
from paper_1812_04315_b200 import _lib, _ops

pytestmark = pytest.mark.gpu


def _problem(n, m, p, noise, seed):
    rng = np.random.default_rng(seed)
    G = rng.random((n, p))
    F = rng.random((p, m))
    X = G @ F + noise * rng.random((n, m))
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    return f32(X), f32(G), f32(F)


def _device_resid(X, G, F, prepared: bool):
    _, torch = _lib.require_device()
    Xd = _lib.to_device(X, "fp32")
    Gt = _lib.to_device(np.ascontiguousarray(G.T), "fp32")
    Fd = _lib.to_device(F, "fp32")
    out = _lib.zeros(1, torch.float64)
    Xp = _ops.prepare_x(Xd, G.shape[1]) if prepared else None
    if prepared:
        assert Xp is not None
    _ops.residual_sumsq(Xd, Gt, Fd, out, Xp=Xp)
    return float(out[0].item())


@pytest.mark.parametrize("n,m,p,noise", [
    (128, 128, 1, 0.01), (300, 257, 6, 0.01), (1000, 777, 16, 0.05), (513, 1100, 17, 0.01),
    (2048, 1536, 32, 0.01), (129, 4000, 20, 0.2)])
def test_resid_prepared_vs_oracle(n, m, p, noise):
    X, G, F = _problem(n, m, p, noise, seed=n + m + p)
    ref = float(np.sum((X - G @ F) ** 2))  # fp64 oracle on the same fp32 inputs
    got = _device_resid(X, G, F, prepared=True)
    ratio = np.linalg.norm(X) / np.sqrt(ref)  # |x| / |r|
    eps = 2.0 ** -17
    tol = 2.0 * eps * ratio + 4.0 * (eps * ratio) ** 2
    assert abs(got - ref) <= tol * ref, (got, ref, tol)
    raw = _device_resid(X, G, F, prepared=False)
    assert abs(raw - ref) <= tol * ref, (raw, ref, tol)


def test_resid_prepared_exact_fit_floor():
    """X = G F exactly (in fp32): the residual is pure representation error;
    its RRE floor stays below 2^-14 (the FP32 path's RRE targets are >= 1e-3)."""
    X, G, F = _problem(700, 650, 12, 0.0, seed=3)
    got = _device_resid(X, G, F, prepared=True)
    assert np.sqrt(got) / np.linalg.norm(X) <= 2.0 ** -14


def test_resid_prepared_fallback_shapes():
    """p > 32 has no prepared form: the call falls back to the raw X (same
    value as the plain entry point)."""
    X, G, F = _problem(300, 200, 40, 0.01, seed=5)
    _, torch = _lib.require_device()
    Xd = _lib.to_device(X, "fp32")
    Xp = _ops.prepare_x(Xd, 8)  # a prepared copy exists (k = 8), the residual's p = 40 does not fit it
    Gt = _lib.to_device(np.ascontiguousarray(G.T), "fp32")
    Fd = _lib.to_device(F, "fp32")
    a, b = _lib.zeros(1, torch.float64), _lib.zeros(1, torch.float64)
    _ops.residual_sumsq(Xd, Gt, Fd, a, Xp=Xp)
    _ops.residual_sumsq(Xd, Gt, Fd, b)
    assert float(a[0].item()) == float(b[0].item())


@pytest.mark.parametrize("trans_b", [False, True])
def test_tiebreak_pair_prepared(trans_b):
    """One vanilla half-step (nenmf_solve_nnls_prepared, V and the tie-break
    pair from the prepared X) against the CUDA-core half-step: the pair of
    explicit residuals (best, start) written to the status agrees to the
    error model, and both take the same decision (returned_best)."""
    _, torch = _lib.require_device()
    n, m, p = 900, 700, 10
    X, G, F = _problem(n, m, p, 0.02, seed=11)
    rng = np.random.default_rng(12)
    Xd = _lib.to_device(X, "fp32")
    Xp = _ops.prepare_x(Xd, p)
    if trans_b:   # G-half: A = F^T (At = F), B = X^T read in place; solve for Gt (p x n)
        At = _lib.to_device(F, "fp32")
        F0 = _lib.to_device(np.ascontiguousarray(G.T) * (1 + 0.3 * rng.random((p, n))), "fp32")
    else:         # F-half: A = G (At = Gt), B = X; solve for F (p x m)
        At = _lib.to_device(np.ascontiguousarray(G.T), "fp32")
        F0 = _lib.to_device(F * (1 + 0.3 * rng.random((p, m))), "fp32")
    res = {}
    for prepared in (False, True):
        Fo = torch.empty_like(F0)
        st = _lib.new_status()
        _ops.solve(At, Xd, F0, Fo, trans_b=trans_b, max_iter=40, grad_tol=1e-6, lipschitz_safety=1.0,
                   status=st, Xp=Xp if prepared else None)
        s = _lib.read_status(st)[0]
        assert int(s["code"]) == 0
        res[prepared] = (int(s["returned_best"]), np.array(s["resid"]), _lib.to_host(Fo))
    (b0, r0, f0), (b1, r1, f1) = res[False], res[True]
    assert b0 == b1 == 1
    eps = 2.0 ** -17
    ratio = np.linalg.norm(X) / np.sqrt(2.0 * r0)  # status holds 1/2 ||R||^2
    tol = 2.0 * eps * ratio + 4.0 * (eps * ratio) ** 2
    assert np.all(np.abs(r1 - r0) <= tol * np.abs(r0)), (r0, r1, tol)
    assert np.linalg.norm(f1 - f0) <= 1e-3 * np.linalg.norm(f0)
