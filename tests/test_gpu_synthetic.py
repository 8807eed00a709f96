"""generate_problem_device against the reference's
generator restated in NumPy (synthetic.py:47-95): G and F bit-identical (same
PCG64 stream), X to rounding (GEMM / norm summation order), realized SNR."""
import math

import numpy as np
import pytest

from paper_1812_04315_b200.synthetic import generate_problem_device

pytestmark = pytest.mark.gpu


def _reference(n, m, p, snr_db, seed):
    rng = np.random.default_rng(seed)
    G = rng.random((n, p))
    F = rng.random((p, m))
    assert (G != 0).all() and (F != 0).all()
    Xc = G @ F
    if snr_db == math.inf:
        return G, F, Xc, math.inf
    N = rng.standard_normal((n, m))
    cn = np.linalg.norm(Xc)
    N *= cn * 10.0 ** (-snr_db / 20.0) / np.linalg.norm(N)
    return G, F, Xc + N, 10.0 * math.log10((cn / np.linalg.norm(N)) ** 2)


@pytest.mark.parametrize("n,m,p,snr,seed", [(300, 200, 7, 20.0, 5), (1000, 1500, 15, 30.0, 9901),
                                            (64, 4000, 3, 0.0, 2 ** 63 + 7), (250, 250, 10, math.inf, 1),
                                            (400, 300, 100, 25.0, 77)])  # p above 64
def test_device_generator_matches_reference(n, m, p, snr, seed):
    G, F, X, real = _reference(n, m, p, snr, seed)
    inst = generate_problem_device(n, m, p, snr, seed)
    assert inst.G_true.cpu().numpy().tobytes() == G.tobytes()
    assert inst.F_true.cpu().numpy().tobytes() == F.tobytes()
    Xd = inst.X.cpu().numpy()
    assert np.abs(Xd - X).max() <= 1e-12 * np.abs(X).max()
    if snr == math.inf:
        assert inst.snr_db_realized == math.inf
    else:
        assert abs(inst.snr_db_realized - real) <= 1e-9 and abs(real - snr) <= 1e-9


def test_device_generator_fp32_and_errors():
    inst = generate_problem_device(200, 300, 5, 20.0, 3, dtype="fp32")
    G, F, X, _ = _reference(200, 300, 5, 20.0, 3)
    assert inst.X.dtype.is_floating_point and inst.X.element_size() == 4
    assert np.abs(inst.X.cpu().numpy() - X.astype(np.float32)).max() <= 1e-6 * np.abs(X).max()
    from paper_1812_04315_b200.errors import DimensionError
    with pytest.raises(DimensionError):
        generate_problem_device(10, 10, 11, 20.0, 1)
    with pytest.raises(ValueError):
        generate_problem_device(10, 10, 2, float("nan"), 1)
