"""Device Gaussian sketch draws (rng.cu) against NumPy itself: the reference
draws Omega_L then Omega_R from one default_rng(seed).standard_normal stream
(compression.py:130-132); the device stream must be BIT-identical (fp64) and
equal to NumPy's values rounded once (fp32)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,nu,seed", [(7, 5, 1, 0), (1000, 1000, 20, 12345), (10000, 10000, 30, 987654321),
                                         (100003, 2001, 26, 2**63 - 25), (333, 77777, 13, 42)])
def test_device_draws_bit_identical(n, m, nu, seed):
    from paper_1812_04315_b200 import _lib
    from paper_1812_04315_b200.compression import sketch_draws, sketch_draws_device

    ol, orr = sketch_draws(n, m, nu, seed)
    for dtype in ("fp64", "fp32"):
        olt, odr, ok = sketch_draws_device(n, m, nu, seed, dtype)
        assert int(ok.item()) == 1
        a, b = olt.cpu().numpy(), odr.cpu().numpy()
        if dtype == "fp64":
            assert np.array_equal(a, ol.T) and np.array_equal(b, orr)
        else:
            assert np.array_equal(a, ol.T.astype(np.float32)) and np.array_equal(b, orr.astype(np.float32))


def test_rsi_device_draws_match_host_draws():
    """The sketch from device draws equals the sketch from host draws bit for bit."""
    import torch
    from paper_1812_04315_b200 import _lib
    from paper_1812_04315_b200.compression import rsi_device, sketch_draws

    rng = np.random.default_rng(1)
    X = rng.random((500, 20)) @ rng.random((20, 400)) + 0.01 * rng.random((500, 400))
    Xd = _lib.to_device(X, "fp64")
    L, Rt, st = rsi_device(Xd, 12, 3, 77)
    ol, orr = sketch_draws(500, 400, 12, 77)
    host = (_lib.to_device(np.ascontiguousarray(ol.T), "fp64"), _lib.to_device(orr, "fp64"),
            torch.ones(1, dtype=torch.int32, device="cuda"))
    L2, Rt2, st2 = rsi_device(Xd, 12, 3, 77, draws=host)
    assert torch.equal(L, L2) and torch.equal(Rt, Rt2)
