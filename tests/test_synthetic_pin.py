"""Pin the NumPy restatement of the reference generator used by
tests/test_gpu_synthetic.py against the reference's own generate_problem
(synthetic.py:47-95), importable in the build container only."""
import importlib
import math
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))
from test_gpu_synthetic import _reference  # noqa: E402


@pytest.mark.parametrize("n,m,p,snr,seed", [(300, 200, 7, 20.0, 5), (64, 400, 3, 0.0, 2 ** 63 + 7),
                                            (50, 50, 10, math.inf, 1)])
def test_restatement_matches_reference(n, m, p, snr, seed):
    src = Path("/root/reference/pkg/src")
    if not src.is_dir():
        pytest.skip("reference not present")
    sys.path.insert(0, str(src))
    try:
        ref = importlib.import_module("nenmf.synthetic")
    finally:
        sys.path.remove(str(src))
    inst = ref.generate_problem(n, m, p, snr, seed)
    G, F, X, real = _reference(n, m, p, snr, seed)
    assert inst.G_true.tobytes() == G.tobytes() and inst.F_true.tobytes() == F.tobytes()
    assert inst.X.tobytes() == X.tobytes()
    assert inst.snr_db_realized == real or (math.isinf(real) and math.isinf(inst.snr_db_realized))
