"""The device restatement of the C library's log1p (csrc/glibc_log1p.cuh),
compiled here for the host from the SAME header, must equal libm's log1p bit
for bit on the arguments the ziggurat tail feeds it (-u, u = k 2^-53 in
[0, 1)); the sketch's Gaussian draws (compression.py:130-132 -> NumPy's
random_standard_normal) are then NumPy's exactly with no host fix-up."""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
HDR = REPO / "paper_1812_04315_b200" / "csrc" / "glibc_log1p.cuh"

HARNESS = r"""
#include "glibc_log1p.cuh"
extern "C" long check_range(unsigned long long seed, long count, double* worst) {
  long bad = 0;
  unsigned long long st = seed;
  for (long i = 0; i < count; ++i) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    const unsigned long long r = st ^ (st >> 29);
    const unsigned long long u53 = (i & 1) ? (r >> 11) : (r >> (11 + (r & 63) % 42));
    const double x = -((double)u53 * (1.0 / 9007199254740992.0));
    if (glibc_log1p(x) != log1p(x)) { ++bad; *worst = x; }
  }
  return bad;
}
extern "C" double restated(double x) { return glibc_log1p(x); }
"""


def _cpu_has_fma() -> bool:
    try:
        return " fma " in Path("/proc/cpuinfo").read_text()
    except OSError:
        return False


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    d = tmp_path_factory.mktemp("l1p")
    src = d / "h.cpp"
    src.write_text(HARNESS)
    so = d / "h.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fno-builtin", "-shared", "-fPIC", f"-I{HDR.parent}",
                    str(src), "-o", str(so), "-lm"], check=True)
    h = ctypes.CDLL(str(so))
    h.check_range.restype = ctypes.c_long
    h.check_range.argtypes = [ctypes.c_ulonglong, ctypes.c_long, ctypes.POINTER(ctypes.c_double)]
    h.restated.restype = ctypes.c_double
    h.restated.argtypes = [ctypes.c_double]
    return h


@pytest.mark.skipif(not _cpu_has_fma(), reason="glibc selects its FMA log1p only on FMA-capable CPUs")
def test_restated_log1p_equals_libm(lib):
    worst = ctypes.c_double(0.0)
    bad = lib.check_range(0x853C49E6748FEA9B, 20_000_000, ctypes.byref(worst))
    assert bad == 0, f"{bad} mismatches, e.g. at {worst.value!r}"


def test_restated_log1p_edges(lib):
    import math

    for x in (0.0, -0.0, -1e-300, -2.0 ** -54, -2.0 ** -30, -1e-9, -0.25, -0.2929, -0.5, -0.75,
              -(1 - 2.0 ** -53), 1e-20, 0.3, 0.41, 1.0, 7.5, 1e300):
        assert lib.restated(x) == math.log1p(x) or (x == 0 and lib.restated(x) == 0), x
    assert lib.restated(-1.0) == -math.inf
    assert np.isnan(lib.restated(-2.0))
