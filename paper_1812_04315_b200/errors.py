"""Exception classes of the drop-in API and the C-ABI status-code mapping.

Class names, base classes and attributes follow the reference hierarchy
(``/root/reference/pkg/src/nenmf/errors.py:6-52``) so that code catching the
reference's exceptions catches these.  Status codes returned by
``libnenmf_b200`` (``include/nenmf_b200.h``) are translated here.
"""

from __future__ import annotations


class NenmfError(Exception):
    """Root of every error this package raises on purpose (errors.py:6)."""


class DimensionError(NenmfError, ValueError):
    """Shapes that cannot be combined, or empty dimensions (errors.py:10)."""


class ZeroMatrixError(NenmfError, ValueError):
    """An operand that must be nonzero is identically zero (errors.py:14)."""


class RankDeficiencyError(NenmfError):
    """Strict QR basis found fewer independent columns (errors.py:18-27)."""

    def __init__(self, message: str, detected_rank: int):
        super().__init__(message)
        self.detected_rank = detected_rank


class NumericalFailureError(NenmfError):
    """Non-finite solver state (errors.py:30-40).

    ``iteration`` is the inner index, ``outer_iteration`` the alternating-loop
    index when raised from a factorization.
    """

    def __init__(self, message: str, iteration: int, outer_iteration: int | None = None):
        super().__init__(message)
        self.iteration = iteration
        self.outer_iteration = outer_iteration


class NumericalCollapseError(NumericalFailureError):
    """Sketch iterate overflowed or lost all directions (errors.py:43-44)."""


class ComparisonValidityError(NenmfError):
    """Traces with mismatched metadata (errors.py:47-48)."""


class ConfigError(NenmfError, ValueError):
    """Run configuration rejected up front (errors.py:51-52)."""


class BackendError(NenmfError, RuntimeError):
    """The CUDA library is missing, or a CUDA/launch error occurred.  There is
    no CPU fallback: every compute entry point raises this instead."""


# C-ABI status codes (include/nenmf_b200.h, enum nenmf_status_code)
ST_OK = 0
ST_DIM = 1
ST_ZERO_MATRIX = 2
ST_NUMERICAL_FAILURE = 3
ST_NUMERICAL_COLLAPSE = 4
ST_VALUE = 5
ST_CUDA = 6
ST_WORKSPACE = 7
ST_UNSUPPORTED = 8
ST_WATCHDOG = 9  # a persistent solve made no progress for NENMF_WATCHDOG_S seconds (default 60)


def raise_for_status(code: int, iteration: int = -1, what: str = "") -> None:
    """Translate a library or device status word into the reference's
    exception class.  ``iteration`` is the device-recorded inner index."""
    if code == ST_OK:
        return
    where = f" ({what})" if what else ""
    if code == ST_DIM:
        raise DimensionError(f"incompatible dimensions{where}")
    if code == ST_ZERO_MATRIX:
        raise ZeroMatrixError(f"operand is all zero or its Gram underflowed{where}")
    if code == ST_NUMERICAL_FAILURE:
        raise NumericalFailureError(f"non-finite iterate{where}", iteration=iteration)
    if code == ST_NUMERICAL_COLLAPSE:
        raise NumericalCollapseError(f"sketch iterate collapsed{where}", iteration=iteration)
    if code == ST_VALUE:
        raise ValueError(f"invalid value{where}")
    if code == ST_UNSUPPORTED:
        raise BackendError(f"shape outside the kernels' supported range{where}")
    if code == ST_WATCHDOG:
        raise BackendError(f"solver made no progress within NENMF_WATCHDOG_S (a stalled peer rank or a "
                           f"preempted device){where}")
    raise BackendError(f"libnenmf_b200 status {code}{where}")
