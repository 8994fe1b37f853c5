"""B200-native powerURV / randUTV behind the utvkit API (arXiv 2106.13402).

Drop-in names mirror utvkit/__init__.py for the hot path; compute runs in
libutvb200.so (hand-written sm_100a CUDA behind a C ABI, include/utv_b200.h).
"""

from .errors import ConsistencyError, ConvergenceError, DimensionError
from .matrix import MACHINE_EPS, RngStream, check_matrix, frobenius_norm, gaussian
from .metrics import trailing_fro_curve
from .powerurv import UrvFactorization, power_urv, power_urv_from_sample, rurv
from .qr import PivotedQr, QFactor, apply_q, hqr_full, hqr_thin, hqrcp, materialize_q
from .randutv import (ErrorTracker, UtvFactorization, error_update, randutv_basic,
                      randutv_boosted, randutv_partial)
from .svd import SvdTriple, svd_dense, svd_tall_thin_left

__all__ = [
    "MACHINE_EPS", "RngStream", "gaussian", "frobenius_norm", "check_matrix",
    "QFactor", "PivotedQr", "hqr_full", "hqr_thin", "hqrcp", "apply_q", "materialize_q",
    "SvdTriple", "svd_dense", "svd_tall_thin_left",
    "UrvFactorization", "power_urv", "power_urv_from_sample", "rurv",
    "UtvFactorization", "ErrorTracker", "error_update", "randutv_basic",
    "randutv_boosted", "randutv_partial",
    "trailing_fro_curve",
    "DimensionError", "ConvergenceError", "ConsistencyError",
]
