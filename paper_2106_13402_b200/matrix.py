"""Host-side matrix basics mirrored from utvkit matrix.py (the parts the hot
path uses): the seeded Gaussian stream that produces G, input validation,
the Frobenius norm and MACHINE_EPS.

The Gaussian draws stay on the host (numpy PCG64 + ziggurat) so that G is
bit-identical to the reference's (matrix.py:16-33, 52-60); all arithmetic on
A happens on the device.
"""

import numpy as np

from .errors import DimensionError

#: Machine epsilon for IEEE double precision (matrix.py:13).
MACHINE_EPS = float(np.finfo(np.float64).eps)


class RngStream:
    """Seeded stream of standard normals; same generator as matrix.py:16-33."""

    def __init__(self, seed):
        self.seed = int(seed)
        self._gen = np.random.Generator(np.random.PCG64(self.seed))

    def standard_normal(self, m, n):
        # large draws: the same stream generated on all host cores (fastrng)
        from .fastrng import standard_normal
        return standard_normal(self._gen, (m, n))

    def __repr__(self):
        return f"RngStream(seed={self.seed})"


def check_matrix(a, name="matrix", finite=True):
    """float64 cast, 2-D, positive dims, all finite (matrix.py:36-49).

    finite=False skips the host scan: callers that upload the matrix anyway
    run the same check on the device (raise_if_nonfinite) before any draw."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {a.shape}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise DimensionError(f"{name} must have positive dimensions, got {a.shape}")
    if finite and not np.isfinite(a).all():
        raise ValueError(f"{name} contains NaN or Inf entries")
    return a


def raise_if_nonfinite(d, name="matrix"):
    """The finite half of check_matrix, on a device copy (DMat): one
    libutvb200 scan (utv_dnonfinite) and a 4-byte read back."""
    import torch
    from ._lib import check, load, stream_ptr
    flag = torch.empty(1, dtype=torch.int32, device="cuda")
    check(load().utv_dnonfinite(d.rows, d.cols, d.ptr, d.ld, flag.data_ptr(), stream_ptr()),
          "utv_dnonfinite")
    if int(flag.item()):
        raise ValueError(f"{name} contains NaN or Inf entries")


def gaussian(m, n, rng):
    """m x n i.i.d. standard normals, C-order draw then Fortran copy (matrix.py:52-60)."""
    if m < 1 or n < 1:
        raise DimensionError(f"gaussian dimensions must be positive, got ({m}, {n})")
    return np.asfortranarray(rng.standard_normal(int(m), int(n)))


def frobenius_norm(a):
    """Square root of the sum of squared entries (matrix.py:79-81)."""
    return float(np.linalg.norm(np.asarray(a, dtype=np.float64)))
