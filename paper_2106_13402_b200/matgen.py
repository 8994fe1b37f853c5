"""Test-matrix generators on the B200 — drop-in for utvkit matgen.py:1-98
(SURVEY.md §8f row 2).  Same names, signatures, spectra and RNG draw order
as the reference, so gen_fast_decay(n, beta, RngStream(s)) yields the
reference's matrix up to roundoff; the orthogonal factors come from our
device Householder QR (K3/K4) instead of the reference's Python column loop
(51 s at n = 2000 there, milliseconds here), and A = U diag(d) V^T is one
DMMA GEMM.  The *_device variants keep the result in HBM (DMat)."""

import numpy as np

from . import device as dv
from ._lib import DMat, dempty, load, stream_ptr
from .errors import DimensionError

KINDS = ("fast", "s", "bie", "kahan", "gaussian")

_S_SHAPE_FLOOR = 1e-2          # matgen.py:41-43
_S_SHAPE_STEEPNESS = 60.0


def _draw_square(n, rng):
    """gaussian(n, n, rng) (matrix.py:52-60) on the device: the C-order draw
    goes up as its transpose and is transposed there."""
    if n < 1:
        raise DimensionError(f"gaussian dimensions must be positive, got ({n}, {n})")
    return dv.from_numpy_any_order(np.asarray(rng.standard_normal(int(n), int(n))))


def random_orthogonal_device(n, rng) -> DMat:
    """Q of hqr_full(gaussian(n, n, rng)), materialised (matgen.py:17-21)."""
    g = _draw_square(n, rng)
    y, t = dv.geqrf(g)
    return dv.orgqr(y, t, n)


def random_orthogonal(n, rng):
    return random_orthogonal_device(n, rng).to_numpy()


def _from_spectrum_device(d, rng) -> DMat:
    """U diag(d) V^T with U, V random orthogonal, U drawn first (matgen.py:24-28)."""
    import torch
    n = d.shape[0]
    u = random_orthogonal_device(n, rng)
    v = random_orthogonal_device(n, rng)
    dd = torch.from_numpy(np.ascontiguousarray(d, dtype=np.float64)).cuda()
    dv.diag_scale("R", dd, v)                         # V diag(d)
    return dv.gemm("N", "T", 1.0, u, v)               # U (V diag(d))^T


def _fast_spectrum(n, beta):
    if n < 2:
        raise DimensionError(f"fast-decay matrix needs n >= 2, got {n}")
    if not 0.0 < beta < 1.0:
        raise ValueError(f"beta must be in (0, 1), got {beta}")
    return beta ** (np.arange(n) / (n - 1))


def _s_spectrum(n):
    if n < 8:
        raise DimensionError(f"S-shaped matrix needs n >= 8, got {n}")
    i = np.arange(1, n + 1, dtype=np.float64)
    d = _S_SHAPE_FLOOR + (1.0 - _S_SHAPE_FLOOR) / (1.0 + np.exp(_S_SHAPE_STEEPNESS * (i - n / 4.0) / n))
    return np.minimum.accumulate(d)


def gen_fast_decay_device(n, beta, rng):
    d = _fast_spectrum(n, beta)
    return _from_spectrum_device(d, rng), d


def gen_fast_decay(n, beta, rng):
    """Geometric spectrum d_i = beta^((i-1)/(n-1)) (matgen.py:31-38)."""
    a, d = gen_fast_decay_device(n, beta, rng)
    return a.to_numpy(), d


def gen_s_shaped_device(n, rng):
    d = _s_spectrum(n)
    return _from_spectrum_device(d, rng), d


def gen_s_shaped(n, rng):
    """Near 1, fast drop, plateau at 1e-2 (matgen.py:46-55)."""
    a, d = gen_s_shaped_device(n, rng)
    return a.to_numpy(), d


def gen_bie_device(n) -> DMat:
    if n < 16:
        raise DimensionError(f"BIE matrix needs n >= 16, got {n}")
    a = dempty(n, n)
    dv.check(load().utv_dgen_bie(n, a.ptr, a.ld, stream_ptr()), "utv_dgen_bie")
    return a


def gen_bie(n):
    """Discretised single-layer log kernel on the unit circle (matgen.py:58-76)."""
    return gen_bie_device(n).to_numpy()


def gen_kahan_device(n, theta=1.2) -> DMat:
    if n < 1:
        raise DimensionError(f"Kahan matrix needs n >= 1, got {n}")
    if not 0.0 < theta < np.pi / 2.0:
        raise ValueError(f"theta must be in (0, pi/2), got {theta}")
    a = dempty(n, n)
    dv.check(load().utv_dgen_kahan(n, float(theta), a.ptr, a.ld, stream_ptr()), "utv_dgen_kahan")
    return a


def gen_kahan(n, theta=1.2):
    """Kahan's upper triangular matrix (matgen.py:79-91)."""
    return gen_kahan_device(n, theta).to_numpy()


def gen_gaussian(n, rng):
    """Square standard Gaussian matrix (matgen.py:94-96): a host draw."""
    return np.asfortranarray(rng.standard_normal(int(n), int(n)))
