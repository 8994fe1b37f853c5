"""Dense SVD with the reference sign convention — drop-in for utvkit
svd.py:18-58 (svd_dense) on the B200 one-sided Jacobi kernel (K6).

Square inputs go straight to Jacobi; tall inputs are QR-reduced first (the
same composition the reference uses in svd_tall_thin_left, svd.py:61-82) and
wide inputs are handled through the transpose.  For rectangular inputs the
columns of the full U (or V) beyond min(m, n) are an orthonormal completion;
like LAPACK's, they are not unique.
"""

from dataclasses import dataclass

import numpy as np

from ._lib import serialized as _serialized
from . import device as dv
from ._lib import dempty, dfrom_numpy
from .errors import ConvergenceError, DimensionError
from .matrix import check_matrix

#: Largest n the one-sided Jacobi kernel (utv_dgesvj, csrc/jacobi.cu) takes:
#: one cooperative grid holds the n x n block and its V in L2 / shared memory
#: and the finish kernel keeps a column per thread (1024 threads).
JACOBI_MAX_N = 1024
MAX_N = JACOBI_MAX_N


@dataclass(frozen=True)
class SvdTriple:
    """A = U @ diag(sigma) @ V.T with sigma sorted descending (svd.py:18-25)."""

    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    thin: bool


def _jacobi(d):
    sig, U, V, status = dv.gesvj(d)
    st = int(status.cpu().item())
    if st < 0:
        raise ConvergenceError(f"SVD failed to converge on shape ({d.rows}, {d.cols})")
    return sig, U, V


def _sign_fix(u, v):
    for j in range(v.shape[1]):
        i = int(np.argmax(np.abs(v[:, j])))
        if v[i, j] < 0.0:
            v[:, j] = -v[:, j]
            u[:, j] = -u[:, j]


@_serialized
def svd_dense(a, mode="full"):
    """Dense SVD with deterministic signs (svd.py:37-58)."""
    a = check_matrix(a)
    if mode not in ("full", "thin"):
        raise ValueError(f"mode must be 'full' or 'thin', got {mode!r}")
    m, n = a.shape
    if m < n:
        t = svd_dense(a.T, mode)
        u, v = np.array(t.V, order="F"), np.array(t.U, order="F")
        r = min(m, n)
        # re-apply the sign rule to the swapped factors (V's largest entry positive)
        _sign_fix(u[:, :r], v[:, :r])
        return SvdTriple(U=u, sigma=t.sigma, V=v, thin=(mode == "thin"))
    if n > MAX_N:
        raise ValueError(f"svd_dense on the B200 path supports min(m, n) <= {MAX_N} "
                         "(the Jacobi kernel's limit)")
    if m == n:
        sig, U, V = _jacobi(dfrom_numpy(a))
        return SvdTriple(U=np.asfortranarray(U.to_numpy()), sigma=sig.cpu().numpy()[:n].copy(),
                         V=np.asfortranarray(V.to_numpy()), thin=(mode == "thin"))
    d = dfrom_numpy(a)
    Y, T = dv.geqrf(d)
    r = dfrom_numpy(d.to_numpy()[:n, :])
    sig, Us, V = _jacobi(r)
    if mode == "thin":
        q = dv.orgqr(Y, T, n)
        u = dv.gemm("N", "N", 1.0, q, Us)
    else:
        c = np.zeros((m, m), order="F")
        c[:n, :n] = Us.to_numpy()
        c[n:, n:] = np.eye(m - n)
        dc = dfrom_numpy(c)
        dv.larfb("L", False, Y, T, dc)
        u = dc
    return SvdTriple(U=np.asfortranarray(u.to_numpy()), sigma=sig.cpu().numpy()[:n].copy(),
                     V=np.asfortranarray(V.to_numpy()), thin=(mode == "thin"))


@_serialized
def svd_tall_thin_left(y):
    """Left singular vectors of a tall thin y (n x w, n >= w) completed to an
    orthogonal n x n W = Q blockdiag(Uhat, I) (svd.py:61-82): one device
    Householder QR of y, the w x w Jacobi SVD of R[:w, :], one compact-WY
    apply of Q to the block-diagonal completion.  w <= JACOBI_MAX_N."""
    y = check_matrix(y)
    n, w = y.shape
    if n < w:
        raise DimensionError(f"svd_tall_thin_left needs rows >= cols, got {y.shape}")
    if w > JACOBI_MAX_N:
        raise ValueError(f"svd_tall_thin_left on the B200 path supports cols <= {JACOBI_MAX_N}")
    d = dfrom_numpy(y)
    Y, T = dv.geqrf(d)                       # d <- R (zeros below the diagonal)
    r = dempty(w, w)
    dv.lacpy(d.sub(0, 0, w, w), r)
    _, uhat, _ = _jacobi(r)
    c = dempty(n, n)
    dv.laset("A", 0.0, 1.0, c)
    dv.lacpy(uhat, c.sub(0, 0, w, w))
    dv.larfb("L", False, Y, T, c)
    return np.asfortranarray(c.to_numpy())
