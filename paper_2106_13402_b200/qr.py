"""Householder QR in compact-WY form — drop-in for utvkit qr.py:17-138.

Same functions, arguments, return types and exceptions as the reference;
the arithmetic runs on the B200 (libutvb200: K3/K4 geqrf, K2 larfb, K5
orgqr).  Inputs are numpy arrays; outputs are fresh float64 F-order arrays.
"""

from dataclasses import dataclass

import numpy as np

from ._lib import serialized as _serialized
from . import device as dv
from ._lib import dfrom_numpy
from .errors import DimensionError
from .matrix import check_matrix


@dataclass(frozen=True)
class QFactor:
    """Q = I - Y @ Twy @ Y.T; Y m x k unit lower trapezoidal, Twy k x k upper (qr.py:17-31)."""

    Y: np.ndarray
    Twy: np.ndarray
    m: int

    @property
    def k(self):
        return self.Y.shape[1]


@dataclass(frozen=True)
class PivotedQr:
    """Column-pivoted QR: ``A[:, perm] = Q @ R`` with |diag R| non-increasing (qr.py:35-40)."""

    q: QFactor
    R: np.ndarray
    perm: np.ndarray


@_serialized
def hqr_full(a):
    """Full unpivoted Householder QR (m >= n) -> (QFactor, R); qr.py:71-100."""
    a = check_matrix(a)
    m, n = a.shape
    if m < n:
        raise DimensionError(f"hqr_full needs m >= n, got {a.shape}; factor the transpose")
    d = dfrom_numpy(a)
    Y, T = dv.geqrf(d)
    return QFactor(Y=Y.to_numpy(), Twy=T.to_numpy(), m=m), d.to_numpy()


@_serialized
def apply_q(q, b, side="left", trans=False):
    """Q @ b, Q.T @ b (left) or b @ Q, b @ Q.T (right), three GEMMs; qr.py:103-121."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 2:
        raise DimensionError(f"apply_q operand must be 2-D, got shape {b.shape}")
    if side == "left":
        if b.shape[0] != q.m:
            raise DimensionError(f"apply_q left: operand has {b.shape[0]} rows, Q is {q.m}x{q.m}")
    elif side == "right":
        if b.shape[1] != q.m:
            raise DimensionError(f"apply_q right: operand has {b.shape[1]} cols, Q is {q.m}x{q.m}")
    else:
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    if b.size == 0:
        return b.copy()
    d = dfrom_numpy(b)
    dv.larfb("L" if side == "left" else "R", bool(trans), dfrom_numpy(q.Y), dfrom_numpy(q.Twy), d)
    return d.to_numpy()


@_serialized
def materialize_q(q, ncols=None):
    """Leading ncols columns of Q (all m by default); qr.py:124-131."""
    ncols = q.m if ncols is None else int(ncols)
    if not 1 <= ncols <= q.m:
        raise DimensionError(f"ncols must be in [1, {q.m}], got {ncols}")
    return dv.orgqr(dfrom_numpy(q.Y), dfrom_numpy(q.Twy), ncols).to_numpy()


@_serialized
def hqr_thin(a):
    """Thin QR: (Qhat m x n orthonormal, Rhat n x n); qr.py:134-138."""
    q, r = hqr_full(a)
    n = np.asarray(a).shape[1]
    return materialize_q(q, ncols=n), np.array(r[:n, :], copy=True)


@_serialized
def hqrcp(a):
    """Column-pivoted Householder QR (greedy largest-norm pivoting) — the
    paper's comparator, qr.py:152-204, as one persistent cooperative kernel
    (csrc/qrcp.cu).  Same pivots (1e-12 tie window, leftmost), skip rule and
    norm downdate/recompute as the reference; any m x n (beyond 16384 rows or
    columns the kernel keeps its per-CTA reflector in global memory)."""
    a = check_matrix(a)
    m, n = a.shape
    lim = dv.geqp3_max_dim()
    if m > lim or n > lim:
        raise DimensionError(f"hqrcp on the B200 path supports up to {lim} rows/cols, got {a.shape}")
    R, Y, T, perm = dv.geqp3(dfrom_numpy(a))
    return PivotedQr(q=QFactor(Y=Y.to_numpy(), Twy=T.to_numpy(), m=m), R=R.to_numpy(),
                     perm=perm.cpu().numpy().astype(np.int64))
