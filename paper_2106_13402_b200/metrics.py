"""Parity metrics: e_k curve bench.py:63-72 and friends."""

import numpy as np

from .matrix import check_matrix


def trailing_fro_curve(t):
    """||T[k:, k:]||_F for k = 1..n-1 via a 2-D suffix sum (bench.py:63-72)."""
    t = check_matrix(t)
    m, n = t.shape
    sq = t * t
    suffix = np.cumsum(np.cumsum(sq[::-1, ::-1], axis=0), axis=1)[::-1, ::-1]
    vals = np.array([suffix[k, k] if k < m else 0.0 for k in range(1, n)])
    return np.sqrt(np.maximum(vals, 0.0))


# ---------------------------------------------------------------------------
# device-side metrics: the same quantities computed in
# HBM, for full-size (n = 16384) parity checks without host copies
# ---------------------------------------------------------------------------

def trailing_fro_curve_device(t_dev):
    """||T[k:, k:]||_F, k = 1..n-1 of a device matrix (bench.py:63-72)."""
    import torch

    from . import _lib
    lib = _lib.load()
    m, n = t_dev.rows, t_dev.cols
    out = torch.zeros(max(n - 1, 1), dtype=torch.float64, device="cuda")
    lw = lib.utv_dtrailing_fro_bufsize(m, n)
    ws = _lib.workspace(lw)
    _lib.check(lib.utv_dtrailing_fro(m, n, t_dev.ptr, t_dev.ld, out.data_ptr(), ws.data_ptr(), lw,
                                     _lib.stream_ptr()), "utv_dtrailing_fro")
    return out[: max(n - 1, 0)].cpu().numpy()


def reconstruction_device(a_dev, u_dev, t_dev, v_dev):
    """||A - U T V^T||_F / ||A||_F on the device (two DMMA GEMMs + reductions)."""
    import math

    from . import device as dv
    w = dv.gemm("N", "N", 1.0, u_dev, t_dev)                 # U T
    r = dv.copy(a_dev)
    dv.gemm("N", "T", -1.0, w, v_dev, 1.0, r)               # A - (U T) V^T
    num = float(dv.sumsq(r).item())
    den = float(dv.sumsq(a_dev).item())
    return math.sqrt(num) / math.sqrt(den)


def orthogonality_device(q_dev):
    """||Q^T Q - I||_F on the device."""
    import math

    from . import device as dv
    g = dv.gemm("T", "N", 1.0, q_dev, q_dev)
    return math.sqrt(float(_offset_identity_sumsq(g)))


def _offset_identity_sumsq(g):
    """sum((G - I)^2) with the identity subtracted on the device."""
    import torch

    from . import device as dv
    n = g.rows
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    idx = torch.arange(n, device="cuda")
    g.t[idx, idx] -= ones
    return dv.sumsq(g).item()
