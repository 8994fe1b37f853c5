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
