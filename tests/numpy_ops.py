"""Host-side (numpy) implementation of the sharded-powerURV building blocks —
TEST INFRASTRUCTURE ONLY.  It lets the multi-rank orchestration of
paper_2106_13402_b200/sharded.py (TSQR tree, collectives, Householder
reconstruction) run under torch.distributed/gloo on CPU, with the oracle's
Householder QR (oracle/utv_oracle.py, pinned to the reference) as the local
factorisation.  The product path never uses it."""
import numpy as np
import torch

from oracle import utv_oracle as orc


class NumpyOps:
    def rows_max(self):
        return 1 << 30

    def empty(self, rows, cols):
        return np.zeros((rows, cols), order="F")

    zeros = empty

    def eye(self, n):
        return np.asfortranarray(np.eye(n))

    def sub(self, m, r0, c0, nr, nc):
        return m[r0:r0 + nr, c0:c0 + nc]

    def shape(self, m):
        return m.shape

    def copy(self, m):
        return np.array(m, order="F", copy=True)

    def lacpy(self, a, b):
        b[...] = a
        return b

    def gemm(self, ta, tb, alpha, a, b, beta=0.0, c=None):
        r = alpha * ((a.T if ta == "T" else a) @ (b.T if tb == "T" else b))
        if c is None:
            return np.asfortranarray(r)
        c[...] = r if beta == 0.0 else r + beta * c
        return c

    def geqrf(self, a):
        y, t, r = orc.householder_qr(a)
        a[...] = r
        return y, t

    def larfb(self, side, trans, y, t, b):
        b[...] = orc.wy_apply(y, t, b, side="left" if side == "L" else "right", trans=trans)
        return b

    def orgqr(self, y, t, ncols):
        return orc.wy_materialize(y, t, ncols)

    def getrf_signed(self, a):
        m, n = a.shape
        s = np.zeros(n)
        for k in range(n):
            s[k] = -1.0 if a[k, k] >= 0.0 else 1.0
            a[k, k] -= s[k]
            a[k + 1:, k] /= a[k, k]
            a[k + 1:, k + 1:] -= np.outer(a[k + 1:, k], a[k, k + 1:])
        return torch.from_numpy(s)

    def trsm_right(self, uplo, trans, diag, a, b):
        n = a.shape[0]
        mat = np.triu(a) if uplo == "U" else np.tril(a).T
        if diag == "U":
            mat = mat - np.diag(np.diag(mat)) + np.eye(n)
        b[...] = np.linalg.solve(mat.T, b.T).T
        return b

    def laset(self, uplo, alpha, beta, a):
        n = min(a.shape)
        if uplo == "A":
            a[...] = alpha
        elif uplo == "U":
            a[np.triu_indices(a.shape[0], 1, a.shape[1])] = alpha
        else:
            a[np.tril_indices(a.shape[0], -1, a.shape[1])] = alpha
        a[np.arange(n), np.arange(n)] = beta
        return a

    def tri_zero(self, uplo, a):
        if uplo == "U":
            a[np.triu_indices(a.shape[0], 1, a.shape[1])] = 0.0
        else:
            a[np.tril_indices(a.shape[0], -1, a.shape[1])] = 0.0
        return a

    def diag_scale(self, side, d, a, alpha=1.0):
        d = d.numpy() if hasattr(d, "numpy") else np.asarray(d)
        if side == "L":
            a *= alpha * d[:, None]
        else:
            a *= alpha * d[None, :]
        return a

    def to_comm(self, m):
        return torch.from_numpy(np.ascontiguousarray(m.T))      # (cols, rows)

    def from_comm(self, t, rows, cols):
        return t.numpy().T[:rows, :cols]
