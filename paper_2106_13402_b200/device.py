"""Device-resident operations over ``DMat`` (column-major FP64 in HBM).

Each function is a thin wrapper over one C-ABI entry point of libutvb200
(include/utv_b200.h).  The numpy-facing drop-in API (qr.py, svd.py,
powerurv.py, randutv.py) and bench.py are built on these.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import DMat, check, dempty, load, stream_ptr, workspace  # noqa: F401


def gemm(transa, transb, alpha, A: DMat, B: DMat, beta=0.0, C: DMat | None = None,
         m=None, n=None, k=None):
    lib = load()
    ta, tb = transa.upper() == "T", transb.upper() == "T"
    m = (A.cols if ta else A.rows) if m is None else m
    k = (A.rows if ta else A.cols) if k is None else k
    n = (B.rows if tb else B.cols) if n is None else n
    if C is None:
        C = dempty(m, n)
        beta = 0.0
    lw = lib.utv_dgemm_bufsize(m, n, k)
    ws = workspace(lw)
    check(lib.utv_dgemm(transa.encode(), transb.encode(), m, n, k, alpha, A.ptr, A.ld, B.ptr, B.ld,
                        beta, C.ptr, C.ld, ws.data_ptr(), lw, stream_ptr()), "utv_dgemm")
    return C


def sgemm_tf32x3(transa, transb, alpha, A: DMat, B: DMat, beta=0.0, C: DMat | None = None):
    """FP32 GEMM on the tensor cores with the 3xTF32 split (utv_sgemm_tf32x3)."""
    import torch
    ta, tb = transa.upper() == "T", transb.upper() == "T"
    m = A.cols if ta else A.rows
    k = A.rows if ta else A.cols
    n = B.rows if tb else B.cols
    if C is None:
        C = dempty(m, n, dtype=torch.float32)
        beta = 0.0
    check(load().utv_sgemm_tf32x3(transa.encode(), transb.encode(), m, n, k, alpha, A.ptr, A.ld,
                                  B.ptr, B.ld, beta, C.ptr, C.ld, stream_ptr()), "utv_sgemm_tf32x3")
    return C


def sumsq(A: DMat):
    import torch
    lib = load()
    out = _lib.dzero_vec(1, torch.float64)
    lw = lib.utv_dsumsq_bufsize()
    ws = workspace(lw)
    check(lib.utv_dsumsq(A.rows, A.cols, A.ptr, A.ld, out.data_ptr(), ws.data_ptr(), lw,
                         stream_ptr()), "utv_dsumsq")
    return out


def geqrf(A: DMat):
    """In place: A <- R. Returns (Y, T)."""
    lib = load()
    m, n = A.rows, A.cols
    Y = dempty(m, n)
    T = dempty(n, n)
    lw = lib.utv_dgeqrf_bufsize(m, n)
    ws = workspace(lw)
    check(lib.utv_dgeqrf(m, n, A.ptr, A.ld, Y.ptr, Y.ld, T.ptr, T.ld, ws.data_ptr(), lw,
                         stream_ptr()), "utv_dgeqrf")
    return Y, T


def geqp3(A: DMat):
    """Column-pivoted QR (utv_dgeqp3_f64); A is destroyed. Returns (R, Y, T, perm)."""
    import torch
    lib = load()
    m, n = A.rows, A.cols
    r = min(m, n)
    R = dempty(m, n)
    Y = dempty(m, r)
    T = dempty(r, r)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    lw = lib.utv_dgeqp3_bufsize(m, n)
    ws = workspace(lw)
    check(lib.utv_dgeqp3_f64(m, n, A.ptr, A.ld, R.ptr, R.ld, Y.ptr, Y.ld, T.ptr, T.ld,
                             perm.data_ptr(), ws.data_ptr(), lw, stream_ptr()), "utv_dgeqp3_f64")
    return R, Y, T, perm


def geqp3_max_dim():
    return int(load().utv_dgeqp3_max_dim())


def larfb(side, trans, Y: DMat, T: DMat, B: DMat):
    lib = load()
    lw = lib.utv_dlarfb_bufsize(B.rows, B.cols, Y.cols)
    ws = workspace(lw)
    check(lib.utv_dlarfb(side.encode(), b"T" if trans else b"N", B.rows, B.cols, Y.rows, Y.cols,
                         Y.ptr, Y.ld, T.ptr, T.ld, B.ptr, B.ld, ws.data_ptr(), lw, stream_ptr()),
          "utv_dlarfb")
    return B


def orgqr(Y: DMat, T: DMat, ncols):
    lib = load()
    Q = dempty(Y.rows, ncols)
    lw = lib.utv_dorgqr_bufsize(Y.rows, ncols, Y.cols)
    ws = workspace(lw)
    check(lib.utv_dorgqr(Y.rows, ncols, Y.cols, Y.ptr, Y.ld, T.ptr, T.ld, Q.ptr, Q.ld,
                         ws.data_ptr(), lw, stream_ptr()), "utv_dorgqr")
    return Q


def gesvj(A: DMat, transpose=None):
    """Returns (sigma tensor, U, V, status tensor).  transpose: None = the
    library default (rounds on A^T), False / True = on A / on A^T."""
    import torch
    lib = load()
    n = A.rows
    sig = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    U = dempty(n, n)
    V = dempty(n, n)
    status = _lib.dzero_vec(1, torch.int32)
    lw = lib.utv_dgesvj_bufsize(n)
    ws = workspace(lw)
    if transpose is None:
        check(lib.utv_dgesvj(n, A.ptr, A.ld, sig.data_ptr(), U.ptr, U.ld, V.ptr, V.ld,
                             status.data_ptr(), ws.data_ptr(), lw, stream_ptr()), "utv_dgesvj")
    else:
        check(lib.utv_dgesvj_ex(n, A.ptr, A.ld, sig.data_ptr(), U.ptr, U.ld, V.ptr, V.ld,
                                status.data_ptr(), 1 if transpose else 0, ws.data_ptr(), lw,
                                stream_ptr()), "utv_dgesvj_ex")
    return sig, U, V, status


def stage_randutv_blocks(blocks, b, dtype=None):
    """Concatenate the C-order k_i x b Gaussian draws into one b x sum(k_i)
    column-major device matrix (block i = G_i^T); ld padded (even for fp64,
    a multiple of 4 for fp32)."""
    torch_ = _lib.torch_cuda()
    dtype = torch_.float64 if dtype is None else dtype
    npdt = np.float64 if dtype == torch_.float64 else np.float32
    total = sum(int(g.shape[0]) for g in blocks)
    G = dempty(b, max(total, 1), dtype=dtype)
    col = 0
    for g in blocks:
        g = np.ascontiguousarray(g, dtype=npdt)             # C order: rows of length b
        k = g.shape[0]
        G.t[col:col + k, :b].copy_(torch_.from_numpy(g))
        col += k
    return G


class RandUtvRun:
    """Device buffers + workspace for repeated randUTV runs of one shape."""

    def __init__(self, m, n, b, q, record_trailing=False):
        import torch
        self.m, self.n, self.b, self.q = m, n, b, q
        lib = load()
        self.lw = lib.utv_randutv_basic_bufsize(m, n, b, q)
        self.ws = workspace(self.lw)
        steps = -(-n // b)
        self.steps = steps
        self.errsq = _lib.dzero_vec(steps, torch.float64)
        self.trail2 = _lib.dzero_vec(steps, torch.float64) if record_trailing else None
        self.status = _lib.dzero_vec(steps, torch.int32)

    def run(self, T: DMat, U: DMat, V: DMat, G: DMat):
        lib = load()
        check(lib.utv_randutv_basic_f64(
            self.m, self.n, self.b, self.q, T.ptr, T.ld, U.ptr, U.ld, V.ptr, V.ld, G.ptr, G.ld,
            self.errsq.data_ptr(), self.trail2.data_ptr() if self.trail2 is not None else None,
            self.status.data_ptr(), self.ws.data_ptr(), self.lw, stream_ptr()),
            "utv_randutv_basic_f64")


class RandUtvRun32:
    """fp32 randUTV (3xTF32 tcgen05 GEMMs): workspace + per-step outputs."""

    def __init__(self, m, n, b, q, record_trailing=False):
        import torch
        self.m, self.n, self.b, self.q = m, n, b, q
        lib = load()
        self.lw = lib.utv_randutv_basic_f32_bufsize(m, n, b, q)
        self.ws = workspace(self.lw)
        steps = -(-n // b)
        self.steps = steps
        self.errsq = _lib.dzero_vec(steps, torch.float64)
        self.trail2 = _lib.dzero_vec(steps, torch.float64) if record_trailing else None
        self.status = _lib.dzero_vec(steps, torch.int32)

    def run(self, T: DMat, U: DMat, V: DMat, G: DMat):
        lib = load()
        check(lib.utv_randutv_basic_f32(
            self.m, self.n, self.b, self.q, T.ptr, T.ld, U.ptr, U.ld, V.ptr, V.ld, G.ptr, G.ld,
            self.errsq.data_ptr(), self.trail2.data_ptr() if self.trail2 is not None else None,
            self.status.data_ptr(), self.ws.data_ptr(), self.lw, stream_ptr()),
            "utv_randutv_basic_f32")


class PowerUrvRun:
    """Device workspace for repeated powerURV runs of one shape."""

    def __init__(self, m, n, q):
        lib = load()
        self.m, self.n, self.q = m, n, q
        self.lw = lib.utv_powerurv_bufsize(m, n, q)
        self.ws = workspace(self.lw)
        self.Uy = dempty(m, n)
        self.Ut = dempty(n, n)
        self.R = dempty(m, n)
        self.Vy = dempty(n, n)
        self.Vt = dempty(n, n)

    @staticmethod
    def _ev(e):
        if e is None:
            return None
        e.record()                     # materialises the CUDA event; re-recorded inside
        return e.cuda_event

    def run(self, A: DMat, G: DMat, vq_event=None, r_event=None):
        """vq_event / r_event (torch.cuda.Event, optional): recorded once Vq,
        resp. R and Uq.Y, are final."""
        lib = load()
        check(lib.utv_powerurv_f64_ev(
            self.m, self.n, self.q, A.ptr, A.ld, G.ptr, G.ld, self.Uy.ptr, self.Uy.ld, self.Ut.ptr,
            self.Ut.ld, self.R.ptr, self.R.ld, self.Vy.ptr, self.Vy.ld, self.Vt.ptr, self.Vt.ld,
            self.ws.data_ptr(), self.lw, stream_ptr(), self._ev(vq_event), self._ev(r_event)),
            "utv_powerurv_f64")

    def run_cols(self, A: DMat, G: DMat | None = None, Yhat0: DMat | None = None, vq_event=None,
                 r_events=None, t_events=None, progress=None):
        """utv_powerurv_f64_cols: G, or (q >= 1) Yhat0 = A G; r_events[j] /
        t_events[j] (torch.cuda.Event lists of ceil(n/256), optional) are
        recorded once columns [256 j, 256 j + 256) of R and Uq.Y, resp. of
        Uq.Twy, are final."""
        import ctypes
        lib = load()
        ngrp = -(-self.n // 256)

        def arr(evs):
            if evs is None:
                return None
            assert len(evs) == ngrp
            return (ctypes.c_void_p * ngrp)(*[self._ev(e) for e in evs])
        ra, ta = arr(r_events), arr(t_events)
        cb = None
        if progress is not None:
            proto = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int)
            cb = proto(lambda _ctx, kind, index: progress(kind, index))
        check(lib.utv_powerurv_f64_cols(
            self.m, self.n, self.q, A.ptr, A.ld, G.ptr if G is not None else None,
            G.ld if G is not None else 2, Yhat0.ptr if Yhat0 is not None else None,
            Yhat0.ld if Yhat0 is not None else 2, self.Uy.ptr, self.Uy.ld, self.Ut.ptr, self.Ut.ld,
            self.R.ptr, self.R.ld, self.Vy.ptr, self.Vy.ld, self.Vt.ptr, self.Vt.ld,
            self.ws.data_ptr(), self.lw, stream_ptr(), self._ev(vq_event), ngrp, ra, ta,
            ctypes.cast(cb, ctypes.c_void_p) if cb is not None else None, None),
            "utv_powerurv_f64_cols")

    def run_yhat(self, A: DMat, Yhat0: DMat, vq_event=None, r_event=None):
        """q >= 1 with the first product Yhat = A G already formed (utv_powerurv_f64_yhat)."""
        lib = load()
        check(lib.utv_powerurv_f64_yhat(
            self.m, self.n, self.q, A.ptr, A.ld, Yhat0.ptr, Yhat0.ld, self.Uy.ptr, self.Uy.ld,
            self.Ut.ptr, self.Ut.ld, self.R.ptr, self.R.ld, self.Vy.ptr, self.Vy.ld, self.Vt.ptr,
            self.Vt.ld, self.ws.data_ptr(), self.lw, stream_ptr(), self._ev(vq_event),
            self._ev(r_event)), "utv_powerurv_f64_yhat")


# ---------------------------------------------------------------------------
# TSQR / Householder-reconstruction building blocks (row-sharded powerURV)
# ---------------------------------------------------------------------------

def geqrf_rows_max():
    return int(load().utv_dgeqrf_rows_max())


def lacpy(A: DMat, B: DMat):
    check(load().utv_dlacpy(A.rows, A.cols, A.ptr, A.ld, B.ptr, B.ld, stream_ptr()), "utv_dlacpy")
    return B


def copy(A: DMat):
    return lacpy(A, dempty(A.rows, A.cols))


def laset(uplo, alpha, beta, A: DMat):
    check(load().utv_dlaset(uplo.encode(), A.rows, A.cols, alpha, beta, A.ptr, A.ld, stream_ptr()),
          "utv_dlaset")
    return A


def transpose(A: DMat, B: DMat | None = None):
    """B = A^T on the device."""
    if B is None:
        B = dempty(A.cols, A.rows)
    check(load().utv_dtranspose(A.rows, A.cols, A.ptr, A.ld, B.ptr, B.ld, stream_ptr()),
          "utv_dtranspose")
    return B


def from_numpy_any_order(a):
    """Device copy of a 2-D float64 array without a host-side layout copy:
    F-order arrays go up as is; C-order arrays go up as their transpose
    (the same bytes) and are transposed on the device."""
    from ._lib import dfrom_numpy
    a = np.asarray(a, dtype=np.float64)
    if a.flags["F_CONTIGUOUS"] or not a.flags["C_CONTIGUOUS"]:
        return dfrom_numpy(a)
    return transpose(dfrom_numpy(a.T))


def tri_zero(uplo, A: DMat):
    """Zero the strictly upper ('U') or strictly lower ('L') part; diagonal kept."""
    check(load().utv_dtri_zero(uplo.encode(), A.rows, A.cols, A.ptr, A.ld, stream_ptr()),
          "utv_dtri_zero")
    return A


def diag_scale(side, d, A: DMat, alpha=1.0):
    """A <- alpha diag(d) A (side 'L') or alpha A diag(d) (side 'R'); d a device tensor."""
    check(load().utv_ddiag_scale(side.encode(), A.rows, A.cols, d.data_ptr(), alpha, A.ptr, A.ld,
                                 stream_ptr()), "utv_ddiag_scale")
    return A


def getrf_signed(A: DMat):
    """In place LU without pivoting of (A - diag(s)); returns s (device tensor)."""
    import torch
    lib = load()
    s = torch.empty(max(A.cols, 1), dtype=torch.float64, device="cuda")
    lw = lib.utv_dgetrf_signed_bufsize(A.rows, A.cols)
    ws = workspace(lw)
    check(lib.utv_dgetrf_signed(A.rows, A.cols, A.ptr, A.ld, s.data_ptr(), ws.data_ptr(), lw,
                                stream_ptr()), "utv_dgetrf_signed")
    return s


def trsm_right(uplo, trans, diag, A: DMat, B: DMat):
    """B <- B op(A)^{-1}, op(A) upper triangular."""
    lib = load()
    lw = lib.utv_dtrsm_bufsize(B.rows, B.cols)
    ws = workspace(lw)
    check(lib.utv_dtrsm_right(uplo.encode(), trans.encode(), diag.encode(), B.rows, B.cols, A.ptr,
                              A.ld, B.ptr, B.ld, ws.data_ptr(), lw, stream_ptr()), "utv_dtrsm_right")
    return B
