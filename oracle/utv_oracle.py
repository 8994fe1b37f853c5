"""CPU oracle for the powerURV / randUTV hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``utvkit``
(arXiv 2106.13402 reference, ``/root/reference/pkg/src/utvkit``) for the
functions on the B200 hot path.  It exists to check the CUDA path; it is
never imported by the product package ``paper_2106_13402_b200`` (only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg).

Pinning: every function here is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py``, fixtures in
``tests/golden/*.npz``) in ``tests/test_oracle_golden.py``.

Conventions restated (each cites the reference line it follows):

* Householder reflector: beta = -sign(alpha)*||x||, sign(0) = +1, v[0] = 1,
  tau = 2 / (1 + sigma / v1^2); skip (tau = 0, identity reflector) when
  ||x|| <= eps*||A||_F or sigma == 0  (qr.py:43-60, qr.py:86-93).
* Compact-WY triangle grown forward column by column (qr.py:63-68).
* apply_q: left  B - Y (T^(T) (Y^T B)); right  B - ((B Y) T^(T)) Y^T
  (qr.py:103-121).
* svd_dense sign rule: flip each pair so the first largest-|.| entry of
  every V column is positive (svd.py:53-57).
* randUTV basic step loop (randutv.py:110-193) with the unstabilised
  sampler (randutv.py:185-193) and the ErrorTracker arithmetic
  (randutv.py:31-62).
"""

from __future__ import annotations

import math

import numpy as np

EPS = float(np.finfo(np.float64).eps)  # matrix.py:13


class OracleError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# Householder QR in compact-WY form
# ---------------------------------------------------------------------------

def householder_qr(a):
    """Unblocked Householder QR of an m x n (m >= n) matrix.

    Follows qr.py:71-100.  Returns (Y m x n, Twy n x n, R m x n).
    """
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m < n:
        raise ValueError("householder_qr needs m >= n")
    work = np.array(a, dtype=np.float64, order="F", copy=True)
    vecs = np.zeros((m, n), order="F")
    tri = np.zeros((n, n), order="F")
    cutoff = EPS * float(np.linalg.norm(a))          # qr.py:86
    for j in range(n):
        col = work[j:, j].copy()
        head = float(col[0])
        tail_sq = float(col[1:] @ col[1:])           # qr.py:50
        nrm = math.sqrt(head * head + tail_sq)       # qr.py:52
        if nrm <= cutoff or tail_sq == 0.0:          # qr.py:53-54 skip rule
            vecs[j, j] = 1.0                         # qr.py:90
            tri[j, j] = 0.0                          # qr.py:91 (tau = 0)
            work[j + 1:, j] = 0.0                    # qr.py:92
            continue
        sgn = 1.0 if head >= 0.0 else -1.0           # qr.py:55
        pivot = head + sgn * nrm                     # qr.py:56
        v = col / pivot                              # qr.py:57
        v[0] = 1.0                                   # qr.py:58
        tau = 2.0 / (1.0 + tail_sq / (pivot * pivot))  # qr.py:59
        # rank-1 update of the trailing block, qr.py:94-95
        w = tau * (v @ work[j:, j:])
        work[j:, j:] -= np.outer(v, w)
        work[j, j] = -sgn * nrm                      # qr.py:96 (beta)
        work[j + 1:, j] = 0.0                        # qr.py:97
        vecs[j:, j] = v                              # qr.py:98
        # forward accumulation of the WY triangle, qr.py:63-68
        tri[j, j] = tau
        if j > 0:
            z = vecs[j:, :j].T @ v
            tri[:j, j] = -tau * (tri[:j, :j] @ z)
    return vecs, tri, work


def wy_apply(y, twy, b, side="left", trans=False):
    """Apply Q = I - Y Twy Y^T (or Q^T) without forming it; qr.py:103-121."""
    b = np.asarray(b, dtype=np.float64)
    t = twy.T if trans else twy
    if side == "left":
        return b - y @ (t @ (y.T @ b))
    if side == "right":
        return b - ((b @ y) @ t) @ y.T
    raise ValueError(side)


def wy_materialize(y, twy, ncols=None):
    """Leading ncols columns of Q; qr.py:124-131."""
    m = y.shape[0]
    c = m if ncols is None else int(ncols)
    out = np.zeros((m, c), order="F")
    out[np.arange(c), np.arange(c)] = 1.0
    return out - y @ (twy @ y[:c, :].T)


# ---------------------------------------------------------------------------
# Dense SVD with the reference sign rule
# ---------------------------------------------------------------------------

def svd_signed(a, full=True):
    """LAPACK SVD + sign normalisation of svd.py:37-58 -> (U, sigma, V)."""
    a = np.asarray(a, dtype=np.float64)
    u, s, vh = np.linalg.svd(a, full_matrices=full)
    v = np.array(vh.T, order="F")
    u = np.array(u, order="F")
    for j in range(s.shape[0]):
        i = int(np.argmax(np.abs(v[:, j])))
        if v[i, j] < 0.0:
            v[:, j] *= -1.0
            u[:, j] *= -1.0
    return u, s, v


# ---------------------------------------------------------------------------
# Random streams (matrix.py:16-60)
# ---------------------------------------------------------------------------

def gaussian_stream(seed):
    return np.random.Generator(np.random.PCG64(int(seed)))


def draw_gaussian(gen, m, n):
    """C-order draw then Fortran copy, as gaussian() does (matrix.py:52-60)."""
    return np.asfortranarray(gen.standard_normal((int(m), int(n))))


def randutv_sample_blocks(gen, m, n, b):
    """All Gaussian blocks randutv_basic draws, in draw order.

    One (m - lo) x b block per regular step (randutv.py:189), none for the
    final dense-SVD branch (randutv.py:164-177).
    """
    steps = max(0, -(-n // b) - 1)
    return [draw_gaussian(gen, m - i * b, b) for i in range(steps)]


# ---------------------------------------------------------------------------
# powerURV (powerurv.py:41-84)
# ---------------------------------------------------------------------------

def power_urv(a, q, g):
    """Algorithm 1 with a caller-supplied G; powerurv.py:41-72.

    Returns dict(Uy, Ut, R, Vy, Vt).
    """
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if q == 0:
        vy, vt, _ = householder_qr(g)
    else:
        v = g
        for _ in range(q):
            yhat = a @ v                                   # powerurv.py:64
            qy, qt, _ = householder_qr(yhat)               # powerurv.py:65
            vhat = wy_materialize(qy, qt, n)
            y = a.T @ vhat                                 # powerurv.py:66
            vy, vt, _ = householder_qr(y)                  # powerurv.py:67
            v = wy_materialize(vy, vt)                     # powerurv.py:68
    ahat = wy_apply(vy, vt, a, side="right")               # powerurv.py:70
    uy, ut, r = householder_qr(ahat)                       # powerurv.py:71
    return dict(Uy=uy, Ut=ut, R=r, Vy=vy, Vt=vt)


# ---------------------------------------------------------------------------
# randomized SVD cross-check (rsvd.py:31-78; SPEC acceptance 2)
# ---------------------------------------------------------------------------

def rsvd(a, g_shared, ell, q):
    """Rank-ell randomized SVD from the first ell columns of G: thin QR between
    every application of A and A^T (rsvd.py:56-63), then the small SVD of
    Q^T A lifted back (rsvd.py:65-67).  Returns (U_rsvd, sigma, V)."""
    a = np.asarray(a, dtype=np.float64)

    def thin_q(x):                                   # hqr_thin (qr.py:134-138)
        y, t, _ = householder_qr(x)
        return wy_materialize(y, t, x.shape[1])

    basis = thin_q(a @ g_shared[:, :ell])
    for _ in range(q):
        basis = thin_q(a @ thin_q(a.T @ basis))
    u_s, s, v = svd_signed(basis.T @ a, full=False)
    return basis @ u_s, s, v


def projector_gap(u1, u2, a):
    """||u1 u1^T a - u2 u2^T a||_F / ||a||_F (rsvd.py:81-98)."""
    d = u1 @ (u1.T @ a) - u2 @ (u2.T @ a)
    return float(np.linalg.norm(d) / np.linalg.norm(a))


# ---------------------------------------------------------------------------
# randUTV basic (randutv.py:110-193, 228-235)
# ---------------------------------------------------------------------------

def randutv_basic(a, b, q, g_blocks, record_trailing=False):
    """Blocked randUTV with pre-drawn Gaussian blocks.

    ``g_blocks[i]`` is the block the reference draws at regular step i+1.
    Returns dict(U, T, V, errors, trailing, steps).
    """
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    t = np.array(a, order="F", copy=True)
    u = np.eye(m, order="F")
    v = np.eye(n, order="F")
    e0 = float(np.linalg.norm(a))
    e_sq = e0 * e0
    e0_sq = e_sq
    errors = []
    trailing = [] if record_trailing else None
    nsteps = -(-n // b)
    steps = 0

    def track(panel):
        nonlocal e_sq
        e_sq -= float(np.sum(panel * panel))               # randutv.py:54
        if e_sq < -1e-10 * e0_sq:                          # randutv.py:55-58
            raise OracleError("tracked squared error went negative")
        if e_sq < 0.0:
            e_sq = 0.0
        errors.append(math.sqrt(e_sq))

    for i in range(nsteps):
        lo = i * b
        mid = lo + b
        ncols = n - lo
        if ncols > b:
            blk = t[lo:, lo:]
            y = blk.T @ g_blocks[i]                        # randutv.py:190
            for _ in range(q):
                y = blk.T @ (blk @ y)                      # randutv.py:191-192
            vy, vt, _ = householder_qr(y)                  # randutv.py:141
            t[:, lo:] = wy_apply(vy, vt, t[:, lo:], "right")
            v[:, lo:] = wy_apply(vy, vt, v[:, lo:], "right")
            uy, ut, rp = householder_qr(t[lo:, lo:mid])    # randutv.py:146
            u[:, lo:] = wy_apply(uy, ut, u[:, lo:], "right")
            t[lo:, mid:] = wy_apply(uy, ut, t[lo:, mid:], "left", trans=True)
            t[mid:, lo:mid] = 0.0                          # randutv.py:149
            su, ss, sv = svd_signed(rp[:b, :])             # randutv.py:151
            u[:, lo:mid] = u[:, lo:mid] @ su
            v[:, lo:mid] = v[:, lo:mid] @ sv
            t[lo:mid, lo:mid] = np.diag(ss)
            t[lo:mid, mid:] = su.T @ t[lo:mid, mid:]
            t[:lo, lo:mid] = t[:lo, lo:mid] @ sv
            steps = i + 1
            track(t[lo:mid, lo:])
            if trailing is not None:
                trailing.append(float(np.linalg.norm(t[mid:, mid:])))
        else:
            su, ss, sv = svd_signed(t[lo:, lo:])           # randutv.py:166
            u[:, lo:] = u[:, lo:] @ su
            v[:, lo:] = v[:, lo:] @ sv
            d = np.zeros((m - lo, ncols), order="F")
            d[np.arange(ss.shape[0]), np.arange(ss.shape[0])] = ss
            t[lo:, lo:] = d
            t[:lo, lo:] = t[:lo, lo:] @ sv
            steps = i + 1
            track(t[lo:, lo:])
            if trailing is not None:
                trailing.append(0.0)
            break
    return dict(U=u, T=t, V=v, errors=errors, trailing=trailing, steps=steps)


def randutv_boosted(a, b, q, p, gen, tol_fro=None, max_rank=None, record_trailing=False):
    """Boosted / partial randUTV (Algorithm 2; randutv.py:110-182 with
    boosted=True, _sample_boosted :196-225, svd_tall_thin_left svd.py:61-82).

    ``gen`` is the numpy Generator of the reference's RngStream; draws are
    made lazily in the reference's order (step 1: m x (b+p), later
    (m-lo) x b) so an early stop leaves the generator where the reference
    would.  Returns dict(U, T, V, errors, trailing, steps).
    """
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    t = np.array(a, order="F", copy=True)
    u = np.eye(m, order="F")
    v = np.eye(n, order="F")
    e0 = float(np.linalg.norm(a))
    e_sq, e0_sq = e0 * e0, e0 * e0
    errors, trailing = [], ([] if record_trailing else None)
    w_next, steps = None, 0

    def track(panel):
        nonlocal e_sq
        e_sq -= float(np.sum(panel * panel))
        if e_sq < -1e-10 * e0_sq:
            raise OracleError("tracked squared error went negative")
        e_sq = max(e_sq, 0.0)
        errors.append(math.sqrt(e_sq))

    for i in range(1, -(-n // b) + 1):
        if tol_fro is not None and math.sqrt(e_sq) <= tol_fro:          # randutv.py:123-124
            break
        lo, mid = (i - 1) * b, (i - 1) * b + b
        nrows, ncols = m - lo, n - lo
        if ncols > b + p:
            blk = t[lo:, lo:]
            if i == 1:                                                 # randutv.py:205-210
                y = blk.T @ draw_gaussian(gen, m, b + p)
                for _ in range(q):
                    y = blk.T @ (blk @ y)
            else:                                                      # randutv.py:211-225
                y = blk.T @ draw_gaussian(gen, nrows, b)
                for _ in range(q - 1):
                    y = blk.T @ (blk @ y)
                x = blk @ y
                if w_next is not None:
                    pad = x.shape[0] - w_next.shape[0]
                    w = np.vstack([w_next, np.zeros((pad, w_next.shape[1]))]) if pad else w_next
                    x = x - w @ (w.T @ x)
                else:
                    w = np.zeros((x.shape[0], 0))
                qy, qt, _ = householder_qr(x)
                y = blk.T @ np.hstack([wy_materialize(qy, qt, b), w])
            # svd_tall_thin_left(y) (svd.py:61-82): W = Q blockdiag(Uhat, I)
            yy, yt, yr = householder_qr(y)
            wc = y.shape[1]
            uhat, _, _ = svd_signed(yr[:wc, :])
            c = np.zeros((ncols, ncols), order="F")
            c[:wc, :wc] = uhat
            if ncols > wc:
                c[wc:, wc:] = np.eye(ncols - wc)
            w_y = wy_apply(yy, yt, c, "left")
            vy, vt, _ = householder_qr(w_y[:, :b])                     # randutv.py:134
            if p > 0 and (ncols - b) > b + p:                          # randutv.py:135-138
                w_next = wy_apply(vy, vt, w_y[:, b:b + p], "left", trans=True)[b:, :]
            else:
                w_next = None
            t[:, lo:] = wy_apply(vy, vt, t[:, lo:], "right")
            v[:, lo:] = wy_apply(vy, vt, v[:, lo:], "right")
            uy, ut, rp = householder_qr(t[lo:, lo:mid])
            u[:, lo:] = wy_apply(uy, ut, u[:, lo:], "right")
            t[lo:, mid:] = wy_apply(uy, ut, t[lo:, mid:], "left", trans=True)
            t[mid:, lo:mid] = 0.0
            su, ss, sv = svd_signed(rp[:b, :])
            u[:, lo:mid] = u[:, lo:mid] @ su
            v[:, lo:mid] = v[:, lo:mid] @ sv
            t[lo:mid, lo:mid] = np.diag(ss)
            t[lo:mid, mid:] = su.T @ t[lo:mid, mid:]
            t[:lo, lo:mid] = t[:lo, lo:mid] @ sv
            steps = i
            track(t[lo:mid, lo:])
            if trailing is not None:
                trailing.append(float(np.linalg.norm(t[mid:, mid:])))
            if max_rank is not None and i * b >= max_rank:
                break
        else:
            su, ss, sv = svd_signed(t[lo:, lo:])
            u[:, lo:] = u[:, lo:] @ su
            v[:, lo:] = v[:, lo:] @ sv
            d = np.zeros((nrows, ncols), order="F")
            d[np.arange(ss.shape[0]), np.arange(ss.shape[0])] = ss
            t[lo:, lo:] = d
            t[:lo, lo:] = t[:lo, lo:] @ sv
            steps = i
            track(t[lo:, lo:])
            if trailing is not None:
                trailing.append(0.0)
            break
    return dict(U=u, T=t, V=v, errors=errors, trailing=trailing, steps=steps)


# ---------------------------------------------------------------------------
# Column-pivoted QR comparator (qr.py:140-204)
# ---------------------------------------------------------------------------

PIVOT_TIE_RTOL = 1e-12   # qr.py:148
DOWNDATE_RTOL = EPS      # qr.py:143


def hqrcp(a):
    """Businger-Golub column-pivoted Householder QR, restating qr.py:152-204.

    Returns (Y m x r, Twy r x r, R m x n in pivoted order, perm), r = min(m, n):
    greedy largest squared-norm pivot; ties within a 1e-12 relative window go
    to the leftmost logical column (qr.py:171-175); reflector + skip rule as in
    householder_qr (qr.py:43-60, 182-194); squared-norm downdate clamped at 0
    with an exact recompute once the estimate is <= eps * its last exact value
    (qr.py:196-202).
    """
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    r = min(m, n)
    work = np.array(a, order="F", copy=True)
    vecs = np.zeros((m, r), order="F")
    tri = np.zeros((r, r), order="F")
    perm = np.arange(n)
    cutoff = EPS * float(np.linalg.norm(a))                  # qr.py:162
    est = np.sum(work * work, axis=0)                        # qr.py:164
    exact = est.copy()                                       # qr.py:165
    for j in range(r):
        rest = est[j:]
        big = float(rest.max())
        k = j + int(np.argmax(rest >= big * (1.0 - PIVOT_TIE_RTOL))) if big > 0.0 else j
        if k != j:                                           # qr.py:176-180
            work[:, [j, k]] = work[:, [k, j]]
            perm[[j, k]] = perm[[k, j]]
            est[[j, k]] = est[[k, j]]
            exact[[j, k]] = exact[[k, j]]
        col = work[j:, j].copy()
        head = float(col[0])
        tail_sq = float(col[1:] @ col[1:])
        nrm = math.sqrt(head * head + tail_sq)
        if nrm <= cutoff or tail_sq == 0.0:                  # skip, qr.py:183-186
            vecs[j, j] = 1.0
            work[j + 1:, j] = 0.0
        else:
            sgn = 1.0 if head >= 0.0 else -1.0
            pivot = head + sgn * nrm
            v = col / pivot
            v[0] = 1.0
            tau = 2.0 / (1.0 + tail_sq / (pivot * pivot))
            w = tau * (v @ work[j:, j:])                     # qr.py:188-189
            work[j:, j:] -= np.outer(v, w)
            work[j, j] = -sgn * nrm
            work[j + 1:, j] = 0.0
            vecs[j:, j] = v
            tri[j, j] = tau                                  # qr.py:63-68
            if j > 0:
                z = vecs[j:, :j].T @ v
                tri[:j, j] = -tau * (tri[:j, :j] @ z)
        if j + 1 < n:                                        # qr.py:196-202
            est[j + 1:] -= work[j, j + 1:] ** 2
            np.maximum(est[j + 1:], 0.0, out=est[j + 1:])
            for c in j + 1 + np.nonzero(est[j + 1:] <= DOWNDATE_RTOL * exact[j + 1:])[0]:
                est[c] = float(work[j + 1:, c] @ work[j + 1:, c])
                exact[c] = est[c]
    return vecs, tri, work, perm


# ---------------------------------------------------------------------------
# Parity metrics (bench.py:63-72)
# ---------------------------------------------------------------------------

def trailing_fro(t):
    """||T[k:, k:]||_F for k = 1..n-1 by a 2-D suffix sum (bench.py:63-72)."""
    t = np.asarray(t, dtype=np.float64)
    m, n = t.shape
    sq = t * t
    suf = np.cumsum(np.cumsum(sq[::-1, ::-1], axis=0), axis=1)[::-1, ::-1]
    vals = np.array([suf[k, k] if k < m else 0.0 for k in range(1, n)])
    return np.sqrt(np.maximum(vals, 0.0))


def reconstruction(a, u, t, v):
    return float(np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a))


def orthogonality(q):
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


# ---------------------------------------------------------------------------
# Test-matrix helpers (matgen.py:17-37 restated with LAPACK QR for speed)
# ---------------------------------------------------------------------------

def random_orthogonal_fast(n, gen):
    """Haar-like orthogonal factor via LAPACK QR of a Gaussian (sign-fixed)."""
    g = gen.standard_normal((n, n))
    qm, rm = np.linalg.qr(g)
    return np.asfortranarray(qm * np.sign(np.diag(rm))[None, :])


def decay_matrix(n, beta, seed, m=None):
    """A = Q1 diag(d) Q2^T with d_i = beta^((i-1)/(n-1)) (matgen.py:30-37)."""
    gen = gaussian_stream(seed)
    m = n if m is None else m
    d = beta ** (np.arange(n) / max(n - 1, 1))
    if m == n:
        q1 = random_orthogonal_fast(m, gen)
    else:                                   # thin factor: never form an m x m matrix
        g = gen.standard_normal((m, n))
        qm, rm = np.linalg.qr(g)
        q1 = qm * np.sign(np.diag(rm))[None, :]
    q2 = random_orthogonal_fast(n, gen)
    return np.asfortranarray(q1 @ (d[:, None] * q2.T)), d
