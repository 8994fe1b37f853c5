"""Blocked randUTV, basic variant — drop-in for utvkit randutv.py
(ErrorTracker 31-62, error_update 65-67, UtvFactorization 70-93,
randutv_basic 228-235 -> _randutv 110-182 / _sample_basic 185-193).

The step loop runs as one device call (libutvb200 utv_randutv_basic_f64).
The Gaussian blocks are drawn on the host from the caller's RngStream in the
reference's order (one (m-lo) x b block per regular step, randutv.py:189) so
G — and therefore U, T, V — match the reference for the same seed.
The per-step panel masses come back from the device and are folded through
the reference's ErrorTracker arithmetic on the host.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import serialized as _serialized
from . import device as dv
from ._lib import deye, dfrom_numpy
from .errors import ConsistencyError, ConvergenceError, DimensionError
from .matrix import raise_if_nonfinite, check_matrix, frobenius_norm
from .svd import JACOBI_MAX_N


@dataclass
class ErrorTracker:
    """Running Frobenius error of the unprocessed trailing block (randutv.py:31-62)."""

    e_sq: float
    e0_sq: float
    history: list = field(default_factory=list)
    # randutv.py:55-58 raises below -1e-10 e0^2 (fp64); the fp32 variant's
    # panel masses carry fp32 rounding, so it uses a fp32-scaled threshold
    neg_tol: float = 1e-10

    @classmethod
    def start(cls, a_fro):
        return cls(e_sq=a_fro * a_fro, e0_sq=a_fro * a_fro)

    @property
    def e(self):
        return math.sqrt(self.e_sq)

    def update_mass(self, mass_sq):
        self.e_sq -= float(mass_sq)
        if self.e_sq < -self.neg_tol * self.e0_sq:
            raise ConsistencyError(f"tracked squared error went negative: {self.e_sq:.3e}")
        if self.e_sq < 0.0:
            self.e_sq = 0.0
        self.history.append(self.e)
        return self

    def update(self, panel):
        panel = np.asarray(panel, dtype=np.float64)
        return self.update_mass(float(np.sum(panel * panel)))


def error_update(tracker, t_panel):
    """Subtract one processed panel's squared mass from the tracker (randutv.py:65-67)."""
    return tracker.update(t_panel)


@dataclass(frozen=True)
class UtvFactorization:
    """A = U @ T @ V.T, orthogonal U, V, upper trapezoidal T (randutv.py:70-93)."""

    U: np.ndarray
    T: np.ndarray
    V: np.ndarray
    b: int
    steps_done: int
    oversample: int
    power: int
    errors: list
    trailing_fro: list | None = None

    @property
    def processed_columns(self):
        return min(self.steps_done * self.b, self.T.shape[1])


def _validate(a, b, q, p, finite=True):
    a = check_matrix(a, finite=finite)
    m, n = a.shape
    if m < n:
        raise DimensionError(f"randutv needs m >= n, got {a.shape}; factor the transpose")
    if b < 1:
        raise ValueError(f"block size must be >= 1, got {b}")
    if q < 0:
        raise ValueError(f"power iteration count must be >= 0, got {q}")
    if p < 0:
        raise ValueError(f"oversampling must be >= 0, got {p}")
    # the b x b (and final <= (b+p)-wide) SVDs run in the Jacobi kernel (K6);
    # checked before any draw so the caller's rng is untouched on failure
    if min(int(b) + int(p), n) > JACOBI_MAX_N:
        raise ValueError(f"b + p must be <= {JACOBI_MAX_N} on the B200 path, got {int(b) + int(p)}")
    return a


def draw_sample_blocks(rng, m, n, b):
    """All Gaussian blocks randutv_basic consumes, in the reference's draw order."""
    steps = max(0, -(-n // b) - 1)
    return [np.asarray(rng.standard_normal(int(m - i * b), int(b))) for i in range(steps)]


def randutv_basic_device(t_dev, b, q, g_dev, record_trailing=False):
    """Device-resident randUTV: t_dev (m x n) is overwritten with T.

    Returns (run, U, V) with run.errsq / run.trail2 / run.status on the device."""
    m, n = t_dev.rows, t_dev.cols
    run = dv.RandUtvRun(m, n, b, q, record_trailing)
    U = deye(m)
    V = deye(n)
    run.run(t_dev, U, V, g_dev)
    return run, U, V


def _eye32(n):
    import torch
    from ._lib import check, dempty, load, stream_ptr
    m = dempty(n, n, dtype=torch.float32)
    check(load().utv_slaset(b"A", n, n, 0.0, 1.0, m.ptr, m.ld, stream_ptr()), "utv_slaset")
    return m


def randutv_basic_device32(t_dev, b, q, g_dev, record_trailing=False):
    """fp32 device-resident randUTV (BASELINE C5 variant): t_dev (fp32) is
    overwritten with T; every GEMM is 3xTF32 on the tensor cores."""
    m, n = t_dev.rows, t_dev.cols
    run = dv.RandUtvRun32(m, n, b, q, record_trailing)
    U = _eye32(m)
    V = _eye32(n)
    run.run(t_dev, U, V, g_dev)
    return run, U, V


@_serialized
def randutv_basic(a, b, q, rng, record_trailing=False, *, dtype=np.float64):
    """Blocked randomized UTV without oversampling (randutv.py:228-235).

    dtype=np.float32 selects the fp32 variant (BASELINE C5): T, U, V are
    computed in fp32 with 3xTF32 tensor-core GEMMs and returned as float32;
    m, n and b must then be multiples of 4.  The default float64 path is the
    reference-exact drop-in."""
    import torch
    f32 = np.dtype(dtype) == np.float32
    a = _validate(a, b, q, 0, finite=f32)   # fp64: the finite scan runs on the device copy
    m, n = a.shape
    b = int(b)
    q = int(q)
    if f32 and (m % 4 or n % 4 or b % 4):
        raise ValueError("the fp32 variant needs m, n and b to be multiples of 4")
    if not f32:
        return _randutv_basic_pipelined(a, b, q, rng, record_trailing)
    blocks = draw_sample_blocks(rng, m, n, b)
    if f32:
        t_dev = dfrom_numpy(a, dtype=torch.float32)
        g_dev = dv.stage_randutv_blocks(blocks, b, dtype=torch.float32)
        run, U, V = randutv_basic_device32(t_dev, b, q, g_dev, record_trailing)
    else:
        t_dev = dfrom_numpy(a)
        g_dev = dv.stage_randutv_blocks(blocks, b)
        run, U, V = randutv_basic_device(t_dev, b, q, g_dev, record_trailing)
    return _finish_basic(a, b, q, run, t_dev, U, V, record_trailing, f32)


def _finish_basic(a, b, q, run, t_dev, U, V, record_trailing, f32, host=None, anorm=None):
    status = run.status.cpu().numpy()
    if (status < 0).any():
        raise ConvergenceError("b x b Jacobi SVD failed to converge")
    masses = run.errsq.cpu().numpy()
    tracker = ErrorTracker.start(frobenius_norm(a) if anorm is None else anorm)
    if f32:
        tracker.neg_tol = 1e-5
    for mass in masses:
        tracker.update_mass(mass)
    trailing = None
    if record_trailing:
        trailing = [float(math.sqrt(max(x, 0.0))) for x in run.trail2.cpu().numpy()]
        trailing[-1] = 0.0
    if host is not None:
        u_h, t_h, v_h = host
    else:
        u_h, t_h, v_h = U.to_numpy(), t_dev.to_numpy(), V.to_numpy()
    return UtvFactorization(
        U=np.asfortranarray(u_h), T=np.asfortranarray(t_h),
        V=np.asfortranarray(v_h), b=b, steps_done=run.steps, oversample=0, power=q,
        errors=list(tracker.history), trailing_fro=trailing)


def _randutv_stepwise(a, b, q, p, rng, boosted, tol_fro=None, max_rank=None,
                      record_trailing=False):
    """Host step loop over utv_randutv_step_f64 (randutv.py:110-182): the
    Gaussian block of each step is drawn right before the step, so the
    caller's rng advances exactly as in the reference even when the run stops
    early (tol_fro / max_rank, randutv.py:123-124,162-163)."""
    import ctypes

    import torch

    from . import _lib
    a = _validate(a, b, q, p)
    m, n = a.shape
    b, q, p = int(b), int(q), int(p)
    lib = _lib.load()
    pe = p if boosted else 0
    t_dev = dfrom_numpy(a)
    U, V = deye(m), deye(n)
    steps_max = -(-n // b)
    errsq = _lib.dzero_vec(steps_max, torch.float64)
    trail2 = _lib.dzero_vec(steps_max, torch.float64) if record_trailing else None
    status = _lib.dzero_vec(steps_max, torch.int32)
    lw = lib.utv_randutv_step_bufsize(m, n, b, pe, q)
    ws = _lib.workspace(lw)
    carried, is_final = ctypes.c_int(0), ctypes.c_int(0)
    tracker = ErrorTracker.start(frobenius_norm(a))
    trailing = [] if record_trailing else None
    steps = 0
    for i in range(1, steps_max + 1):
        if tol_fro is not None and tracker.e <= tol_fro:
            break
        lo = (i - 1) * b
        ncols = n - lo
        g_dev = None
        if ncols > b + pe:
            rows, cols = (m, b + pe) if (boosted and i == 1) else (m - lo, b)
            g_dev = dv.stage_randutv_blocks([np.asarray(rng.standard_normal(rows, cols))], cols)
        check = _lib.check
        check(lib.utv_randutv_step_f64(
            i - 1, m, n, b, pe, q, 1 if boosted else 0, t_dev.ptr, t_dev.ld, U.ptr, U.ld, V.ptr, V.ld,
            g_dev.ptr if g_dev is not None else None, g_dev.ld if g_dev is not None else 2,
            errsq.data_ptr(), trail2.data_ptr() if trail2 is not None else None, status.data_ptr(),
            ctypes.byref(carried), ctypes.byref(is_final), ws.data_ptr(), lw, _lib.stream_ptr()),
            "utv_randutv_step_f64")
        steps = i
        if int(status[i - 1].item()) < 0:
            raise ConvergenceError("b x b Jacobi SVD failed to converge")
        tracker.update_mass(float(errsq[i - 1].item()))
        if trailing is not None:
            trailing.append(0.0 if is_final.value else float(math.sqrt(max(float(trail2[i - 1].item()), 0.0))))
        if is_final.value:
            break
        if max_rank is not None and i * b >= max_rank:
            break
    return UtvFactorization(
        U=np.asfortranarray(U.to_numpy()), T=np.asfortranarray(t_dev.to_numpy()),
        V=np.asfortranarray(V.to_numpy()), b=b, steps_done=steps, oversample=p, power=q,
        errors=list(tracker.history), trailing_fro=trailing)


_GRING = {}


def _pinned_pair(nbytes):
    """Two cached pinned host buffers of >= nbytes (the G-block staging ring)."""
    import torch
    key = 1 << max(20, (int(nbytes) - 1).bit_length())
    if key not in _GRING:
        _GRING.clear()
        _GRING[key] = [(torch.empty(key // 8, dtype=torch.float64, pin_memory=True), torch.cuda.Event())
                       for _ in range(2)]
    return _GRING[key]


def _draw_into(rng, k, b, out):
    """rng.standard_normal(k, b) written into out (same draws as the reference)."""
    gen = getattr(rng, "_gen", None)
    if gen is not None:
        from .fastrng import standard_normal_into
        standard_normal_into(gen, out)
    else:
        out[...] = rng.standard_normal(k, b)


def _randutv_basic_pipelined(a, b, q, rng, record_trailing):
    """fp64 randutv_basic with the host RNG overlapped with the device loop:
    the Gaussian blocks of the next group of steps are drawn straight into a
    pinned buffer and copied up on a side stream while the current group
    runs (utv_randutv_basic_steps_f64); draw order and values are exactly the
    reference's (randutv.py:189)."""
    import torch

    from . import _lib
    m, n = a.shape
    lib = _lib.load()
    steps = -(-n // b)
    sizes = [m - i * b for i in range(max(0, steps - 1))]       # rows of each drawn block
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64) if sizes else np.zeros(1, np.int64)
    t_dev = dfrom_numpy(a)
    raise_if_nonfinite(t_dev)                               # before any draw, as the reference
    anorm = math.sqrt(float(dv.sumsq(t_dev).item()))        # ErrorTracker's ||A||_F (matrix.py:79-81)
    run = dv.RandUtvRun(m, n, b, q, record_trailing)
    U, V = deye(m), deye(n)
    G = _lib.dempty(b, max(int(offs[-1]), 1))               # block i = columns offs[i]:offs[i+1]
    groups, i = [], 0
    for width in [1, 3] + [4] * steps:                      # small first group: start the GPU early
        if i >= steps:
            break
        groups.append((i, min(steps, i + width)))
        i += width
    maxcols = max((offs[min(j1, len(sizes))] - offs[j0] for j0, j1 in groups), default=1)
    ring = _pinned_pair(8 * b * max(int(maxcols), 1))
    copy_stream = torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    # results leave the GPU while later steps run: after steps [j0, j1) the
    # columns < j1*b of T, U and V are final (later steps only touch columns
    # >= lo, randutv.py:143-156)
    contiguous = t_dev.ld == m and U.ld == m and V.ld == n
    out = None
    if contiguous:
        out = (np.empty((m, m), order="F"), np.empty((m, n), order="F"), np.empty((n, n), order="F"))
        d2h = _lib.AsyncD2H()
        d2h.prefault(list(out))
        done_cols = 0
    for gi, (j0, j1) in enumerate(groups):
        d0, d1 = min(j0, len(sizes)), min(j1, len(sizes))
        ncol = int(offs[d1] - offs[d0])
        if ncol > 0:
            buf, ev = ring[gi % 2]
            ev.synchronize()                                  # previous upload from this buffer done
            host = buf.numpy()
            for j in range(d0, d1):
                lo, hi = int(offs[j] - offs[d0]) * b, int(offs[j + 1] - offs[d0]) * b
                _draw_into(rng, sizes[j], b, host[lo:hi].reshape(sizes[j], b))
            with torch.cuda.stream(copy_stream):
                G.t[int(offs[d0]):int(offs[d1]), :b].copy_(buf[: ncol * b].view(ncol, b), non_blocking=True)
                ev.record(copy_stream)
            comp.wait_event(ev)
        gptr = G.at(0, int(offs[d0])) if ncol > 0 else G.ptr
        # the b x b SVD of a group's last step stays in flight into the next
        # group (its rotations land there), so group boundaries do not drain
        # the SVD pipeline; only columns < (j1 - 1) b are final on return
        carry = (1 if gi > 0 else 0) | (2 if j1 < steps else 0)
        _lib.check(lib.utv_randutv_basic_steps_carry_f64(
            j0, j1, carry, m, n, b, q, t_dev.ptr, t_dev.ld, U.ptr, U.ld, V.ptr, V.ld, gptr, G.ld,
            run.errsq.data_ptr(), run.trail2.data_ptr() if run.trail2 is not None else None,
            run.status.data_ptr(), run.ws.data_ptr(), run.lw, _lib.stream_ptr()),
            "utv_randutv_basic_steps_carry_f64")
        if contiguous:
            fin = min(n, (j1 - 1) * b) if j1 < steps else n
            if fin > done_cols:
                ev = torch.cuda.Event()
                ev.record(comp)
                blocks = [(U, out[0], done_cols, fin if j1 < steps else m), (t_dev, out[1], done_cols, fin),
                          (V, out[2], done_cols, fin)]
                d2h.push(ev, blocks)
                done_cols = fin
    if contiguous:
        d2h.finish()
    return _finish_basic(a, b, q, run, t_dev, U, V, record_trailing, False, host=out, anorm=anorm)


@_serialized
def randutv_boosted(a, b, q, p, rng, record_trailing=False):
    """Algorithm 2: oversampling + sample recycling (randutv.py:238-247)."""
    if q < 1:
        raise ValueError(f"randutv_boosted requires q >= 1, got {q}")
    return _randutv_stepwise(a, b, q, p, rng, boosted=True, record_trailing=record_trailing)


@_serialized
def randutv_partial(a, b, q, p, rng, tol_fro=None, max_rank=None, record_trailing=False):
    """Boosted randUTV halted by error tolerance or column budget (randutv.py:250-264)."""
    if q < 1:
        raise ValueError(f"randutv_partial requires q >= 1, got {q}")
    if tol_fro is None and max_rank is None:
        raise ValueError("randutv_partial needs tol_fro or max_rank")
    return _randutv_stepwise(a, b, q, p, rng, boosted=True, tol_fro=tol_fro, max_rank=max_rank,
                             record_trailing=record_trailing)
