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

from . import device as dv
from ._lib import deye, dfrom_numpy
from .errors import ConsistencyError, ConvergenceError, DimensionError
from .matrix import check_matrix, frobenius_norm


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


def _validate(a, b, q, p):
    a = check_matrix(a)
    m, n = a.shape
    if m < n:
        raise DimensionError(f"randutv needs m >= n, got {a.shape}; factor the transpose")
    if b < 1:
        raise ValueError(f"block size must be >= 1, got {b}")
    if q < 0:
        raise ValueError(f"power iteration count must be >= 0, got {q}")
    if p < 0:
        raise ValueError(f"oversampling must be >= 0, got {p}")
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
    from ._lib import dempty
    m = dempty(n, n, dtype=torch.float32)
    m.t.zero_()
    idx = torch.arange(n, device="cuda")
    m.t[idx, idx] = 1.0
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


def randutv_basic(a, b, q, rng, record_trailing=False, *, dtype=np.float64):
    """Blocked randomized UTV without oversampling (randutv.py:228-235).

    dtype=np.float32 selects the fp32 variant (BASELINE C5): T, U, V are
    computed in fp32 with 3xTF32 tensor-core GEMMs and returned as float32;
    m, n and b must then be multiples of 4.  The default float64 path is the
    reference-exact drop-in."""
    import torch
    a = _validate(a, b, q, 0)
    m, n = a.shape
    b = int(b)
    q = int(q)
    f32 = np.dtype(dtype) == np.float32
    if f32 and (m % 4 or n % 4 or b % 4):
        raise ValueError("the fp32 variant needs m, n and b to be multiples of 4")
    blocks = draw_sample_blocks(rng, m, n, b)
    if f32:
        t_dev = dfrom_numpy(a, dtype=torch.float32)
        g_dev = dv.stage_randutv_blocks(blocks, b, dtype=torch.float32)
        run, U, V = randutv_basic_device32(t_dev, b, q, g_dev, record_trailing)
    else:
        t_dev = dfrom_numpy(a)
        g_dev = dv.stage_randutv_blocks(blocks, b)
        run, U, V = randutv_basic_device(t_dev, b, q, g_dev, record_trailing)
    status = run.status.cpu().numpy()
    if (status < 0).any():
        raise ConvergenceError("b x b Jacobi SVD failed to converge")
    masses = run.errsq.cpu().numpy()
    tracker = ErrorTracker.start(frobenius_norm(a))
    if f32:
        tracker.neg_tol = 1e-5
    for mass in masses:
        tracker.update_mass(mass)
    trailing = None
    if record_trailing:
        trailing = [float(math.sqrt(max(x, 0.0))) for x in run.trail2.cpu().numpy()]
        trailing[-1] = 0.0
    return UtvFactorization(
        U=np.asfortranarray(U.to_numpy()), T=np.asfortranarray(t_dev.to_numpy()),
        V=np.asfortranarray(V.to_numpy()), b=b, steps_done=run.steps, oversample=0, power=q,
        errors=list(tracker.history), trailing_fro=trailing)


def randutv_boosted(a, b, q, p, rng, record_trailing=False):
    """Algorithm 2 (randutv.py:238-247) — next row of the build plan."""
    raise NotImplementedError("randutv_boosted is not on the B200 path yet (SURVEY.md §8f row 1)")


def randutv_partial(a, b, q, p, rng, tol_fro=None, max_rank=None, record_trailing=False):
    """Partial boosted randUTV (randutv.py:250-264) — next row."""
    raise NotImplementedError("randutv_partial is not on the B200 path yet (SURVEY.md §8f row 1)")
