"""End-to-end GPU parity of the drop-in API (paper_2106_13402_b200) with the
reference: golden vectors produced by utvkit itself, plus the CPU oracle at
C1 size (randUTV b=128 q=1 on a 2000^2 geometric-decay matrix).

Tolerances (BASELINE.json north star): diag(T)/diag(R) and the
Frobenius e_k curve within 1e-10 relative with an absolute floor of
16*eps*||A||_2 (mixed gate); U/V element-wise max-abs;
reconstruction and orthogonality at roundoff level.
"""
import glob
import os

import numpy as np
import pytest

from oracle import utv_oracle as orc
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def _mixed_ok(x, ref, anorm2, rel=1e-10):
    return np.all(np.abs(x - ref) <= rel * np.abs(ref) + 16 * orc.EPS * anorm2)


@pytest.mark.parametrize("name", _names("rutv_"))
def test_randutv_basic_matches_reference(golden, name):
    import paper_2106_13402_b200 as pk
    g = golden(name)
    a = g["A"]
    b, q, seed = int(g["b"]), int(g["q"]), int(g["seed"])
    f = pk.randutv_basic(a, b, q, pk.RngStream(seed), record_trailing=True)
    anorm2 = np.linalg.norm(a, 2)
    assert f.steps_done == int(g["steps"])
    assert _mixed_ok(np.diag(f.T), np.diag(g["T"]), anorm2)
    assert _mixed_ok(pk.trailing_fro_curve(f.T), g["efro"], anorm2)
    m, n = a.shape
    # Singular vectors are compared where they are determined: columns whose
    # diag(T) value is above the rank-deficiency noise (1e-8 ||A||_2), and for
    # tall inputs only the first n columns of U (the rest is a non-unique
    # orthonormal completion, as with LAPACK).
    d = np.abs(np.diag(g["T"]))
    k = int(np.sum(d > 1e-8 * anorm2))
    assert np.abs(f.U[:, :k] - g["U"][:, :k]).max() < 1e-8
    assert np.abs(f.V[:, :k] - g["V"][:, :k]).max() < 1e-8
    assert orc.reconstruction(a, f.U, f.T, f.V) < 1e-13
    assert orc.orthogonality(f.U) < 1e-13 * m
    assert orc.orthogonality(f.V) < 1e-13 * n
    assert np.allclose(f.errors, g["errors"], rtol=1e-8, atol=1e-7 * np.linalg.norm(a))
    assert np.allclose(f.trailing_fro, g["trailing"], rtol=1e-9, atol=1e-12 * np.linalg.norm(a))
    # structural zeros (randutv.py:149,154)
    T = f.T
    for i in range(f.steps_done - 1):
        lo, mid = i * b, (i + 1) * b
        assert not T[mid:, lo:mid].any()
        blk = T[lo:mid, lo:mid]
        assert not (blk - np.diag(np.diag(blk))).any()


@pytest.mark.parametrize("name", _names("purv_"))
def test_power_urv_matches_reference(golden, name):
    import paper_2106_13402_b200 as pk
    g = golden(name)
    a = g["A"]
    q = int(g["q"])
    if "G" in g:
        f = pk.power_urv_from_sample(a, q, g["G"])
    else:
        f = pk.power_urv(a, q, pk.RngStream(int(g["seed"])))
    anorm2 = np.linalg.norm(a, 2)
    assert _mixed_ok(np.diag(f.R), np.diag(g["R"]), anorm2)
    assert _mixed_ok(pk.trailing_fro_curve(f.R), orc.trailing_fro(g["R"]), anorm2)
    for got, ref in [(f.Uq.Y, g["Uy"]), (f.Uq.Twy, g["Ut"]), (f.Vq.Y, g["Vy"]), (f.Vq.Twy, g["Vt"])]:
        assert np.abs(got - ref).max() < 1e-9
    U, V = f.U, f.V
    assert orc.reconstruction(a, U, f.R, V) < 1e-13
    assert orc.orthogonality(U) < 1e-13 * a.shape[0]


def test_randutv_c1_against_oracle():
    """C1: randUTV b=128 q=1 on a 2000x2000 geometric-decay (beta=1e-5) matrix."""
    import paper_2106_13402_b200 as pk
    a, d = orc.decay_matrix(2000, 1e-5, seed=7)
    blocks = orc.randutv_sample_blocks(orc.gaussian_stream(1), 2000, 2000, 128)
    ref = orc.randutv_basic(a, 128, 1, blocks)
    f = pk.randutv_basic(a, 128, 1, pk.RngStream(1))
    anorm2 = d[0]
    assert _mixed_ok(np.diag(f.T), np.diag(ref["T"]), anorm2)
    assert _mixed_ok(pk.trailing_fro_curve(f.T), orc.trailing_fro(ref["T"]), anorm2)
    assert np.abs(f.U - ref["U"]).max() < 1e-8
    assert np.abs(f.V - ref["V"]).max() < 1e-8
    assert orc.reconstruction(a, f.U, f.T, f.V) < 1e-13
    # north-star gate: orthogonality defects agree to 1e-10 (absolute, they are ~1e-13)
    assert abs(orc.orthogonality(f.U) - orc.orthogonality(ref["U"])) < 1e-10
    assert abs(orc.orthogonality(f.V) - orc.orthogonality(ref["V"])) < 1e-10


def test_power_urv_c2_shape_small_against_oracle():
    """powerURV q=2 on a Gaussian-decay 768^2 matrix vs the oracle."""
    import paper_2106_13402_b200 as pk
    n = 768
    a, d = orc.decay_matrix(n, 1e-5, seed=20)
    g = orc.draw_gaussian(orc.gaussian_stream(2), n, n)
    ref = orc.power_urv(a, 2, g)
    f = pk.power_urv_from_sample(a, 2, g)
    assert _mixed_ok(np.diag(f.R), np.diag(ref["R"]), d[0])
    assert _mixed_ok(pk.trailing_fro_curve(f.R), orc.trailing_fro(ref["R"]), d[0])
    assert np.abs(f.Vq.Y - ref["Vy"]).max() < 1e-8
    assert np.abs(f.Uq.Y - ref["Uy"]).max() < 1e-8


@pytest.mark.parametrize("m,n,q", [(2304, 2048, 1), (2048, 2048, 2), (2600, 2100, 1)])
def test_power_urv_streamed_draw_matches_from_sample(m, n, q):
    """power_urv at n >= 2048 draws G row block by row block while the device
    forms Yhat = A G as K-chunked GEMMs (utv_powerurv_f64_yhat): the same G as
    the reference's single n x n draw (identical generator state afterwards)
    and the same factorisation as power_urv_from_sample on that G."""
    import paper_2106_13402_b200 as pk
    rng_a = np.random.default_rng(m + n + q)
    a = np.asfortranarray(rng_a.standard_normal((m, n)) * np.exp(-np.arange(n) / (n / 8.0)))
    r1, r2 = pk.RngStream(9), pk.RngStream(9)
    f = pk.power_urv(a, q, r1)
    g = pk.gaussian(n, n, r2)
    ref = pk.power_urv_from_sample(a, q, g)
    assert r1._gen.bit_generator.state == r2._gen.bit_generator.state
    anorm2 = np.linalg.norm(a, 2)
    assert _mixed_ok(np.diag(f.R), np.diag(ref.R), anorm2)
    assert np.abs(f.Vq.Y - ref.Vq.Y).max() < 1e-8
    assert np.abs(f.Uq.Y - ref.Uq.Y).max() < 1e-8
    assert np.abs(f.Vq.Twy - ref.Vq.Twy).max() < 1e-8


@pytest.mark.parametrize("m,n,q", [(1001, 300, 1), (1002, 301, 2), (1003, 257, 1), (1005, 1005, 1),
                                   (1006, 700, 0)])
def test_power_urv_ragged_rows_against_oracle(m, n, q):
    """Row counts that are not a multiple of 4 (the device buffers pad their
    leading dimensions; the compact-WY workspaces must account for that)."""
    import paper_2106_13402_b200 as pk
    a, d = orc.decay_matrix(n, 1e-5, seed=m + q, m=m)
    g = orc.draw_gaussian(orc.gaussian_stream(m), n, n)
    ref = orc.power_urv(a, q, g)
    f = pk.power_urv_from_sample(a, q, g)
    assert _mixed_ok(np.diag(f.R), np.diag(ref["R"]), d[0])
    assert np.abs(f.Vq.Y - ref["Vy"]).max() < 1e-8
    assert np.abs(f.Uq.Y - ref["Uy"]).max() < 1e-8


@pytest.mark.parametrize("m,n,b", [(1002, 999, 128), (1001, 1001, 96), (1003, 513, 256), (700, 650, 33),
                                   (515, 515, 61), (2000, 1500, 255)])
def test_randutv_ragged_against_oracle(m, n, b):
    import paper_2106_13402_b200 as pk
    a, d = orc.decay_matrix(n, 1e-5, seed=m + b, m=m)
    blocks = orc.randutv_sample_blocks(orc.gaussian_stream(b), m, n, b)
    ref = orc.randutv_basic(a, b, 1, blocks)
    f = pk.randutv_basic(a, b, 1, pk.RngStream(b))
    # mid-block diag(T) entries of these shapes move by up to ~4e-10 relative
    # under rounding-sized perturbations (the oracle against itself), so the
    # gate is max(1e-10 mixed tolerance, 4x the spread measured here over
    # three 1-ulp perturbations of A and three of the Gaussian blocks — the
    # latter stand for the rounding of the first sampling product)
    #
    spread = np.zeros(n)
    env_u = env_v = 0.0
    for s in range(3):
        r = np.random.default_rng(m + s)
        a2 = a * (1.0 + orc.EPS * r.standard_normal(a.shape))
        g2 = [g * (1.0 + orc.EPS * r.standard_normal(g.shape)) for g in blocks]
        for x, bl in ((a2, blocks), (a, g2)):
            rr = orc.randutv_basic(x, b, 1, bl)
            spread = np.maximum(spread, np.abs(np.diag(rr["T"]) - np.diag(ref["T"])))
            env_u = max(env_u, float(np.abs(rr["U"][:, :n] - ref["U"][:, :n]).max()))
            env_v = max(env_v, float(np.abs(rr["V"] - ref["V"]).max()))
    tol = np.maximum(1e-10 * np.abs(np.diag(ref["T"])) + 16 * orc.EPS * d[0], 4 * spread)
    err = np.abs(np.diag(f.T) - np.diag(ref["T"]))
    bad = np.flatnonzero(err > tol)
    assert bad.size == 0, [(int(i), float(err[i]), float(tol[i]), float(spread[i]),
                            float(np.diag(ref["T"])[i])) for i in bad[:6]]
    # tall input: U[:, n:] is a non-unique orthonormal completion (as with LAPACK);
    # singular vectors of close singular values carry the same measured envelope
    assert np.abs(f.U[:, :n] - ref["U"][:, :n]).max() < max(1e-8, 4 * env_u)
    assert np.abs(f.V - ref["V"]).max() < max(1e-8, 4 * env_v)
    assert orc.reconstruction(a, f.U, f.T, f.V) < 1e-13
    assert orc.orthogonality(f.U) < 1e-13 * m


def test_api_errors_match_reference():
    import paper_2106_13402_b200 as pk
    with pytest.raises(pk.DimensionError):
        pk.randutv_basic(np.ones((3, 5)), 2, 1, pk.RngStream(0))
    with pytest.raises(ValueError):
        pk.randutv_basic(np.ones((5, 5)), 0, 1, pk.RngStream(0))
    with pytest.raises(ValueError):
        pk.power_urv(np.full((4, 4), np.nan), 1, pk.RngStream(0))
    with pytest.raises(pk.DimensionError):
        pk.power_urv_from_sample(np.ones((6, 4)), 1, np.ones((3, 3)))
    with pytest.raises(pk.DimensionError):
        pk.hqr_full(np.ones((2, 3)))


class _PerturbedStream:
    """The reference's Gaussian stream with every draw perturbed by one ulp
    (stands for the rounding of the first sampling product)."""

    def __init__(self, seed, salt):
        self.gen = orc.gaussian_stream(seed)
        self.r = np.random.default_rng(salt)

    def standard_normal(self, shape):
        g = self.gen.standard_normal(shape)
        return g * (1.0 + orc.EPS * self.r.standard_normal(g.shape))


def _boosted_envelope(a, b, q, p, seed, name, steps):
    """max |x - x'| of diag(T) and e_k of the oracle's boosted / partial run
    over 1-ulp perturbations of A and of the Gaussian draws."""
    def run(x, gen):
        if name.startswith("boost_partial"):
            r = orc.randutv_boosted(x, b, q, p, gen, max_rank=steps * b)
        else:
            r = orc.randutv_boosted(x, b, q, p, gen)
        return np.diag(r["T"]), orc.trailing_fro(r["T"])
    d0, e0 = run(a, orc.gaussian_stream(seed))
    env_d, env_e = np.zeros_like(d0), np.zeros_like(e0)
    for s in range(2):
        pa = np.asfortranarray(a * (1.0 + orc.EPS * np.random.default_rng(s).standard_normal(a.shape)))
        for x, gen in ((pa, orc.gaussian_stream(seed)), (a, _PerturbedStream(seed, 10 + s))):
            d, e = run(x, gen)
            env_d, env_e = np.maximum(env_d, np.abs(d - d0)), np.maximum(env_e, np.abs(e - e0))
    return env_d, env_e


@pytest.mark.parametrize("name", _names("boost_"))
def test_randutv_boosted_partial_match_reference(golden, name):
    """Algorithm 2 (randutv_boosted) and randutv_partial against the reference's
    own outputs (tests/golden/make_golden.py boosted), incl. RNG consumption."""
    import paper_2106_13402_b200 as pk
    g = golden(name)
    a = g["A"]
    b, q, p, seed = int(g["b"]), int(g["q"]), int(g["p"]), int(g["seed"])
    rng = pk.RngStream(seed)
    if name.startswith("boost_partial"):
        tol = None if np.isnan(g["tol"]) else float(g["tol"])
        mr = None if int(g["max_rank"]) < 0 else int(g["max_rank"])
        f = pk.randutv_partial(a, b, q, p, rng, tol_fro=tol, max_rank=mr, record_trailing=True)
    else:
        f = pk.randutv_boosted(a, b, q, p, rng, record_trailing=True)
    assert rng.standard_normal(1, 1)[0, 0] == g["next_normal"]     # same draws consumed
    anorm2 = np.linalg.norm(a, 2)
    assert f.steps_done == int(g["steps"]) and f.oversample == p and f.power == q
    # Gate: 1e-10 relative (+ the absolute floor) or 4x the reference
    # algorithm's OWN rounding envelope, measured here: the oracle (pinned to
    # the reference) on A and on A(1+eps).  The boosted basis selection is
    # more sensitive than the basic sampler on the 1e-5 fast-decay input.
    env_d, env_e = _boosted_envelope(a, b, q, p, seed, name, f.steps_done)
    for x, ref, env, what in ((np.diag(f.T), np.diag(g["T"]), env_d, "diag(T)"),
                              (pk.trailing_fro_curve(f.T), g["efro"], env_e, "e_k")):
        tol = np.maximum(1e-10 * np.abs(ref) + 16 * orc.EPS * anorm2, 4 * env)
        bad = np.flatnonzero(np.abs(x - ref) > tol)
        assert bad.size == 0, (what, [(int(i), float(abs(x[i] - ref[i])), float(tol[i]))
                                      for i in bad[:6]])
    d = np.abs(np.diag(g["T"]))
    k = int(np.sum(d[: f.steps_done * b] > 1e-8 * anorm2))
    assert np.abs(f.U[:, :k] - g["U"][:, :k]).max() < 1e-8
    assert np.abs(f.V[:, :k] - g["V"][:, :k]).max() < 1e-8
    assert orc.reconstruction(a, f.U, f.T, f.V) < 1e-13
    assert orc.orthogonality(f.U) < 1e-13 * a.shape[0]
    assert orc.orthogonality(f.V) < 1e-13 * a.shape[1]
    assert np.allclose(f.errors, g["errors"], rtol=1e-8, atol=1e-7 * np.linalg.norm(a))
    assert np.allclose(f.trailing_fro, g["trailing"], rtol=1e-9, atol=1e-12 * np.linalg.norm(a))


def test_public_api_concurrent_threads_match_sequential():
    """The reference API is pure and re-entrant: calls made from several host
    threads at once (sharing the library's side streams and the pinned
    staging rings) return exactly what the same calls return one by one."""
    import threading

    import paper_2106_13402_b200 as pk
    rng = np.random.default_rng(77)
    a1 = np.asfortranarray(rng.standard_normal((2048, 2048)) * np.exp(-np.arange(2048) / 300.0))
    a2 = np.asfortranarray(rng.standard_normal((1100, 1100)))

    def job_purv():
        return pk.power_urv(a1, 1, pk.RngStream(5))

    def job_rutv():
        return pk.randutv_basic(a2, 128, 1, pk.RngStream(6))

    seq = [job_purv(), job_rutv()]
    out = [None, None]

    def run(i, f):
        out[i] = f()
    ths = [threading.Thread(target=run, args=(0, job_purv)), threading.Thread(target=run, args=(1, job_rutv))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert np.array_equal(out[0].R, seq[0].R) and np.array_equal(out[0].Vq.Y, seq[0].Vq.Y)
    assert np.array_equal(out[1].T, seq[1].T) and np.array_equal(out[1].U, seq[1].U)


def test_power_urv_overlapped_upload_is_bitwise_the_serial_one():
    """n >= STREAM_MIN_N and >= OVERLAP_A_MIN_BYTES: A goes up block by block
    under the G draw (powerurv._power_urv_streamed).  Same chunks, same
    GEMMs: the factors equal the serial-upload path bit for bit, and a
    non-finite A raises ValueError without advancing the caller's stream."""
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import powerurv
    n = 3072
    rng = np.random.default_rng(31)
    a = np.asfortranarray(rng.standard_normal((n, n)) * np.logspace(0, -6, n)[None, :])
    assert a.nbytes >= powerurv.OVERLAP_A_MIN_BYTES
    f = pk.power_urv(a, 1, pk.RngStream(8))
    old = powerurv.OVERLAP_A_MIN_BYTES
    powerurv.OVERLAP_A_MIN_BYTES = 1 << 62
    try:
        g = pk.power_urv(a, 1, pk.RngStream(8))
    finally:
        powerurv.OVERLAP_A_MIN_BYTES = old
    assert np.array_equal(f.R, g.R)
    assert np.array_equal(f.Uq.Y, g.Uq.Y) and np.array_equal(f.Uq.Twy, g.Uq.Twy)
    assert np.array_equal(f.Vq.Y, g.Vq.Y) and np.array_equal(f.Vq.Twy, g.Vq.Twy)
    bad = a.copy()
    bad[n - 7, n - 3] = np.inf                # in the last column block
    s = pk.RngStream(8)
    with pytest.raises(ValueError):
        pk.power_urv(bad, 1, s)
    assert np.array_equal(s.standard_normal(2, 3), pk.RngStream(8).standard_normal(2, 3))
