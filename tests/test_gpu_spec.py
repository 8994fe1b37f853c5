"""SPEC.md acceptance criteria and powerURV invariants on the B200 path
(VERDICT r1 "What's missing" 4): the reference states them in SPEC.md but
ships no executable tests, so they are ported here against the GPU results.

  * acceptance 1  reconstruction / orthogonality of every algorithm
  * acceptance 2  Theorem 3.1 projector equivalence, shared-G powerURV vs
                  RSVD (oracle.rsvd, pinned to the reference's own rsvd) (:656)
  * acceptance 4/5/7  error-curve ordering, oversampling fix and the
                  Eckart-Young floor at the paper's n=400, b=50 (:658-661)
  * acceptance 8  Kahan: hqrcp overestimates sigma_n >= 10x, boosted within 2x (:662)
  * acceptance 9  randutv_partial prefix bitwise identical to the full run (:663)
  * acceptance 10 determinism (:664)
  * powerURV KAT A = I_n and sorted |sigma(R)| = sigma(A)
"""
import numpy as np
import pytest

from oracle import utv_oracle as orc

pytestmark = pytest.mark.gpu


def _spectral_curve(t):
    n = t.shape[1]
    r = min(t.shape)
    return np.array([np.linalg.svd(t[k:r, k:], compute_uv=False)[0] if k < r else 0.0
                     for k in range(1, n)])


def _svd_curve(sig):
    return sig[1:]


def test_acceptance1_reconstruction_and_orthogonality():
    import paper_2106_13402_b200 as pk
    rng = pk.RngStream(101)
    a = pk.gaussian(300, 200, rng)
    fro = np.linalg.norm(a)
    cases = {}
    q, r = pk.hqr_full(a)
    cases["hqr"] = (pk.materialize_q(q), r, np.eye(200))
    f = pk.hqrcp(a)
    cases["hqrcp"] = (pk.materialize_q(f.q), f.R, np.eye(200)[:, f.perm])
    for qq in (0, 1, 2):
        u = pk.power_urv(a, qq, pk.RngStream(102 + qq))
        cases[f"powerurv_q{qq}"] = (u.U, u.R, u.V)
    b = pk.randutv_basic(a, 50, 2, pk.RngStream(110))
    cases["randutv_basic"] = (b.U, b.T, b.V)
    bo = pk.randutv_boosted(a, 50, 2, 50, pk.RngStream(111))
    cases["randutv_boosted"] = (bo.U, bo.T, bo.V)
    for name, (u, t, v) in cases.items():
        assert np.linalg.norm(a - u @ t @ v.T) <= 1e-12 * fro, name
        for f_ in (u, v):
            assert np.linalg.norm(f_.T @ f_ - np.eye(f_.shape[1])) <= 1e-12 * 300, name


@pytest.mark.parametrize("q", [0, 1, 2])
def test_acceptance2_projector_equivalence(golden, q):
    """U(:, 1:ell) U(:, 1:ell)^T A = U_rsvd U_rsvd^T A (Theorem 3.1): the GPU
    powerURV's leading basis against the oracle's RSVD with the same G."""
    import paper_2106_13402_b200 as pk
    z = golden("rsvd_gauss60x40")
    a, g = z["A"], z["G"]
    f = pk.power_urv_from_sample(a, q, g)
    for ell in (1, 5, 10, 20, 40):
        u_rs, _, _ = orc.rsvd(a, g, ell, q)
        gap = orc.projector_gap(pk.materialize_q(f.Uq, ell), u_rs, a)
        assert gap <= 1e-10, (ell, gap)


#: (max_k e_k/sigma_{k+1} - 1) of randutv_boosted(q=2, p=b) and randutv_basic(q=2)
#: on gen_fast_decay(400, 1e-5, RngStream(200 + 10 s)), s = 0..4, as the
#: reference utvkit computes them (build container, oracle/_ref copy)
REF_ACC5 = [(0.12409582393329655, 0.17815345097949087), (0.12634014996758114, 0.15252227044882893),
            (0.11330716108793903, 0.19557983978393081), (0.1226435540546138, 0.1604878425338876),
            (0.21769218287180414, 0.14802547572356994)]


def _curves(kind, seed):
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import matgen
    n, b = 400, 50
    if kind == "fast":
        a, sig = matgen.gen_fast_decay(n, 1e-5, pk.RngStream(seed))
    else:
        a, sig = matgen.gen_s_shaped(n, pk.RngStream(seed))
    sig = np.sort(np.asarray(sig))[::-1]
    out = {"svd": _svd_curve(sig)}
    out["boosted"] = _spectral_curve(pk.randutv_boosted(a, b, 2, b, pk.RngStream(seed + 1)).T)
    out["basic"] = _spectral_curve(pk.randutv_basic(a, b, 2, pk.RngStream(seed + 1)).T)
    out["powerurv"] = _spectral_curve(pk.power_urv(a, 2, pk.RngStream(seed + 1)).R)
    out["cpqr"] = _spectral_curve(pk.hqrcp(a).R)
    return out


@pytest.mark.parametrize("kind", ["fast", "s"])
def test_acceptance4_5_7_error_curves(kind):
    """Median-over-k spectral error ordering SVD <= boosted <= basic <=
    powerURV <= CPQR across 5 seeds (Fig. 4/6), boosted's max relative metric
    below basic's on fast decay (acceptance 5), and every curve above the
    Eckart-Young floor (acceptance 7)."""
    order = ["svd", "boosted", "basic", "powerurv", "cpqr"]
    wins = []
    for seed in range(5):
        c = _curves(kind, 200 + 10 * seed)
        med = [float(np.median(c[k] / c["svd"])) for k in order]
        assert all(med[i] <= med[i + 1] * (1 + 1e-12) for i in range(len(med) - 1)), (seed, med)
        for k in order[1:]:
            assert np.all(c[k] >= c["svd"] - 1e-9), (seed, k)
        if kind == "fast":
            ok = c["svd"] > 1e-300
            rel_b = np.max(c["boosted"][ok] / c["svd"][ok] - 1)
            rel_basic = np.max(c["basic"][ok] / c["svd"][ok] - 1)
            wins.append(rel_b < rel_basic)
            # the values are the reference's: utvkit itself gives
            # (rel_boosted, rel_basic) = (0.12410, 0.17815), (0.12634, 0.15252),
            # (0.11331, 0.19558), (0.12264, 0.16049), (0.21769, 0.14803) on
            # these five matrices (tests/golden/make_golden.py spec_acc5)
            ref = REF_ACC5[seed]
            assert abs(rel_b - ref[0]) < 1e-6 and abs(rel_basic - ref[1]) < 1e-6, (seed, rel_b, rel_basic)
    if kind == "fast":
        # acceptance 5 holds on 4 of the 5 seeds — for the reference as well
        # (seed 240 is a counterexample to SPEC.md:659 in utvkit itself)
        assert sum(wins) >= 4, wins


def test_acceptance8_kahan():
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import matgen
    a = matgen.gen_kahan(100, 1.2)
    sn = np.linalg.svd(a, compute_uv=False)[-1]
    r = pk.hqrcp(a).R
    assert abs(r[99, 99]) >= 10 * sn
    t = pk.randutv_boosted(a, 50, 2, 50, pk.RngStream(7)).T
    assert sn / 2 <= abs(t[99, 99]) <= 2 * sn


def test_acceptance9_partial_prefix_bitwise():
    import paper_2106_13402_b200 as pk
    rng = np.random.default_rng(9)
    a = rng.standard_normal((400, 400)) * np.logspace(0, -5, 400)
    b, q, p = 50, 2, 50
    full = pk.randutv_boosted(a, b, q, p, pk.RngStream(12))
    part = pk.randutv_partial(a, b, q, p, pk.RngStream(12), max_rank=2 * b)
    assert part.steps_done == 2
    k = 2 * b
    assert np.array_equal(part.T[:, :k], full.T[:, :k])
    assert np.array_equal(part.U[:, :k], full.U[:, :k])
    assert np.array_equal(part.V[:, :k], full.V[:, :k])
    # the reference's partial run records e0 and one tracked error per step
    # before the max_rank stop (checked against utvkit itself: 2 entries here)
    assert part.errors == full.errors[:len(part.errors)]


def test_acceptance10_determinism():
    import paper_2106_13402_b200 as pk
    a = pk.gaussian(257, 190, pk.RngStream(3))
    for fn in (lambda: pk.randutv_basic(a, 64, 2, pk.RngStream(4)),
               lambda: pk.randutv_boosted(a, 64, 1, 16, pk.RngStream(4))):
        x, y = fn(), fn()
        for key in ("U", "T", "V"):
            assert np.array_equal(getattr(x, key), getattr(y, key)), key
    u1, u2 = pk.power_urv(a, 2, pk.RngStream(4)), pk.power_urv(a, 2, pk.RngStream(4))
    assert np.array_equal(u1.R, u2.R)
    assert np.array_equal(u1.Uq.Y, u2.Uq.Y) and np.array_equal(u1.Vq.Twy, u2.Vq.Twy)


@pytest.mark.parametrize("q", [0, 1, 2])
def test_powerurv_identity_kat(q):
    """A = I_n: |diag(R)| = 1 within 1e-13, e_k = Eckart-Young within 1e-12
    (SPEC.md:333)."""
    import paper_2106_13402_b200 as pk
    n = 64
    f = pk.power_urv(np.eye(n), q, pk.RngStream(5))
    assert np.abs(np.abs(np.diag(f.R)) - 1.0).max() < 1e-13
    e = pk.trailing_fro_curve(f.R)
    ey = np.sqrt(np.arange(n - 1, 0, -1, dtype=float))
    assert np.abs(e - ey).max() < 1e-12


@pytest.mark.parametrize("q", [0, 2])
def test_powerurv_singular_values_preserved(q):
    """sorted |sigma(R)| = sigma(A) within 1e-11 relative."""
    import paper_2106_13402_b200 as pk
    a, d = orc.decay_matrix(150, 1e-6, seed=8, m=200)
    f = pk.power_urv(a, q, pk.RngStream(9))
    s_r = np.linalg.svd(f.R, compute_uv=False)
    s_a = np.linalg.svd(a, compute_uv=False)
    assert np.abs(s_r - s_a).max() <= 1e-11 * s_a[0]
