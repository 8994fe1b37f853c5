"""Pin the CPU oracle (oracle/utv_oracle.py) to golden vectors produced by the
reference package itself (tests/golden/make_golden.py).  CPU only."""
import glob
import os

import numpy as np
import pytest

from oracle import utv_oracle as orc
from tests.conftest import GOLDEN


def _names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


@pytest.mark.parametrize("name", _names("hqr_"))
def test_householder_qr_matches_reference(golden, name):
    g = golden(name)
    y, t, r = orc.householder_qr(g["A"])
    scale = max(1.0, np.abs(g["A"]).max())
    assert np.abs(y - g["Y"]).max() <= 1e-12
    assert np.abs(t - g["Twy"]).max() <= 1e-12
    assert np.abs(r - g["R"]).max() <= 1e-12 * scale
    # exact structural zeros below the diagonal of R, above the diagonal of Y
    assert not np.tril(r, -1).any()
    assert not np.triu(y, 1).any()


def test_wy_apply_matches_reference(golden):
    g = golden("applyq_50x30")
    y, t, _ = orc.householder_qr(g["A"])
    assert np.abs(orc.wy_apply(y, t, g["BL"], "left") - g["left"]).max() < 1e-13
    assert np.abs(orc.wy_apply(y, t, g["BL"], "left", True) - g["left_t"]).max() < 1e-13
    assert np.abs(orc.wy_apply(y, t, g["BR"], "right") - g["right"]).max() < 1e-13
    assert np.abs(orc.wy_apply(y, t, g["BR"], "right", True) - g["right_t"]).max() < 1e-13
    assert np.abs(orc.wy_materialize(y, t) - g["Q"]).max() < 1e-14
    assert np.abs(orc.wy_materialize(y, t, 30) - g["Q30"]).max() < 1e-14


@pytest.mark.parametrize("name", _names("svd_"))
def test_svd_signed_matches_reference(golden, name):
    g = golden(name)
    u, s, v = orc.svd_signed(g["A"])
    assert np.abs(s - g["sigma"]).max() <= 1e-13 * max(1.0, g["sigma"].max())
    if name in ("svd_rank1",):      # null-space vectors are not unique
        assert np.abs(np.abs(u[:, 0]) - np.abs(g["U"][:, 0])).max() < 1e-12
        return
    assert np.abs(u - g["U"]).max() < 1e-12
    assert np.abs(v - g["V"]).max() < 1e-12


@pytest.mark.parametrize("name", _names("purv_"))
def test_power_urv_matches_reference(golden, name):
    g = golden(name)
    if "G" in g:
        gm = g["G"]
    else:
        gm = orc.draw_gaussian(orc.gaussian_stream(int(g["seed"])), g["A"].shape[1], g["A"].shape[1])
    f = orc.power_urv(g["A"], int(g["q"]), gm)
    for k in ("Uy", "Ut", "Vy", "Vt"):
        assert np.abs(f[k] - g[k]).max() < 1e-9, k
    assert np.abs(f["R"] - g["R"]).max() < 1e-10 * np.abs(g["A"]).max()


@pytest.mark.parametrize("name", _names("rutv_"))
def test_randutv_basic_matches_reference(golden, name):
    g = golden(name)
    a = g["A"]
    m, n = a.shape
    b, q = int(g["b"]), int(g["q"])
    blocks = orc.randutv_sample_blocks(orc.gaussian_stream(int(g["seed"])), m, n, b)
    f = orc.randutv_basic(a, b, q, blocks, record_trailing=True)
    anorm = np.linalg.norm(a, 2)
    tol = lambda ref: 1e-10 * np.abs(ref) + 16 * orc.EPS * anorm  # noqa: E731
    assert f["steps"] == int(g["steps"])
    assert (np.abs(np.diag(f["T"]) - np.diag(g["T"])) <= tol(np.diag(g["T"]))).all()
    ek = orc.trailing_fro(f["T"])
    assert (np.abs(ek - g["efro"]) <= tol(g["efro"])).all()
    assert np.abs(f["U"] - g["U"]).max() < 1e-8
    assert np.abs(f["V"] - g["V"]).max() < 1e-8
    assert np.allclose(f["errors"], g["errors"], rtol=1e-8, atol=1e-7 * np.linalg.norm(a))
    assert orc.reconstruction(a, f["U"], f["T"], f["V"]) < 1e-13


@pytest.mark.parametrize("name", sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "boost_*.npz"))))
def test_oracle_boosted_matches_reference(golden, name):
    """The boosted / partial restatement against the reference's own outputs,
    including where the generator is left (next draw)."""
    g = golden(name)
    gen = orc.gaussian_stream(int(g["seed"]))
    tol = None if np.isnan(g["tol"]) else float(g["tol"])
    mr = None if int(g["max_rank"]) < 0 else int(g["max_rank"])
    out = orc.randutv_boosted(g["A"], int(g["b"]), int(g["q"]), int(g["p"]), gen, tol_fro=tol,
                              max_rank=mr, record_trailing=True)
    assert gen.standard_normal((1, 1))[0, 0] == g["next_normal"]
    assert out["steps"] == int(g["steps"])
    assert np.abs(out["T"] - g["T"]).max() < 1e-9 * max(1.0, np.abs(g["T"]).max())
    assert np.abs(np.diag(out["T"]) - np.diag(g["T"])).max() < 1e-11
    assert np.allclose(out["errors"], g["errors"], rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("name", _names("qrcp_"))
def test_oracle_hqrcp_matches_reference(golden, name):
    """Column-pivoted QR restatement (qr.py:152-204): identical pivots, and the
    factors to roundoff, on tie / skip / recompute / wide / degenerate inputs."""
    g = golden(name)
    y, t, r, perm = orc.hqrcp(g["A"] if "A" in g else g["a"])
    assert (perm == g["perm"]).all()
    scale = max(1.0, np.abs(g["R"]).max())
    assert np.abs(r - g["R"]).max() <= 1e-13 * scale
    assert np.abs(y - g["Y"]).max() <= 1e-12
    assert np.abs(t - g["Twy"]).max() <= 1e-12


def test_oracle_rsvd_matches_reference(golden):
    """The oracle's rsvd / projector_gap restatement against the reference's
    own outputs (tests/golden/make_golden.py rsvd)."""
    z = golden("rsvd_gauss60x40")
    a, g = z["A"], z["G"]
    for q in (0, 1, 2):
        urv = orc.power_urv(a, q, g)
        for ell in (1, 5, 10, 20, 40):
            u, s, _ = orc.rsvd(a, g, ell, q)
            assert np.abs(s - z[f"sigma_q{q}_l{ell}"]).max() < 1e-12 * s[0]
            assert np.abs(np.abs(u) - np.abs(z[f"U_rsvd_q{q}_l{ell}"])).max() < 1e-10
            gap = orc.projector_gap(orc.wy_materialize(urv["Uy"], urv["Ut"], ell), u, a)
            assert gap <= 1e-10 and abs(gap - float(z[f"gap_q{q}_l{ell}"])) < 1e-12
