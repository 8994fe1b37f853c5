"""GPU generators (matgen drop-in) and device metrics
against the reference's own generator outputs and the host metrics."""
import numpy as np
import pytest

from oracle import utv_oracle as orc

pytestmark = pytest.mark.gpu


def test_generators_match_reference(golden):
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import matgen as mg
    g = golden("matgen_small")
    a, d = mg.gen_fast_decay(64, 1e-3, pk.RngStream(71))
    assert np.array_equal(d, g["fast_d"])
    assert np.abs(a - g["fast"]).max() < 1e-13
    b, e = mg.gen_s_shaped(48, pk.RngStream(72))
    assert np.array_equal(e, g["s_d"])
    assert np.abs(b - g["s"]).max() < 1e-13
    assert np.abs(mg.random_orthogonal(40, pk.RngStream(73)) - g["orth"]).max() < 1e-13
    assert np.abs(mg.gen_bie(20) - g["bie"]).max() < 1e-15
    assert np.abs(mg.gen_kahan(12) - g["kahan"]).max() < 1e-15
    assert np.abs(mg.gen_kahan(9, 0.7) - g["kahan_th"]).max() < 1e-15
    assert np.array_equal(mg.gen_gaussian(10, pk.RngStream(74)), g["gauss"])


@pytest.mark.parametrize("shape", [(2, 2), (50, 30), (257, 257), (1000, 700)])
def test_trailing_fro_device_matches_host(shape):
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200._lib import dfrom_numpy
    from paper_2106_13402_b200.metrics import trailing_fro_curve_device
    rng = np.random.default_rng(shape[0])
    t = rng.standard_normal(shape)
    host = pk.trailing_fro_curve(t)
    dev = trailing_fro_curve_device(dfrom_numpy(t))
    assert dev.shape == host.shape
    assert np.allclose(dev, host, rtol=1e-12, atol=1e-12)


def test_device_reconstruction_orthogonality():
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200._lib import dfrom_numpy
    from paper_2106_13402_b200.metrics import orthogonality_device, reconstruction_device
    a, _ = orc.decay_matrix(300, 1e-5, seed=3)
    f = pk.randutv_basic(a, 64, 1, pk.RngStream(1))
    r_dev = reconstruction_device(dfrom_numpy(a), dfrom_numpy(f.U), dfrom_numpy(f.T), dfrom_numpy(f.V))
    assert abs(r_dev - orc.reconstruction(a, f.U, f.T, f.V)) < 1e-15
    o_dev = orthogonality_device(dfrom_numpy(f.U))
    assert abs(o_dev - orc.orthogonality(f.U)) < 1e-15


def test_cli_time_and_factor(tmp_path, capsys):
    from paper_2106_13402_b200 import cli
    assert cli.main(["gen", "--kind", "fast", "--n", "120", "--out", str(tmp_path / "a.mtx")]) == 0
    assert cli.main(["factor", "--algo", "randutv", "--b", "32", "--q", "1", "--in", str(tmp_path / "a.mtx"),
                     "--out-prefix", str(tmp_path / "f")]) == 0
    a = cli.load_text(str(tmp_path / "a.mtx"))
    u, t, v = (cli.load_text(str(tmp_path / f"f.{x}.mtx")) for x in "UTV")
    assert np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a) < 1e-13
    assert cli.main(["errors", "--in", str(tmp_path / "a.mtx"), "--factors", str(tmp_path / "f"),
                     "--norm", "fro", "--csv", str(tmp_path / "e.csv")]) == 0
    rows = (tmp_path / "e.csv").read_text().splitlines()
    assert rows[0] == "k,e_k,e_opt,rel" and len(rows) == 120
    assert cli.main(["check-rsvd", "--n", "64", "--ell", "8", "--q", "1"]) == 0
    assert cli.main(["time", "--algo", "powerurv", "--n", "200", "--q", "1", "--reps", "2",
                     "--csv", str(tmp_path / "t.csv")]) == 0
    out = capsys.readouterr().out
    assert "powerurv n=200: median" in out


def test_cli_cpqr_factor(tmp_path):
    """cli.py:65-68 semantics for the GPU comparator: U = Q, T = R, V = I[:, perm]."""
    from paper_2106_13402_b200 import cli
    assert cli.main(["gen", "--kind", "kahan", "--n", "60", "--out", str(tmp_path / "k.mtx")]) == 0
    assert cli.main(["factor", "--algo", "cpqr", "--in", str(tmp_path / "k.mtx"),
                     "--out-prefix", str(tmp_path / "c")]) == 0
    a = cli.load_text(str(tmp_path / "k.mtx"))
    u, t, v = (cli.load_text(str(tmp_path / f"c.{x}.mtx")) for x in "UTV")
    assert np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a) < 1e-13
    assert np.abs(np.tril(t, -1)).max() == 0.0


def test_cli_b200_backend_inside_the_reference_harness(tmp_path):
    """Plug-in mode on the GPU box: the reference harness (the unmodified copy
    oracle/_ref, test infrastructure) drives this package's randUTV through
    `--backend b200`; the factors it writes reconstruct A."""
    import sys

    from oracle import build_ref
    if not build_ref.available():
        pytest.skip("oracle/_ref not built")
    build_ref.load()                      # puts the verified copy on sys.path as `utvkit`
    from paper_2106_13402_b200 import cli
    assert cli.reference_cli() is not None
    a_path = tmp_path / "a.mtx"
    assert cli.main(["gen", "--kind", "gaussian", "--n", "96", "--out", str(a_path)]) == 0
    assert cli.main(["factor", "--algo", "randutv", "--b", "32", "--q", "1", "--in", str(a_path),
                     "--out-prefix", str(tmp_path / "f")]) == 0
    a = cli.load_text(str(a_path))
    u, t, v = (cli.load_text(str(tmp_path / f"f.{x}.mtx")) for x in "UTV")
    assert np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a) < 1e-13
    assert cli.main(["errors", "--in", str(a_path), "--factors", str(tmp_path / "f"),
                     "--norm", "fro", "--csv", str(tmp_path / "e.csv")]) == 0
    for mod in [m for m in sys.modules if m == "utvkit" or m.startswith("utvkit.")]:
        sys.modules.pop(mod)
    if build_ref.DST_ROOT in sys.path:
        sys.path.remove(build_ref.DST_ROOT)
