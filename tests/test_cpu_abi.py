"""CPU-only checks: the C-ABI library loads without a GPU and exports every
symbol include/utv_b200.h declares; ctypes signatures cover them; FLOP model
matches SURVEY §8d; the product path refuses to run without CUDA."""
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "utv_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(utv_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2106_13402_b200 import _lib
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name


def test_version_and_no_device():
    from paper_2106_13402_b200 import _lib
    lib = _lib.load()
    assert lib.utv_version() == 100
    assert lib.utv_launch_count() == 0 or lib.utv_launch_count() > 0


def test_argument_validation_without_device():
    from paper_2106_13402_b200 import _lib
    lib = _lib.load()
    # odd leading dimension -> -8 (LAPACK-style argument index), no launch
    assert lib.utv_dgemm(b"N", b"N", 4, 4, 4, 1.0, 0, 5, 0, 4, 0.0, 0, 4, 0, 0, 0) == -8
    assert lib.utv_dgemm(b"X", b"N", 4, 4, 4, 1.0, 0, 4, 0, 4, 0.0, 0, 4, 0, 0, 0) == -1
    assert lib.utv_dgeqrf(3, 4, 0, 4, 0, 4, 0, 4, 0, 0, 0) == -2          # n > m
    assert lib.utv_randutv_basic_f64(4, 4, 0, 1, 0, 4, 0, 4, 0, 4, 0, 4, 0, 0, 0, 0, 0, 0) == -3
    assert lib.utv_powerurv_f64(4, 4, -1, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 0, 0) == -3
    # the Yhat-seeded entry: q >= 1, Yhat required, LAPACK-style indices
    yh = [4, 4, 1, 0, 4, 8, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 0, 0, None, None]
    assert lib.utv_powerurv_f64_yhat(*(yh[:2] + [0] + yh[3:])) == -3       # q = 0
    assert lib.utv_powerurv_f64_yhat(*(yh[:5] + [0] + yh[6:])) == -6       # Yhat null
    assert lib.utv_powerurv_f64_yhat(*(yh[:6] + [3] + yh[7:])) == -7       # ldy0 < m
    assert lib.utv_powerurv_f64_yhat(5, 6, *yh[2:]) == -2                  # n > m
    # both event arguments of the _ev entry are optional
    assert lib.utv_powerurv_f64_ev(4, 4, -1, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 4, 0, 0, 0,
                                   None, None) == -3
    # step ranges with the carried SVD: range order, carry flags, argument indices
    st = [0, 2, 0, 8, 8, 4, 1, 0, 8, 0, 8, 0, 8, 0, 8, 0, 0, 0, 0, 0, 0]
    assert lib.utv_randutv_basic_steps_carry_f64(*([2, 1] + st[2:])) == -1           # i1 < i0
    assert lib.utv_randutv_basic_steps_carry_f64(*(st[:2] + [4] + st[3:])) == -3     # carry bits
    assert lib.utv_randutv_basic_steps_carry_f64(*(st[:3] + [4, 8] + st[5:])) == -4  # m < n
    assert lib.utv_randutv_basic_steps_carry_f64(*(st[:5] + [0] + st[6:])) == -6     # b < 1
    assert lib.utv_randutv_basic_steps_carry_f64(*(st[:8] + [7] + st[9:])) == -9     # ldt < m


def test_flop_model_matches_survey():
    import bench
    assert abs(bench.randutv_flops(16384, 16384, 256, 2) / 4.85e13 - 1) < 2e-3
    assert abs(bench.powerurv_flops(16384, 16384, 2) / 9.68e13 - 1) < 2e-3
    assert abs(bench.randutv_flops(2000, 2000, 128, 1) / 8.55e10 - 1) < 2e-3
    assert abs(bench.powerurv_flops(8192, 8192, 2) / 1.21e13 - 1) < 2e-3


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2106_13402_b200 as pk
    with pytest.raises(RuntimeError):
        pk.randutv_basic(np.eye(8), 4, 1, pk.RngStream(0))
    with pytest.raises(RuntimeError):
        pk.hqr_full(np.eye(4))


def test_validation_errors_raised_before_device():
    import paper_2106_13402_b200 as pk
    with pytest.raises(pk.DimensionError):
        pk.randutv_basic(np.ones((3, 5)), 2, 1, pk.RngStream(0))
    with pytest.raises(ValueError):
        pk.randutv_basic(np.ones((5, 5)), 0, 1, pk.RngStream(0))
    with pytest.raises(ValueError):
        pk.power_urv_from_sample(np.ones((5, 5)), -1, np.ones((5, 5)))
    with pytest.raises(pk.DimensionError):
        pk.power_urv_from_sample(np.ones((6, 4)), 1, np.ones((3, 3)))


def test_rng_stream_matches_reference_draw_order():
    """draw_sample_blocks consumes the stream exactly like randutv.py:189."""
    import paper_2106_13402_b200 as pk
    from oracle import utv_oracle as orc
    blocks = pk.randutv.draw_sample_blocks(pk.RngStream(5), 300, 260, 64)
    ref = orc.randutv_sample_blocks(orc.gaussian_stream(5), 300, 260, 64)
    assert len(blocks) == len(ref) == 4
    for x, y in zip(blocks, ref):
        assert np.array_equal(x, y)


def test_cli_usage_and_exit_codes(tmp_path):
    from paper_2106_13402_b200 import cli
    assert cli.main(["time"]) == 1                       # missing required args -> usage error
    assert cli.main(["bogus"]) == 1
    a = np.arange(12.0).reshape(4, 3) + 0.5
    p = tmp_path / "a.mtx"
    cli.save_text(a, str(p))
    assert np.array_equal(cli.load_text(str(p)), a)    # %.17g round-trips bitwise
    assert cli.main(["factor", "--algo", "nope", "--in", str(p), "--out-prefix", "x"]) == 1
    # missing input file: OSError -> exit 1 (cli.py:248-253)
    assert cli.main(["factor", "--algo", "randutv", "--in", str(tmp_path / "missing.mtx"),
                     "--out-prefix", str(tmp_path / "f")]) == 1
    assert cli.main(["--backend", "cuda", "time"]) == 1


def test_cli_plugs_into_the_reference_harness(tmp_path, monkeypatch):
    """Plug-in mode: with utvkit importable, the reference's own harness runs;
    --backend b200 serves its factorisation names from this package for the
    duration of the call, --backend reference leaves it untouched."""
    import sys

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference package not present (GPU box)")
    monkeypatch.setattr(sys, "path", [ref] + sys.path)
    monkeypatch.setattr(sys, "dont_write_bytecode", True)
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import cli
    refcli = cli.reference_cli()
    assert refcli is not None
    orig = refcli.power_urv
    with cli.b200_backend(refcli):
        assert refcli.power_urv is pk.power_urv
        assert refcli.randutv_basic is pk.randutv_basic
        assert refcli.hqrcp is pk.hqrcp
    assert refcli.power_urv is orig
    out = tmp_path / "g.mtx"
    assert cli.main(["--backend", "reference", "gen", "--kind", "gaussian", "--n", "6",
                     "--seed", "3", "--out", str(out)]) == 0
    import utvkit
    a = utvkit.read_matrix(str(out))
    assert np.array_equal(a, utvkit.gen_gaussian(6, utvkit.RngStream(3)))
    assert np.array_equal(cli.load_text(str(out)), a)
    assert cli.main(["--backend", "reference", "time"]) == 1        # the reference's usage exit


def test_comm_and_sharded_validation_without_device():
    """utv_comm_* / utv_powerurv_sharded_f64 argument checks (no device): the
    local-group communicator is host-only state; null handles are rejected."""
    import ctypes

    from paper_2106_13402_b200 import _lib
    lib = _lib.load()
    assert lib.utv_comm_init_local(0, None) == -1
    hs = (ctypes.c_void_p * 3)()
    assert lib.utv_comm_init_local(3, hs) == 0
    assert [lib.utv_comm_rank(hs[r]) for r in range(3)] == [0, 1, 2]
    assert all(lib.utv_comm_size(hs[r]) == 3 for r in range(3))
    assert lib.utv_comm_broadcast_f64(hs[0], None, 0, 5, None) == -4
    for r in range(3):
        assert lib.utv_comm_destroy(hs[r]) == 0
    assert lib.utv_comm_rank(None) == -1
    assert lib.utv_comm_allreduce_sum_f64(None, None, 1, None) == -1
    assert lib.utv_comm_init_nccl(None, 1, 0, None) == -1
    assert lib.utv_powerurv_sharded_f64(None, 10, 4, 1, 0, 10, 0, 4, 0, 10, 0, 4, 0, 4, 0, 4, 0, 4,
                                        0, 0, 0, None) == -1
    assert lib.utv_powerurv_sharded_bufsize(524288, 4096, 1, 0) > 2 * 524288 * 4096 * 8
    assert lib.utv_dnonfinite(-1, 2, 0, 2, 0, None) == -1
    assert lib.utv_slaset(b"X", 2, 2, 0.0, 1.0, 0, 2, None) == -1
