"""GPU tests of the row-sharded powerURV path through the
C ABI: the reconstruction kernels (signed LU, right triangular solve), the
single-rank TSQR path with row chunking, and P = 2/3/4 ranks emulated as
threads sharing one B200 (ThreadComm) — all against the CPU oracle."""
import threading

import numpy as np
import pytest

from oracle import utv_oracle as orc
from tests.numpy_ops import NumpyOps
from tests.test_sharded_cpu import _case, _check

pytestmark = pytest.mark.gpu


def _dm(a):
    from paper_2106_13402_b200._lib import dfrom_numpy
    return dfrom_numpy(a)


@pytest.mark.parametrize("m,n", [(64, 64), (300, 70), (5000, 257), (3000, 600)])
def test_getrf_signed_matches_numpy(m, n):
    import paper_2106_13402_b200.device as dv
    rng = np.random.default_rng(m + n)
    q, _ = np.linalg.qr(rng.standard_normal((m, n)))
    ref = np.array(q, order="F")
    s_ref = NumpyOps().getrf_signed(ref).numpy()
    d = _dm(q)
    s = dv.getrf_signed(d).cpu().numpy()
    assert np.array_equal(s, s_ref)
    assert np.abs(d.to_numpy() - ref).max() < 1e-12


@pytest.mark.parametrize("n", [200, 600])
@pytest.mark.parametrize("uplo,trans,diag", [("U", "N", "N"), ("L", "T", "U"), ("U", "N", "U")])
def test_trsm_right_matches_numpy(uplo, trans, diag, n):
    import paper_2106_13402_b200.device as dv
    rng = np.random.default_rng(7)
    m = 1500
    # well-conditioned triangle (a unit diagonal with O(1) off-diagonal entries
    # has an inverse of size ~1e20 and no reference digits to compare)
    a = rng.standard_normal((n, n)) * (0.5 / np.sqrt(n)) + np.eye(n)
    b = rng.standard_normal((m, n))
    ref = np.array(b, order="F")
    NumpyOps().trsm_right(uplo, trans, diag, a, ref)
    db = _dm(b)
    dv.trsm_right(uplo, trans, diag, _dm(a), db)
    assert np.abs(db.to_numpy() - ref).max() < 1e-11 * np.abs(ref).max()


def _to_host(out):
    return {k: v.to_numpy() for k, v in out.items()}


@pytest.mark.parametrize("q,chunk", [(0, None), (1, None), (1, 500), (2, 700)])
def test_sharded_single_rank_device(q, chunk):
    from paper_2106_13402_b200.sharded import Comm, power_urv_sharded
    a, g = _case(2400, 96, 21 + q)
    out = _to_host(power_urv_sharded(_dm(a), _dm(g), q, Comm(), chunk_rows=chunk))
    _check(out, orc.power_urv(a, q, g), a)


@pytest.mark.parametrize("world,chunk", [(2, None), (3, 300), (4, None)])
def test_sharded_thread_ranks_device(world, chunk):
    import torch
    from paper_2106_13402_b200.sharded import ThreadComm, power_urv_sharded
    q = 1
    a, g = _case(2400, 96, 31 + world)
    rows = np.array_split(np.arange(a.shape[0]), world)
    hub = ThreadComm.make(world)
    results, errors = [None] * world, []

    def run(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = ThreadComm(hub, r, st)
                out = power_urv_sharded(_dm(a[rows[r]]), _dm(g), q, comm, chunk_rows=chunk)
                st.synchronize()
                results[r] = _to_host(out)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            hub.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    out = dict(results[0])
    out["Uy"] = np.vstack([results[r]["Uy"] for r in range(world)])
    for r in range(1, world):
        for k in ("Ut", "R", "Vy", "Vt"):
            assert np.array_equal(results[r][k], results[0][k])
    _check(out, orc.power_urv(a, q, g), a)


def test_tsqr_odd_row_chunks_match_device_driver():
    """Row chunks of odd height at odd offsets inside one buffer (the C4 P=1
    leaves: 524288 rows -> 74899/74898-row chunks): every chunk's QR must leave
    its neighbours untouched, so the chunked path gives the device driver's R."""
    import torch
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import dempty
    from paper_2106_13402_b200.sharded import Comm, power_urv_sharded
    m, n = 74898, 512
    a = dempty(m, n)
    a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(40))
    g = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(4)))
    run = dv.PowerUrvRun(m, n, 1)
    run.run(a, g)
    d_dev = torch.diagonal(run.R.tensor()[:n, :n]).abs()
    res = power_urv_sharded(a, g, 1, Comm(), chunk_rows=37449)
    d_sh = torch.diagonal(res["R"].tensor()).abs()
    assert ((d_sh - d_dev).abs().max() / d_dev.max()).item() < 1e-13
