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


# ---------------------------------------------------------------------------
# product path: utv_powerurv_sharded_f64 (csrc/tsqr.cu) with the collectives
# inside libutvb200 (csrc/comm.cu)
# ---------------------------------------------------------------------------

def _run_native_group(a, g, q, world, chunk=None):
    import torch
    from paper_2106_13402_b200.sharded import NativeComm, power_urv_sharded_native
    rows = np.array_split(np.arange(a.shape[0]), world)
    comms = NativeComm.local_group(world)
    results, errors = [None] * world, []

    def run(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out = power_urv_sharded_native(_dm(a[rows[r]]), _dm(g), q, comms[r], chunk_rows=chunk)
                st.synchronize()
                results[r] = _to_host(out)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        c.close()
    assert not errors, errors
    out = dict(results[0])
    out["Uy"] = np.vstack([results[r]["Uy"] for r in range(world)])
    for r in range(1, world):       # replicated outputs agree bitwise across ranks
        for k in ("Ut", "R", "Vy", "Vt"):
            assert np.array_equal(results[r][k], results[0][k]), k
    return out


@pytest.mark.parametrize("q,chunk", [(0, None), (1, None), (1, 500), (2, 700)])
def test_native_sharded_single_rank(q, chunk):
    a, g = _case(2400, 96, 21 + q)
    out = _run_native_group(a, g, q, 1, chunk)
    _check(out, orc.power_urv(a, q, g), a)


@pytest.mark.parametrize("world,chunk,q", [(2, None, 1), (3, 300, 1), (4, None, 2), (2, 260, 0)])
def test_native_sharded_local_group(world, chunk, q):
    a, g = _case(2400, 96, 31 + world)
    out = _run_native_group(a, g, q, world, chunk)
    _check(out, orc.power_urv(a, q, g), a)


def test_native_sharded_nccl_one_rank():
    """The NCCL backend of the C-ABI entry (1-rank communicator on the one
    B200 the box has) against the oracle."""
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200.sharded import NativeComm, power_urv_sharded_native
    if not _lib.load().utv_comm_nccl_available():
        pytest.fail("libnccl could not be loaded")
    comm = NativeComm.nccl_single()
    assert (comm.rank, comm.size) == (0, 1)
    a, g = _case(1800, 80, 77)
    out = _to_host(power_urv_sharded_native(_dm(a), _dm(g), 1, comm, chunk_rows=600))
    comm.close()
    _check(out, orc.power_urv(a, 1, g), a)


def test_native_nccl_bootstrap_through_torch_distributed():
    """NativeComm.nccl(): unique id shipped by torch.distributed (world 1,
    127.0.0.1 rendezvous); plus TorchComm over NCCL with device DMat
    payloads driving the Python mirror of the schedule."""
    import os

    import torch
    import torch.distributed as dist
    from paper_2106_13402_b200.sharded import (NativeComm, TorchComm, power_urv_sharded,
                                                 power_urv_sharded_native)
    from tests.test_sharded_cpu import _free_port
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = NativeComm.nccl()
        a, g = _case(1200, 64, 78)
        ref = orc.power_urv(a, 2, g)
        _check(_to_host(power_urv_sharded_native(_dm(a), _dm(g), 2, comm)), ref, a)
        comm.close()
        _check(_to_host(power_urv_sharded(_dm(a), _dm(g), 2, TorchComm())), ref, a)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 3])
def test_local_group_collectives(world):
    import torch
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200.sharded import NativeComm
    lib = _lib.load()
    comms = NativeComm.local_group(world)
    cnt = 1001
    bufs = [torch.arange(cnt, dtype=torch.float64, device="cuda") * (r + 1) for r in range(world)]
    gat = [torch.empty(world * cnt, dtype=torch.float64, device="cuda") for _ in range(world)]
    bc = [torch.full((cnt,), float(r), dtype=torch.float64, device="cuda") for r in range(world)]
    errs = []

    def run(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            h, sp = comms[r].handle, st.cuda_stream
            src = bufs[r].clone()
            rc = [lib.utv_comm_allgather_f64(h, src.data_ptr(), gat[r].data_ptr(), cnt, sp),
                  lib.utv_comm_allreduce_sum_f64(h, bufs[r].data_ptr(), cnt, sp),
                  lib.utv_comm_broadcast_f64(h, bc[r].data_ptr(), cnt, world - 1, sp)]
            st.synchronize()
            if any(rc):
                errs.append(rc)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    for c in comms:
        c.close()
    assert not errs, errs
    base = torch.arange(cnt, dtype=torch.float64, device="cuda")
    tot = sum(range(1, world + 1))
    for r in range(world):
        assert torch.equal(bufs[r], base * tot)
        assert torch.equal(gat[r], torch.cat([base * (p + 1) for p in range(world)]))
        assert torch.equal(bc[r], torch.full((cnt,), float(world - 1), dtype=torch.float64,
                                             device="cuda"))


def test_native_matches_python_schedule_bitwise_r():
    """The C++ driver and the Python mirror run the same schedule on the same
    kernels: |diag R| agree to roundoff of the split reconstruction."""
    from paper_2106_13402_b200.sharded import Comm, power_urv_sharded
    a, g = _case(3000, 128, 5)
    nat = _run_native_group(a, g, 1, 2, 800)
    py = _to_host(power_urv_sharded(_dm(a), _dm(g), 1, Comm(), chunk_rows=800))
    assert np.abs(np.abs(np.diag(nat["R"])) - np.abs(np.diag(py["R"]))).max() < 1e-12 * np.abs(py["R"]).max()


@pytest.mark.parametrize("m,n", [(80000, 64), (152000, 40)])
def test_geqrf_taller_than_panel_limit(m, n):
    """geqrf beyond the fused panel kernel's row limit (utv_dgeqrf_rows_max)
    goes through the TSQR + Householder reconstruction: Y, Twy and R match
    the oracle's hqr_full (qr.py:71-100)."""
    import paper_2106_13402_b200.device as dv
    assert m > dv.geqrf_rows_max()
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, n)) * np.logspace(0, -6, n)
    y_ref, t_ref, r_ref = orc.householder_qr(np.asfortranarray(a))
    d = _dm(a)
    y, t = dv.geqrf(d)
    r = d.to_numpy()
    scale = np.abs(r_ref).max()
    assert np.abs(r - r_ref).max() < 1e-11 * scale
    assert np.abs(y.to_numpy() - y_ref).max() < 1e-9
    assert np.abs(t.to_numpy() - t_ref).max() < 1e-9


def test_power_urv_taller_than_panel_limit():
    """The public single-GPU power_urv_from_sample on a matrix taller than the
    panel kernel's limit (previously a generic UtvError)."""
    import paper_2106_13402_b200 as pk
    m, n = 90000, 48
    a, g = _case(m, n, 91)
    f = pk.power_urv_from_sample(a, 1, g)
    ref = orc.power_urv(a, 1, g)
    _check({"R": f.R[:n], "Ut": f.Uq.Twy, "Uy": f.Uq.Y, "Vy": f.Vq.Y, "Vt": f.Vq.Twy}, ref, a)
