"""CPU tests of the row-sharded powerURV orchestration:
world_size 1 and 2 over torch.distributed/gloo, local factorisations by the
numpy test backend (tests/numpy_ops.py), checked against the oracle's
single-process power_urv (pinned to the reference's golden vectors)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import utv_oracle as orc


def _case(m, n, seed):
    rng = np.random.default_rng(seed)
    a, _ = orc.decay_matrix(n, 1e-5, seed=seed, m=m)
    g = orc.draw_gaussian(orc.gaussian_stream(seed + 1), n, n)
    return a, g


def _check(out, ref, a):
    n = a.shape[1]
    anorm = np.linalg.norm(a, 2)
    tol = 1e-10 * np.abs(np.diag(ref["R"])) + 16 * orc.EPS * anorm
    assert np.all(np.abs(np.diag(out["R"]) - np.diag(ref["R"])) <= tol)
    assert np.abs(out["R"] - ref["R"][:n]).max() < 1e-9 * anorm
    assert np.abs(out["Ut"] - ref["Ut"]).max() < 1e-8
    assert np.abs(out["Uy"] - ref["Uy"]).max() < 1e-8
    assert np.abs(out["Vy"] - ref["Vy"]).max() < 1e-9
    assert np.abs(out["Vt"] - ref["Vt"]).max() < 1e-9


def test_row_chunks():
    from paper_2106_13402_b200.sharded import _row_chunks
    assert _row_chunks(100, 10, 200) == [(0, 100)]
    ch = _row_chunks(1000, 50, 300)
    assert sum(c[1] for c in ch) == 1000 and all(50 <= c[1] <= 300 for c in ch)
    assert [c[0] for c in ch] == [0, 250, 500, 750]
    with pytest.raises(ValueError):
        _row_chunks(1000, 400, 300)


@pytest.mark.parametrize("chunk", [None, 150])
@pytest.mark.parametrize("q", [0, 1, 2])
def test_sharded_single_rank_numpy(q, chunk):
    from paper_2106_13402_b200.sharded import Comm, power_urv_sharded
    from tests.numpy_ops import NumpyOps
    a, g = _case(600, 40, 3 + q)
    out = power_urv_sharded(np.asfortranarray(a), g, q, Comm(), NumpyOps(), chunk_rows=chunk)
    _check(out, orc.power_urv(a, q, g), a)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, chunk, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_13402_b200.sharded import TorchComm, power_urv_sharded
    from tests.numpy_ops import NumpyOps
    a, g = _case(600, 40, 11 + q)
    rows = np.array_split(np.arange(a.shape[0]), world)[rank]
    out = power_urv_sharded(np.asfortranarray(a[rows]), g, q, TorchComm(), NumpyOps(), chunk_rows=chunk)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("q,chunk", [(1, None), (2, 120)])
def test_sharded_gloo_world2(tmp_path, q, chunk):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), q, chunk, str(tmp_path)), nprocs=world, join=True)
    parts = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]
    a, g = _case(600, 40, 11 + q)
    out = dict(parts[0])
    out["Uy"] = np.vstack([p["Uy"] for p in parts])
    for r in range(1, world):          # replicated outputs agree bitwise across ranks
        for k in ("Ut", "R", "Vy", "Vt"):
            assert np.array_equal(parts[r][k], parts[0][k])
    _check(out, orc.power_urv(a, q, g), a)
