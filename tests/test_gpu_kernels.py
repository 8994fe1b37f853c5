"""GPU parity of the individual kernels through the C ABI (K1 GEMM, K3/K4
geqrf, K2 larfb, K5 orgqr, K6 Jacobi SVD) against the reference's golden
vectors and numpy fp64."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dv():
    import paper_2106_13402_b200.device as dv
    return dv


def _dm(a):
    from paper_2106_13402_b200._lib import dfrom_numpy
    return dfrom_numpy(a)


GEMM_SHAPES = [
    (1, 1, 1), (7, 5, 3), (128, 128, 16), (129, 130, 17), (300, 64, 1000),
    (64, 256, 4096), (256, 256, 8192), (1000, 300, 77), (513, 257, 255), (33, 700, 2048),
]


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_dgemm_matches_numpy(dv, ta, tb, shape):
    m, n, k = shape
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    C0 = rng.standard_normal((m, n))
    ref = 1.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.5 * C0
    C = _dm(C0)
    dv.gemm("T" if ta else "N", "T" if tb else "N", 1.5, _dm(A), _dm(B), beta=-0.5, C=C)
    out = C.to_numpy()
    # forward error bound of a dot product of length k
    bound = 4 * k * np.finfo(float).eps * (np.abs(A).max() * np.abs(B).max() * 1.5 + 1)
    assert np.abs(out - ref).max() <= bound * max(1.0, np.sqrt(k))


def test_dgemm_unaligned_submatrices(dv):
    """Odd row offsets (pointer not 16B aligned) and ragged edges."""
    from paper_2106_13402_b200._lib import DMat, check, load, stream_ptr, workspace
    rng = np.random.default_rng(5)
    big = rng.standard_normal((301, 260))
    Bm = rng.standard_normal((260, 90))
    dA, dB = _dm(big), _dm(Bm)
    for (r0, c0, m, k) in [(1, 3, 200, 150), (3, 0, 77, 257), (0, 1, 300, 33)]:
        sub = DMat(dA.t, m, k, dA.ld)
        ptr = dA.at(r0, c0)
        C = _dm(np.zeros((m, 90)))
        lib = load()
        lw = lib.utv_dgemm_bufsize(m, 90, k)
        ws = workspace(lw)
        check(lib.utv_dgemm(b"N", b"N", m, 90, k, 1.0, ptr, sub.ld, dB.ptr, dB.ld, 0.0, C.ptr, C.ld,
                            ws.data_ptr(), lw, stream_ptr()), "dgemm")
        ref = big[r0:r0 + m, c0:c0 + k] @ Bm[:k]
        assert np.abs(C.to_numpy() - ref).max() < 1e-12 * k


def test_dgemm_rejects_odd_ld(dv):
    from paper_2106_13402_b200._lib import load
    lib = load()
    st = lib.utv_dgemm(b"N", b"N", 4, 4, 4, 1.0, 0, 5, 0, 4, 0.0, 0, 4, 0, 0, 0)
    assert st == -8


HQR = ["hqr_eye4", "hqr_col34", "hqr_rand100x60", "hqr_rankdef40x24", "hqr_collinear6x3",
       "hqr_square33"]


@pytest.mark.parametrize("name", HQR)
def test_geqrf_matches_reference_golden(dv, golden, name):
    g = golden(name)
    d = _dm(g["A"])
    Y, T = dv.geqrf(d)
    scale = max(1.0, np.abs(g["A"]).max())
    assert np.abs(Y.to_numpy() - g["Y"]).max() <= 1e-12
    assert np.abs(T.to_numpy() - g["Twy"]).max() <= 1e-12
    R = d.to_numpy()
    assert np.abs(R - g["R"]).max() <= 1e-12 * scale
    assert not np.tril(R, -1).any()


@pytest.mark.parametrize("shape", [(500, 256), (2048, 256), (1500, 700), (640, 33), (9000, 64)])
def test_geqrf_matches_oracle_large(dv, shape):
    from oracle import utv_oracle as orc
    m, n = shape
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n))
    d = _dm(A)
    Y, T = dv.geqrf(d)
    y, t, r = orc.householder_qr(A) if m * n <= 600_000 else (None, None, None)
    Yd, Td, Rd = Y.to_numpy(), T.to_numpy(), d.to_numpy()
    if y is not None:
        assert np.abs(Yd - y).max() < 1e-11
        assert np.abs(Td - t).max() < 1e-11
        assert np.abs(Rd - r).max() < 1e-11 * np.abs(A).max() * np.sqrt(m)
    # reconstruction through the compact WY form
    Q = orc.wy_materialize(Yd, Td, n)
    assert np.linalg.norm(Q @ Rd[:n] - A) / np.linalg.norm(A) < 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) < 1e-13 * max(m, n)


def test_larfb_orgqr_match_reference_golden(dv, golden):
    g = golden("applyq_50x30")
    d = _dm(g["A"])
    Y, T = dv.geqrf(d)
    for side, trans, key, B in [("L", False, "left", g["BL"]), ("L", True, "left_t", g["BL"]),
                                ("R", False, "right", g["BR"]), ("R", True, "right_t", g["BR"])]:
        dB = _dm(B)
        dv.larfb(side, trans, Y, T, dB)
        assert np.abs(dB.to_numpy() - g[key]).max() < 1e-13, key
    assert np.abs(dv.orgqr(Y, T, 50).to_numpy() - g["Q"]).max() < 1e-14
    assert np.abs(dv.orgqr(Y, T, 30).to_numpy() - g["Q30"]).max() < 1e-14


SVD = ["svd_diag321", "svd_rand20", "svd_zero5", "svd_upper64"]


@pytest.mark.parametrize("name", SVD)
def test_gesvj_matches_reference_golden(dv, golden, name):
    g = golden(name)
    sig, U, V, st = dv.gesvj(_dm(g["A"]))
    n = g["A"].shape[0]
    assert int(st.cpu().item()) > 0
    s = sig.cpu().numpy()[:n]
    assert np.abs(s - g["sigma"]).max() <= 1e-13 * max(1.0, g["sigma"].max())
    # singular vectors are determined to ~eps*||A||/gap (Davis-Kahan); compare
    # each pair against that bound instead of a flat 1e-12
    sg = g["sigma"]
    gap = np.minimum(np.abs(np.diff(sg, prepend=np.inf)), np.abs(np.diff(sg, append=-np.inf)))
    tol = np.minimum(2.0, 1e-12 + 64 * np.finfo(float).eps * max(sg.max(), 1e-300) / np.maximum(gap, 1e-300))
    # U = A V / sigma: a column whose sigma sits at the roundoff floor
    # (svd_upper64: sigma_64 = 4e-16 * sigma_1) is undetermined to O(1)
    tol_u = np.minimum(2.0, tol + 64 * np.finfo(float).eps * max(sg.max(), 1e-300) / np.maximum(sg, 1e-300))
    assert np.all(np.abs(U.to_numpy() - g["U"]).max(axis=0) <= tol_u)
    assert np.all(np.abs(V.to_numpy() - g["V"]).max(axis=0) <= tol)


@pytest.mark.parametrize("n", [1, 2, 17, 128, 200, 256, 384])
def test_gesvj_random_upper(dv, n):
    from oracle import utv_oracle as orc
    rng = np.random.default_rng(n)
    A = np.triu(rng.standard_normal((n, n)))
    A[:, :n // 3] *= 1e-4
    sig, U, V, st = dv.gesvj(_dm(A))
    assert int(st.cpu().item()) > 0
    u, s, v = orc.svd_signed(A)
    sd = sig.cpu().numpy()[:n]
    assert np.all(np.abs(sd - s) <= 1e-10 * s + 16 * orc.EPS * s.max())
    Ud, Vd = U.to_numpy(), V.to_numpy()
    assert np.linalg.norm(Ud.T @ Ud - np.eye(n)) < 1e-12 * n
    assert np.linalg.norm(Vd.T @ Vd - np.eye(n)) < 1e-12 * n
    assert np.linalg.norm(Ud @ np.diag(sd) @ Vd.T - A) < 1e-13 * np.linalg.norm(A) * np.sqrt(n)
    # singular vectors match LAPACK's (sign rule) where the gap is healthy
    gap = np.minimum(np.abs(np.diff(s, prepend=np.inf)), np.abs(np.diff(s, append=-np.inf)))
    ok = gap > 1e-3 * s.max()
    assert np.abs(Vd[:, ok] - v[:, ok]).max() < 1e-9


def test_gesvj_rank_deficient_completes_u(dv):
    rng = np.random.default_rng(3)
    n = 64
    A = np.triu(rng.standard_normal((n, n)))
    A[:, 40:] = 0.0
    A[40:, :] = 0.0
    sig, U, V, st = dv.gesvj(_dm(A))
    Ud = U.to_numpy()
    assert np.linalg.norm(Ud.T @ Ud - np.eye(n)) < 1e-12 * n
    assert np.all(sig.cpu().numpy()[40:] == 0.0)


@pytest.mark.parametrize("ta,tb", [(True, False), (True, True), (False, True), (False, False)])
@pytest.mark.parametrize("ra,rb", [(1, 0), (0, 1), (1, 1), (3, 2)])
def test_dgemm_parity_offsets_all_ops(dv, ta, tb, ra, rb):
    """Every op combination with odd/even sub-matrix row offsets on both operands."""
    from paper_2106_13402_b200._lib import check, load, stream_ptr, workspace
    rng = np.random.default_rng(ra * 10 + rb)
    m, n, k = 150, 70, 300
    Abig = rng.standard_normal((400, 400))
    Bbig = rng.standard_normal((400, 400))
    A = Abig[ra:ra + (k if ta else m), 2:2 + (m if ta else k)]
    B = Bbig[rb:rb + (n if tb else k), 5:5 + (k if tb else n)]
    dA, dB = _dm(Abig), _dm(Bbig)
    C = _dm(np.zeros((m, n)))
    lib = load()
    lw = lib.utv_dgemm_bufsize(m, n, k)
    ws = workspace(lw)
    check(lib.utv_dgemm(b"T" if ta else b"N", b"T" if tb else b"N", m, n, k, 1.0, dA.at(ra, 2), dA.ld,
                        dB.at(rb, 5), dB.ld, 0.0, C.ptr, C.ld, ws.data_ptr(), lw, stream_ptr()), "dgemm")
    ref = (A.T if ta else A) @ (B.T if tb else B)
    assert np.abs(C.to_numpy() - ref).max() < 1e-12 * k


@pytest.mark.parametrize("M,N,K,ta,tb,beta", [(20001, 300, 256, "N", "N", 1.0), (20001, 44, 256, "N", "T", 1.0),
                                               (20003, 200, 512, "N", "N", 1.0), (3001, 300, 64, "T", "N", 1.0),
                                               (20001, 44, 256, "N", "N", 0.0)])
def test_gemm_writes_stay_inside_the_view(M, N, K, ta, tb, beta):
    """C is a view on the top rows of a taller buffer (a TSQR row chunk): no
    kernel may write below it — a TMA store of an odd-M tile once did (its
    16-byte granule covered row M)."""
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dempty
    big = dempty(M + 64, N)
    big.t.normal_()
    C = big.sub(0, 0, M, N)
    A = dempty(K if ta == "T" else M, M if ta == "T" else K)
    A.t.normal_()
    B = dempty(N if tb == "T" else K, K if tb == "T" else N)
    B.t.normal_()
    view = lambda d: d.tensor().T
    below = view(big)[M:M + 64, :N].clone()
    c0 = view(C)[:M, :N].clone()
    a, b = view(A)[:A.rows, :A.cols], view(B)[:B.rows, :B.cols]
    ref = -((a.T if ta == "T" else a) @ (b.T if tb == "T" else b)) + beta * c0
    dv.gemm(ta, tb, -1.0, A, B, beta, C)
    torch.cuda.synchronize()
    assert torch.equal(view(big)[M:M + 64, :N], below)
    assert ((view(C)[:M, :N] - ref).abs().max() / ref.abs().max()).item() < 1e-13


@pytest.mark.parametrize("rows,cols", [(20001, 300), (37449, 300), (20001, 257), (9001, 600), (513, 512)])
def test_geqrf_writes_stay_inside_the_view(rows, cols):
    """geqrf on the top rows of a taller buffer (a TSQR chunk) leaves the rows
    below untouched and still factors its view exactly (thin Q R = A)."""
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dempty
    view = lambda d: d.tensor().T
    big = dempty(2 * rows + 1, cols)
    big.t.normal_()
    sub = big.sub(0, 0, rows, cols)
    A = view(sub)[:rows, :cols].clone()
    below = view(big)[rows:2 * rows + 1, :cols].clone()
    Y, T = dv.geqrf(sub)
    torch.cuda.synchronize()
    assert torch.equal(view(big)[rows:2 * rows + 1, :cols], below)
    Yd, Td, Rd = view(Y)[:rows, :cols], view(T)[:cols, :cols], torch.triu(view(sub)[:cols, :cols])
    E = torch.zeros(rows, cols, device="cuda", dtype=torch.float64)
    E[:cols] = torch.eye(cols, device="cuda", dtype=torch.float64)
    Q = E - Yd @ (Td @ Yd[:cols].T)
    assert ((Q @ Rd - A).abs().max() / A.abs().max()).item() < 1e-13


def test_fused_splitk_matches_reduce_kernel_bitwise(tmp_path):
    """The fused split-K epilogue (per-tile turn counters, splits summed in
    split order, last split applies alpha/beta) gives the same bits as the
    separate fixed-order reduce kernel (UTV_SPLITK_FUSE_MAX=0)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for tag, env in (("fused", {}), ("reduce", {"UTV_SPLITK_FUSE_MAX": "0"})):
        path = str(tmp_path / f"{tag}.npz")
        subprocess.run([sys.executable, os.path.join(root, "tools", "splitk_bits.py"), path],
                       check=True, env={**os.environ, **env}, timeout=600)
        outs[tag] = np.load(path)
    for key in outs["fused"].files:
        assert np.array_equal(outs["fused"][key], outs["reduce"][key]), key


@pytest.mark.parametrize("m,n,q", [(1500, 1024, 1), (1300, 700, 2), (900, 900, 0)])
def test_powerurv_progressive_columns_match_the_plain_driver(m, n, q):
    """utv_powerurv_f64_cols: per-panel progress events for R / Uq.Y and
    Uq.Twy (merged on the low-priority stream while the final QR runs) —
    every event completes and the outputs equal the plain driver's bitwise."""
    import torch
    import paper_2106_13402_b200.device as dv
    rng = np.random.default_rng(m + n)
    a = _dm(rng.standard_normal((m, n)) * np.logspace(0, -6, n))
    g = _dm(rng.standard_normal((n, n)))
    ref = dv.PowerUrvRun(m, n, q)
    ref.run(a, g)
    run = dv.PowerUrvRun(m, n, q)
    ngrp = -(-n // 256)
    r_evs = [torch.cuda.Event() for _ in range(ngrp)]
    t_evs = [torch.cuda.Event() for _ in range(ngrp)]
    run.run_cols(a, g, None, r_events=r_evs, t_events=t_evs)
    for e in r_evs + t_evs:
        e.synchronize()
    torch.cuda.synchronize()
    for k in ("Uy", "Ut", "R", "Vy", "Vt"):
        x, y = getattr(run, k).to_numpy(), getattr(ref, k).to_numpy()
        assert np.array_equal(x, y), k
    if q >= 1:          # the Yhat0 form gives the same factors
        yh = dv.gemm("N", "N", 1.0, a, g)
        run2 = dv.PowerUrvRun(m, n, q)
        run2.run_cols(a, None, yh)
        torch.cuda.synchronize()
        assert np.abs(run2.R.to_numpy() - ref.R.to_numpy()).max() < 1e-12 * np.abs(ref.R.to_numpy()).max()


@pytest.mark.parametrize("groups", [[1, 3, 4, 4], [2, 2, 5], [1] * 12])
def test_randutv_step_ranges_with_carried_svd_are_bitwise_one_call(groups):
    """utv_randutv_basic_steps_carry_f64 over host-fed groups (the last
    step's SVD left in flight into the next group) gives exactly the bits
    of one utv_randutv_basic_f64 call; columns < (j1-1) b are final when a
    carrying group returns."""
    import torch

    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import dempty, deye, dfrom_numpy
    m, n, b, q = 700, 660, 64, 2
    steps = -(-n // b)
    rng = np.random.default_rng(17)
    a = rng.standard_normal((m, n)) * np.logspace(0, -6, n)[None, :]
    blocks = [rng.standard_normal((m - i * b, b)) for i in range(steps - 1)]
    G = dv.stage_randutv_blocks(blocks, b)
    run = dv.RandUtvRun(m, n, b, q)
    T1, U1, V1 = dfrom_numpy(a), deye(m), deye(n)
    run.run(T1, U1, V1, G)
    ref = [x.to_numpy() for x in (T1, U1, V1)] + [run.errsq.cpu().numpy()]
    run2 = dv.RandUtvRun(m, n, b, q)
    T2, U2, V2 = dfrom_numpy(a), deye(m), deye(n)
    lib = _lib.load()
    offs = np.concatenate([[0], np.cumsum([m - i * b for i in range(steps - 1)])]).astype(int)
    j0 = 0
    for gi, w in enumerate(groups + [steps]):
        j1 = min(steps, j0 + w)
        if j0 >= j1:
            break
        carry = (1 if gi > 0 else 0) | (2 if j1 < steps else 0)
        gptr = G.at(0, int(offs[min(j0, steps - 1)]))
        _lib.check(lib.utv_randutv_basic_steps_carry_f64(
            j0, j1, carry, m, n, b, q, T2.ptr, T2.ld, U2.ptr, U2.ld, V2.ptr, V2.ld, gptr, G.ld,
            run2.errsq.data_ptr(), None, run2.status.data_ptr(), run2.ws.data_ptr(), run2.lw,
            _lib.stream_ptr()), "steps_carry")
        if j1 < steps:       # the carried step's columns are not final yet, the earlier ones are
            torch.cuda.synchronize()
            fin = (j1 - 1) * b
            assert np.array_equal(U2.to_numpy()[:, :fin], ref[1][:, :fin])
            assert np.array_equal(V2.to_numpy()[:, :fin], ref[2][:, :fin])
        j0 = j1
    got = [x.to_numpy() for x in (T2, U2, V2)] + [run2.errsq.cpu().numpy()]
    for x, y in zip(got, ref):
        assert np.array_equal(x, y)
