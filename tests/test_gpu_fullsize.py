"""Parity at BASELINE.json's full sizes through size-independent properties
(the CPU oracle cannot run there): reconstruction, orthogonality and the
e_k curve against the known spectrum, all computed in HBM with the device
metrics.  C3: randUTV b=256 q=2 on 16384^2 fp64; powerURV q=2 on 16384^2;
C5: fp32 randUTV b=512 q=2 on 32768^2 rank 2000."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _decay(n, seed):
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dempty
    gen = torch.Generator(device="cuda").manual_seed(seed)
    qs = []
    for _ in range(2):
        g = dempty(n, n)
        g.t.normal_(generator=gen)
        y, t = dv.geqrf(g)
        qs.append(dv.orgqr(y, t, n))
    d = np.maximum(np.exp(-(np.arange(n) / (n / 4.0)) ** 2), 1e-5)
    dd = torch.from_numpy(d).cuda()
    dv.diag_scale("R", dd, qs[1])
    return dv.gemm("N", "T", 1.0, qs[0], qs[1]), d


def test_randutv_c3_fullsize():
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200.metrics import (orthogonality_device, reconstruction_device,
                                               trailing_fro_curve_device)
    from paper_2106_13402_b200.randutv import randutv_basic_device
    n, b, q = 16384, 256, 2
    a, d = _decay(n, 30)
    t = dv.copy(a)
    g = dv.stage_randutv_blocks(pk.randutv.draw_sample_blocks(pk.RngStream(3), n, n, b), b)
    run, U, V = randutv_basic_device(t, b, q, g)
    assert (run.status.cpu().numpy() > 0).all()
    assert reconstruction_device(a, U, t, V) < 1e-13
    assert orthogonality_device(U) < 1e-11
    assert orthogonality_device(V) < 1e-11
    ek = trailing_fro_curve_device(t)
    tail = np.sqrt(np.cumsum((d ** 2)[::-1])[::-1])
    ey = tail[1:]                                   # Eckart-Young, rank k = 1..n-1
    assert np.all(ek >= ey * (1 - 1e-8) - 1e-12)
    assert np.mean(ek <= 2.0 * ey) > 0.95


def test_powerurv_fullsize():
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200.metrics import orthogonality_device, reconstruction_device
    from paper_2106_13402_b200.powerurv import power_urv_device
    n, q = 16384, 2
    a, d = _decay(n, 20)
    g = dv.from_numpy_any_order(np.asarray(pk.RngStream(2).standard_normal(n, n)))
    run = power_urv_device(a, g, q)
    U = dv.orgqr(run.Uy, run.Ut, n)
    V = dv.orgqr(run.Vy, run.Vt, n)
    assert reconstruction_device(a, U, run.R, V) < 1e-13
    assert orthogonality_device(U) < 1e-11
    assert orthogonality_device(V) < 1e-11
    r = np.abs(np.diag(run.R.to_numpy()))
    assert r.max() <= d[0] * (1 + 1e-10)            # |R_kk| <= ||A||_2 = sigma_1
    assert r[-1] >= d[-1] * (1 - 1e-6) * 0.1        # rank revealed down to the 1e-5 floor


def test_randutv_fp32_c5_fullsize():
    import torch
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200.randutv import randutv_basic_device32
    import bench
    n, r, b, q = 32768, 2000, 512, 2
    a = bench.make_rank_deficient_f32(n, r, 50)
    t = dv.DMat(a.t.clone(), a.rows, a.cols, a.ld) if hasattr(dv, "DMat") else None
    g = dv.stage_randutv_blocks(pk.randutv.draw_sample_blocks(pk.RngStream(5), n, n, b), b,
                                dtype=torch.float32)
    run, U, V = randutv_basic_device32(t, b, q, g)
    assert (run.status.cpu().numpy() > 0).all()
    # reconstruction ||A - U T V^T||_F / ||A||_F, evaluated in fp64 (DMMA
    # GEMMs on the fp32 factors promoted exactly) so the check itself adds
    # no fp32 error
    from paper_2106_13402_b200._lib import dempty
    del g, run
    torch.cuda.empty_cache()

    def f64(x):
        y = dempty(x.rows, x.cols)
        y.t[:x.cols, :x.rows].copy_(x.t[:x.cols, :x.rows])
        return y
    from paper_2106_13402_b200.metrics import orthogonality_device, reconstruction_device
    a64, u64 = f64(a), f64(U)
    del U
    t64 = f64(t)
    del t
    v64 = f64(V)
    del V
    torch.cuda.empty_cache()
    rel = reconstruction_device(a64, u64, t64, v64)
    print("C5 reconstruction", rel)
    assert rel < 1e-4
    # e_k (Frobenius, from T) against Eckart-Young of the known spectrum
    # (svd.py:85-100, bench.py:63-72; SURVEY §8c C5 criterion)
    from paper_2106_13402_b200.metrics import trailing_fro_curve_device
    e = trailing_fro_curve_device(t64)
    d = 10.0 ** (-3.0 * np.arange(r) / (r - 1))
    tail = np.sqrt(np.cumsum((d ** 2)[::-1])[::-1])            # ||d[k:]||_2, k = 0..r-1
    ey = np.concatenate([tail[1:], np.zeros(n - r)])[: n - 1]  # e_opt(k), k = 1..n-1
    fro = float(tail[0])
    slack = 1e-5 * fro                                         # fp32 sampling / storage noise
    assert np.all(e >= ey - slack), "e_k below the Eckart-Young floor"
    ks = np.arange(1, r)
    ratio = e[ks - 1] / ey[ks - 1]
    assert np.mean(ratio <= 2.0) >= 0.9, np.percentile(ratio, [50, 90, 99])
    assert e[r + b - 1:].max() < 1e-4 * fro                   # past the rank: fp32 noise
    print("C5 e_k/EY median", float(np.median(ratio)), "p90", float(np.percentile(ratio, 90)))
    # the trailing block past the rank is fp32 noise
    tt = t64.t[r + b:, r + b:n]
    assert (tt.norm() / a64.t[:n, :n].norm()).item() < 1e-4
    ou = orthogonality_device(u64) / np.sqrt(n)       # normalised
    print("C5 orthogonality(U)/sqrt(n)", ou)
    assert ou < 1e-4
