"""Randomised DMMA GEMM stress against numpy: all ops, alpha/beta, odd/even
sub-matrix offsets on A, B and C, ragged shapes, multi-tile persistence."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2106_13402_b200._lib import check, load, stream_ptr, workspace, dfrom_numpy

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
lib = load()
bad = 0
shapes = [(80, 80, 80), (80, 48, 32), (256, 256, 256), (1000, 300, 77), (2000, 1500, 32),
          (129, 2000, 256), (3000, 3000, 64), (33, 4000, 1000), (16, 16, 4000), (4000, 16, 4000)]
for it in range(120):
    m, n, k = shapes[it % len(shapes)]
    ta, tb = bool(rng.integers(2)), bool(rng.integers(2))
    ra, rb, rc = [int(x) for x in rng.integers(0, 3, 3)]
    beta = [0.0, 1.0, -0.5][it % 3]
    alpha = [1.0, -1.0, 0.75][(it // 3) % 3]
    ar, ac = (k, m) if ta else (m, k)
    br, bc = (n, k) if tb else (k, n)
    Abig = rng.standard_normal((ar + 3, ac)); Bbig = rng.standard_normal((br + 3, bc)); Cbig = rng.standard_normal((m + 3, n))
    dA, dB, dC = dfrom_numpy(Abig), dfrom_numpy(Bbig), dfrom_numpy(Cbig)
    lw = lib.utv_dgemm_bufsize(m, n, k); ws = workspace(lw)
    check(lib.utv_dgemm(b"T" if ta else b"N", b"T" if tb else b"N", m, n, k, alpha, dA.at(ra, 0), dA.ld,
                        dB.at(rb, 0), dB.ld, beta, dC.at(rc, 0), dC.ld, ws.data_ptr(), lw, stream_ptr()), "dgemm")
    A = Abig[ra:ra + ar]; B = Bbig[rb:rb + br]
    ref = alpha * ((A.T if ta else A) @ (B.T if tb else B)) + beta * Cbig[rc:rc + m]
    out = dC.to_numpy()
    err = np.abs(out[rc:rc + m] - ref).max()
    # untouched rows outside the C block
    untouched = np.abs(np.delete(out, np.s_[rc:rc + m], axis=0) - np.delete(Cbig, np.s_[rc:rc + m], axis=0)).max() if m + 3 > m else 0
    ok = err < 1e-12 * k and untouched == 0
    if not ok:
        bad += 1
    print(f"{'OK ' if ok else 'BAD'} m={m} n={n} k={k} ta={ta} tb={tb} ra={ra} rb={rb} rc={rc} a={alpha} b={beta} err={err:.2e} untouched={untouched:.1e}", flush=True)
print("bad", bad)
