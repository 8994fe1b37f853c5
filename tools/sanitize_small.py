"""Small-shape runs of every kernel family for compute-sanitizer."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2106_13402_b200 as pk
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dfrom_numpy
from oracle import utv_oracle as orc
rng = np.random.default_rng(0)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "gemm"):
    for (m, n, k, ta, tb) in [(130, 70, 45, "N", "N"), (129, 257, 300, "T", "T"), (300, 20, 1000, "T", "N"), (64, 300, 16, "N", "T")]:
        A = rng.standard_normal((k, m) if ta == "T" else (m, k)); B = rng.standard_normal((n, k) if tb == "T" else (k, n))
        C = dfrom_numpy(rng.standard_normal((m, n)))
        dv.gemm(ta, tb, 1.0, dfrom_numpy(A), dfrom_numpy(B), 0.5, C)
        A32 = dfrom_numpy(A, dtype=torch.float32); B32 = dfrom_numpy(B, dtype=torch.float32)
        dv.sgemm_tf32x3(ta, tb, 1.0, A32, B32)
if what in ("all", "qr"):
    a = dfrom_numpy(rng.standard_normal((700, 300))); dv.geqrf(a)
    a = dfrom_numpy(rng.standard_normal((96, 40))); dv.geqrf(a)
if what in ("all", "svd"):
    dv.gesvj(dfrom_numpy(np.triu(rng.standard_normal((70, 70)))))
    dv.gesvj(dfrom_numpy(rng.standard_normal((256, 256)) * np.logspace(0, -4, 256)))   # 4-CTA clusters
    dv.gesvj(dfrom_numpy(rng.standard_normal((20, 20))))
if what in ("all", "qrcp"):
    pk.hqrcp(rng.standard_normal((300, 200)))
if what in ("all", "rutv"):
    a, _ = orc.decay_matrix(200, 1e-5, seed=3)
    pk.randutv_basic(a, 48, 1, pk.RngStream(1), record_trailing=True)
    pk.randutv_boosted(a, 48, 1, 16, pk.RngStream(2))
    pk.randutv_basic(np.asfortranarray(a), 48, 1, pk.RngStream(1), dtype=np.float32)
if what in ("all", "purv"):
    a, _ = orc.decay_matrix(96, 1e-5, seed=4, m=300)
    pk.power_urv(a, 2, pk.RngStream(2))
    from paper_2106_13402_b200.sharded import Comm, power_urv_sharded
    power_urv_sharded(dfrom_numpy(a), dfrom_numpy(orc.draw_gaussian(orc.gaussian_stream(1), 96, 96)), 1, Comm(), chunk_rows=140)
if what in ("all", "lu"):
    q0, _ = np.linalg.qr(rng.standard_normal((900, 600)))
    dv.getrf_signed(dfrom_numpy(q0))
    t = np.eye(600) + rng.standard_normal((600, 600)) * 0.01
    for uplo, trans, diag in (("U", "N", "N"), ("L", "T", "U")):
        dv.trsm_right(uplo, trans, diag, dfrom_numpy(t), dfrom_numpy(rng.standard_normal((500, 600))))
if what in ("all", "purv_stream"):
    import paper_2106_13402_b200.powerurv as pu
    pu.STREAM_MIN_N = 64
    a, _ = orc.decay_matrix(200, 1e-5, seed=5, m=260)
    pk.power_urv(a, 1, pk.RngStream(3))
if what in ("all", "purv_overlap"):
    import paper_2106_13402_b200.powerurv as pu
    pu.STREAM_MIN_N = 64
    pu.OVERLAP_A_MIN_BYTES = 1 << 16
    a, _ = orc.decay_matrix(200, 1e-5, seed=6, m=260)
    pk.power_urv(a, 1, pk.RngStream(3))
torch.cuda.synchronize()
print("done", what)
