import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dfrom_numpy, dempty
from paper_2106_13402_b200.sharded import tsqr, Comm, DeviceOps
rng = np.random.default_rng(0)
ops = DeviceOps()
def chk(label, m, n, chunk):
    a = rng.standard_normal((m, n))
    q, r = tsqr(dfrom_numpy(a), Comm(), ops, chunk_rows=chunk)
    Q = q.to_numpy(); R = r.to_numpy()
    rec = np.abs(Q @ R - a).max() / np.abs(a).max()
    orth = np.abs(Q.T @ Q - np.eye(n)).max()
    print(f"{label:28s} m={m} n={n} chunk={chunk}: recon {rec:.1e} orth {orth:.1e}", flush=True)
chk("even chunks", 2400, 96, 700)
chk("odd m", 2401, 96, 700)
chk("odd chunk heights", 2403, 96, 601)
chk("big odd", 9001, 300, 2250)
# single ops at odd offsets
a = rng.standard_normal((701, 300)); big = dfrom_numpy(np.vstack([rng.standard_normal((3, 300)), a]))
sub = big.sub(3, 0, 701, 300)
Y, T = dv.geqrf(sub); R = np.triu(sub.to_numpy()[:300])
print("geqrf odd offset |diag R| vs numpy:", np.abs(np.abs(np.diag(R)) - np.abs(np.diag(np.linalg.qr(a)[1]))).max())
