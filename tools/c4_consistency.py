"""|diag R| of powerURV q=1 on a tall Gaussian A: device driver (utv_powerurv_f64)
vs the row-sharded SPMD path with P = 1, 2 emulated ranks (and chunked TSQR)."""
import sys
import threading
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2106_13402_b200 as pk
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200 import _lib
from paper_2106_13402_b200._lib import dempty
from paper_2106_13402_b200.sharded import Comm, ThreadComm, power_urv_sharded

m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
a = dempty(m, n)
a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(40))
g = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(4)))
run = dv.PowerUrvRun(m, n, 1)
run.run(a, g)
torch.cuda.synchronize()
d_dev = torch.diagonal(run.R.tensor()[:n, :n]).abs().cpu().numpy()


def sharded(P, chunk=None):
    bounds = np.linspace(0, m, P + 1).astype(int)
    if P == 1:
        res = power_urv_sharded(a, g, 1, Comm(), chunk_rows=chunk)
        return torch.diagonal(res["R"].tensor()).abs().cpu().numpy()
    hub = ThreadComm.make(P)
    out = [None] * P

    def runr(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res = power_urv_sharded(a.sub(int(bounds[r]), 0, int(bounds[r + 1] - bounds[r]), n), g, 1,
                                    ThreadComm(hub, r, st), chunk_rows=chunk)
            st.synchronize()
            out[r] = torch.diagonal(res["R"].tensor()).abs().cpu().numpy()
    th = [threading.Thread(target=runr, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join() for t in th]
    return out[0]


for label, d in [("sharded P=1", sharded(1)), ("sharded P=1 chunk m/4", sharded(1, m // 4)),
                 ("sharded P=2", sharded(2)), ("sharded P=4", sharded(4))]:
    print(f"{label:24s} max rel diff vs device driver {np.abs(d - d_dev).max() / d_dev.max():.2e}", flush=True)
