"""Stage timeline of the public power_urv e2e path at n=16384 (host clock):
draw, check+upload, device run, D2H tail. Mirrors powerurv.power_urv."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2106_13402_b200 as pk
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import AsyncD2H, dfrom_numpy
from paper_2106_13402_b200.matrix import check_matrix

n, q = 16384, 2
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
for rep in range(3):
    t = [("start", time.perf_counter())]
    rng = pk.RngStream(2)
    g = np.asarray(rng.standard_normal(n, n))
    t.append(("draw G", time.perf_counter()))
    a_dev = dfrom_numpy(check_matrix(a, finite=False))
    torch.cuda.synchronize()
    t.append(("H2D A", time.perf_counter()))
    g_dev = dv.from_numpy_any_order(g)
    torch.cuda.synchronize()
    t.append(("H2D G", time.perf_counter()))
    run = dv.PowerUrvRun(n, n, q)
    vq_ev = torch.cuda.Event()
    run.run(a_dev, g_dev, vq_event=vq_ev)
    vy, vt = np.empty((n, n), order="F"), np.empty((n, n), order="F")
    uy, ut, r = np.empty((n, n), order="F"), np.empty((n, n), order="F"), np.empty((n, n), order="F")
    d2h = AsyncD2H()
    if "--nofault" not in sys.argv:
        d2h.prefault([vy, vt, r, uy, ut])
    d2h.push(vq_ev, [(run.Vy, vy, 0, n), (run.Vt, vt, 0, n)])
    end_ev = torch.cuda.Event()
    end_ev.record()
    t.append(("launch", time.perf_counter()))
    vq_ev.synchronize()
    t.append(("Vq final", time.perf_counter()))
    d2h.push(end_ev, [(run.R, r, 0, n), (run.Uy, uy, 0, n), (run.Ut, ut, 0, n)])
    end_ev.synchronize()
    t.append(("device done", time.perf_counter()))
    d2h.finish()
    t.append(("D2H done", time.perf_counter()))
    print(" | ".join(f"{k} {v - t[0][1]:.3f}" for k, v in t[1:]), flush=True)
    del run, a_dev, g_dev
