"""Host timeline of the public power_urv / randutv_basic e2e calls at n=16384
(monkeypatched stage hooks; host clock): where the time outside the device
factorisation goes."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2106_13402_b200 as pk
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200 import _lib, powerurv

marks = []


def mark(label):
    marks.append((label, time.perf_counter()))


def wrap(obj, name, label):
    f = getattr(obj, name)

    def g(*a, **k):
        mark(label + ">")
        r = f(*a, **k)
        mark(label + "<")
        return r
    setattr(obj, name, g)


wrap(powerurv, "dfrom_numpy", "H2D A")
wrap(powerurv, "raise_if_nonfinite", "finite")
wrap(dv.PowerUrvRun, "run_cols", "launch driver")
wrap(_lib.AsyncD2H, "finish", "D2H finish")

n, q = 16384, 2
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
torch.zeros(1, device="cuda")
for rep in range(5):
    marks.clear()
    mark("start")
    f = pk.power_urv(a, q, pk.RngStream(2))
    mark("end")
    t0 = marks[0][1]
    print(" | ".join(f"{k} {v - t0:.3f}" for k, v in marks[1:]), flush=True)
    del f
