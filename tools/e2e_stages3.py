"""Host timeline of the public randutv_basic / power_urv e2e calls at n=16384
next to the device-only time of the same factorisation (where the e2e
overhead goes); also the AsyncD2H throughput into pre-faulted arrays."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2106_13402_b200 as pk
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200 import _lib, powerurv, randutv

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


wrap(randutv, "dfrom_numpy", "H2D A")
wrap(randutv, "raise_if_nonfinite", "finite")
wrap(_lib.AsyncD2H, "finish", "D2H finish")
wrap(randutv, "_finish_basic", "finish_basic")

n, b, q = 16384, 256, 2
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
torch.zeros(1, device="cuda")
for rep in range(3):
    marks.clear()
    mark("start")
    f = pk.randutv_basic(a, b, q, pk.RngStream(3))
    mark("end")
    t0 = marks[0][1]
    print("randutv: " + " | ".join(f"{k} {v - t0:.3f}" for k, v in marks[1:]), flush=True)
    del f
# device-only randUTV of the same input
t_dev = _lib.dfrom_numpy(a)
blocks = pk.randutv.draw_sample_blocks(pk.RngStream(3), n, n, b)
G = dv.stage_randutv_blocks(blocks, b)
run = dv.RandUtvRun(n, n, b, q)
T = _lib.dempty(n, n)
U, V = _lib.deye(n), _lib.deye(n)
for rep in range(2):
    _lib.check(_lib.load().utv_dlacpy(n, n, t_dev.ptr, t_dev.ld, T.ptr, T.ld, _lib.stream_ptr()), "cp")
    U, V = _lib.deye(n), _lib.deye(n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run.run(T, U, V, G)
    e1.record()
    torch.cuda.synchronize()
    print(f"randutv device-only {e0.elapsed_time(e1) / 1e3:.3f} s", flush=True)
# AsyncD2H throughput, destinations pre-faulted
outs = [np.empty((n, n), order="F") for _ in range(3)]
for o in outs:
    o.reshape(-1, order="F")[::512] = 0.0
ev = torch.cuda.Event()
ev.record()
T0 = time.perf_counter()
d2h = _lib.AsyncD2H()
d2h.push(ev, [(T, outs[0], 0, n), (U, outs[1], 0, n), (V, outs[2], 0, n)])
d2h.finish()
dt = time.perf_counter() - T0
print(f"AsyncD2H 6 GiB into pre-faulted arrays: {dt:.3f} s ({3 * n * n * 8 / dt / 1e9:.1f} GB/s)", flush=True)
