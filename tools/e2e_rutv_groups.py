"""Where randUTV's e2e time outside the device loop goes: CUDA events
around every step group of the pipelined public call (device timeline) next
to the host timeline (group launch, draw, D2H finish)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2106_13402_b200 as pk
from paper_2106_13402_b200 import _lib, randutv

n, b, q = 16384, 256, 2
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
lib = _lib.load()
orig = lib.utv_randutv_basic_steps_carry_f64
log = []


class Wrap:
    def __getattr__(self, k):
        return getattr(lib, k)

    def utv_randutv_basic_steps_carry_f64(self, *args):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record()
        r = orig(*args)
        e1.record()
        log.append((args[0], args[1], h0, time.perf_counter(), e0, e1))
        return r


torch.zeros(1, device="cuda")
real_load = _lib.load
for rep in range(2):
    log.clear()
    _lib.load = lambda: Wrap()
    t0 = time.perf_counter()
    f = pk.randutv_basic(a, b, q, pk.RngStream(3))
    t1 = time.perf_counter()
    _lib.load = real_load
    torch.cuda.synchronize()
    first = log[0][4]
    print(f"rep {rep}: e2e {t1 - t0:.3f} s; first group launched at {log[0][2] - t0:.3f} s")
    for j0, j1, h0, h1, e0, e1 in log[-6:]:
        print(f"  steps {j0:2d}-{j1:2d}: host launch {h0 - t0:.3f}-{h1 - t0:.3f}  device {first.elapsed_time(e0) / 1e3:.3f}-{first.elapsed_time(e1) / 1e3:.3f}")
    print(f"  device span {first.elapsed_time(log[-1][5]) / 1e3:.3f} s; returned {t1 - t0 - (log[0][2] - t0):.3f} s after the first launch")
    del f
