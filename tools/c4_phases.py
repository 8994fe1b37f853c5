"""Per-op device times of the row-sharded powerURV (C4) on one GPU.

Every DeviceOps call is bracketed by CUDA events (synchronised, so the
times add up to the step); totals are grouped by op name and shape.
usage: python tools/c4_phases.py [rows] [cols] [chunk_rows]
"""
import collections
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2106_13402_b200 as pk
from paper_2106_13402_b200 import _lib, sharded
from paper_2106_13402_b200._lib import dempty

m = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else None

acc = collections.OrderedDict()


class TimedOps(sharded.DeviceOps):
    pass


def _wrap(name):
    base = getattr(sharded.DeviceOps, name)

    def f(self, *a, **k):
        shp = tuple((x.rows, x.cols) for x in a if hasattr(x, "rows"))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = base(self, *a, **k)
        e1.record()
        torch.cuda.synchronize()
        key = (name, tuple(s for s in a if isinstance(s, str)), shp)
        t, c = acc.get(key, (0.0, 0))
        acc[key] = (t + e0.elapsed_time(e1), c + 1)
        return r
    setattr(TimedOps, name, f)


for nm in ["copy", "lacpy", "zeros", "eye", "gemm", "geqrf", "larfb", "orgqr", "getrf_signed",
           "trsm_right", "laset", "tri_zero", "diag_scale", "apply_q_top", "householder_tsqr_q"]:
    if hasattr(sharded.DeviceOps, nm):
        _wrap(nm)

a = dempty(m, n)
a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(40))
g = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(4)))
torch.cuda.synchronize()
for rep in range(2):
    acc.clear()
    t0 = time.perf_counter()
    out = sharded.power_urv_sharded(a, g, 1, ops=TimedOps(), chunk_rows=chunk)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    del out
tot = sum(t for t, _ in acc.values())
print(f"C4 phases m={m} n={n}: wall {wall*1e3:.0f} ms, sum of ops {tot:.0f} ms")
for k, (t, c) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{t:9.1f} ms  x{c:3d}  {k[0]} {k[1]} {k[2]}")
