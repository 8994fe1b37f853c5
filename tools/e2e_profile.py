"""Stage timings of the public-API (host numpy in/out) path at n=16384."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2106_13402_b200 as pk
n, b, q = 16384, 256, 2
rng = np.random.default_rng(0)
t = time.perf_counter
a = np.asfortranarray(rng.standard_normal((n, n)))
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
for rep in range(2):
    T0 = t(); f = pk.randutv_basic(a, b, q, pk.RngStream(3)); T1 = t(); print("TOTAL randutv_basic", T1 - T0, flush=True)
    del f
    T0 = t(); fp = pk.power_urv(a, q, pk.RngStream(2)); T1 = t(); print("TOTAL power_urv", T1 - T0, flush=True)
    del fp
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); fp = pk.power_urv(a, q, pk.RngStream(2)); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
pr = cProfile.Profile(); pr.enable(); f = pk.randutv_basic(a, b, q, pk.RngStream(3)); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
# raw host costs
g = pk.RngStream(2)
T0 = t(); z = g._gen.standard_normal((n, n)); print("draw n^2 normals", t() - T0)
T0 = t(); z2 = np.empty((n, n)); g._gen.standard_normal(out=z2); print("draw into preallocated", t() - T0)
T0 = t(); dt = torch.from_numpy(z2).cuda(); torch.cuda.synchronize(); print("H2D pageable 2 GiB", t() - T0)
T0 = t(); back = dt.cpu().numpy(); print("D2H pageable 2 GiB", t() - T0)
import os
print("cpus", os.cpu_count())
