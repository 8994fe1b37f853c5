"""Full-size C4 (powerURV q=1 on 524288 x 4096) through the SPMD row-sharded
path with P = 1, 2, 4 ranks emulated as threads on one B200 (ThreadComm:
each rank its own stream, allgather/allreduce/broadcast through the hub).
All ranks share the one GPU, so the time is the total work of P ranks plus
the exchange, not a scaling number; the point is that the P > 1 code path
runs at the full size and gives the same R (replicated) as P = 1.
usage: python tools/c4_threadcomm.py [rows] [cols]"""
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2106_13402_b200 as pk
from paper_2106_13402_b200 import _lib
from paper_2106_13402_b200._lib import dempty
from paper_2106_13402_b200.sharded import ThreadComm, power_urv_sharded

m = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
a = dempty(m, n)
a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(40))
g = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(4)))
torch.cuda.synchronize()
ref = None
for P in (1, 2, 4):
    bounds = np.linspace(0, m, P + 1).astype(int)
    hub = ThreadComm.make(P)
    out, errs = [None] * P, []

    def run(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = ThreadComm(hub, r, st)
                res = power_urv_sharded(a.sub(int(bounds[r]), 0, int(bounds[r + 1] - bounds[r]), n), g, 1,
                                        comm)
                st.synchronize()
                out[r] = torch.diagonal(res["R"].tensor()).abs().cpu().numpy()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            hub.barrier.abort()

    for rep in range(2):  # the first run warms the caching allocator
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    if errs:
        raise errs[0]
    d = out[0]
    same = max(float(np.abs(o - d).max()) for o in out)
    if ref is None:
        ref = d
    rel = float(np.abs(d - ref).max() / ref.max())
    print(f"P={P}: {dt:.2f} s wall on 1 GPU (all ranks), |diag R| ranks agree to {same:.1e}, "
          f"vs P=1: max rel diff {rel:.1e}", flush=True)
