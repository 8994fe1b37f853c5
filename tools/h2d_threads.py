"""H2D of a 2 GiB F-order array through _lib's pinned staging ring: GB/s vs
memcpy threads and ring chunk size (the head of every public call)."""
import sys
import time

sys.path.insert(0, ".")
import concurrent.futures
import os

import numpy as np
import torch

from paper_2106_13402_b200 import _lib

print("host cpus", os.cpu_count())
n = 16384
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
m = _lib.dempty(n, n)
torch.zeros(1, device="cuda")
flat = a.reshape(-1, order="F").view(np.uint8)
dst = m.t.view(-1)[m.off: m.off + n * n].view(torch.uint8)
for workers, nthr, chunk in [(8, 8, 64), (16, 8, 64), (8, 8, 64), (16, 8, 64), (16, 12, 64), (16, 8, 32), (16, 8, 128)]:
    _lib._RING = None
    _lib._H2D_RING = None
    _lib._RING_CHUNK = chunk << 20
    _lib._ring()
    _lib._POOL = concurrent.futures.ThreadPoolExecutor(max_workers=workers)
    ts = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib._h2d_bytes(flat, dst, torch.cuda.current_stream(), nthr=nthr)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"pool {workers:2d} nthr {nthr:2d} chunk {chunk:3d} MiB: {min(ts) * 1e3:6.1f} ms {flat.nbytes / min(ts) / 1e9:5.1f} GB/s",
          flush=True)
