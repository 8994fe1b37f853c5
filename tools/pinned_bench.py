"""Cost of fresh page-locked host buffers (torch CachingHostAllocator ->
cudaHostAlloc) vs re-use from torch's pinned cache, and a direct D2H DMA
into a pinned-backed F-order numpy result."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2106_13402_b200._lib import dempty

n = 16384
nb = n * n * 8
d = dempty(n, n)
d.t.normal_()
torch.cuda.synchronize()
t = time.perf_counter
for rep in range(3):
    T0 = t()
    p = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    T1 = t()
    host = p.view(torch.float64).view(n, n)
    host.copy_(d.t[:n, :n], non_blocking=True)
    torch.cuda.synchronize()
    T2 = t()
    arr = host.numpy().T                     # F-order (rows, cols)
    assert arr.flags.f_contiguous
    print(f"pinned alloc 2 GiB {T1 - T0:.3f} s | DMA {T2 - T1:.3f} s ({nb / (T2 - T1) / 1e9:.1f} GB/s)", flush=True)
    del p, host, arr
for rep in range(2):
    T0 = t()
    bufs = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(5)]
    print(f"5 x 2 GiB pinned (cache after free): {t() - T0:.3f} s", flush=True)
    del bufs
