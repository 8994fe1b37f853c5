"""D2H options for a 2 GiB result array: the staged pinned ring (_lib.d2h_numpy)
vs cudaHostRegister of the (pre-faulted) numpy destination + one DMA."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2106_13402_b200 import _lib
from paper_2106_13402_b200._lib import dempty

n = 16384
d = dempty(n, n)
d.t.normal_()
torch.cuda.synchronize()
t = time.perf_counter
for rep in range(2):
    T0 = t()
    h = _lib.d2h_numpy(d)
    print(f"staged ring D2H 2 GiB: {t() - T0:.3f} s", flush=True)
cudart = torch.cuda.cudart()
for rep in range(2):
    out = np.empty((n, n), order="F")
    T0 = t()
    out.reshape(-1, order="F")[:: 512] = 0.0          # pre-fault (4 KiB pages)
    T1 = t()
    r = cudart.cudaHostRegister(out.ctypes.data, out.nbytes, 0)
    T2 = t()
    src = d.t.view(-1)[: n * n]
    dst = torch.from_numpy(out.reshape(-1, order="F"))
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    T3 = t()
    cudart.cudaHostUnregister(out.ctypes.data)
    T4 = t()
    print(f"prefault {T1 - T0:.3f} s | hostRegister {T2 - T1:.3f} s (rc {r}) | DMA {T3 - T2:.3f} s "
          f"({out.nbytes / (T3 - T2) / 1e9:.1f} GB/s) | unregister {T4 - T3:.3f} s", flush=True)
    assert np.array_equal(out[:4, :4], d.tensor().T[:4, :4].cpu().numpy())
