import sys, numpy as np
sys.path.insert(0, '.')
from paper_2106_13402_b200._lib import DMat, check, load, stream_ptr, workspace, dfrom_numpy
import torch
rng = np.random.default_rng(5)
big = rng.standard_normal((301, 260)); Bm = rng.standard_normal((260, 90))
dA, dB = dfrom_numpy(big), dfrom_numpy(Bm)
r0, c0, m, k = [int(x) for x in sys.argv[1:5]]
C = dfrom_numpy(np.zeros((m, 90)))
lib = load(); lw = lib.utv_dgemm_bufsize(m, 90, k); ws = workspace(lw)
check(lib.utv_dgemm(b"N", b"N", m, 90, k, 1.0, dA.at(r0, c0), dA.ld, dB.ptr, dB.ld, 0.0, C.ptr, C.ld, ws.data_ptr(), lw, stream_ptr()), "dgemm")
torch.cuda.synchronize()
ref = big[r0:r0 + m, c0:c0 + k] @ Bm[:k]
print(r0, c0, m, k, "maxerr", np.abs(C.to_numpy() - ref).max())
