"""Single representative DMMA GEMM launches for ncu --set full captures."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

def rnd(m, n):
    d = dempty(m, n); d.t.normal_(); return d

shape = sys.argv[1] if len(sys.argv) > 1 else "nt"
if shape == "nt":      # rank-256 trailing update B -= W Y^T (qr.py:120 / larfb right)
    m, n, k, ta, tb = 16384, 16384, 256, "N", "T"
elif shape == "tt":    # sampling Y = B^T G^T (randutv.py:190)
    m, n, k, ta, tb = 16384, 256, 16384, "T", "T"
else:                  # square
    m, n, k, ta, tb = 8192, 8192, 8192, "N", "N"
A = rnd(k, m) if ta == "T" else rnd(m, k)
B = rnd(n, k) if tb == "T" else rnd(k, n)
C = rnd(m, n)
for _ in range(3):
    dv.gemm(ta, tb, 1.0, A, B, 1.0, C)
torch.cuda.synchronize()
