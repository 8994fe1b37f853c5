"""One NN 16384^2 x 256 beta=0 DMMA GEMM launch (the K=256 per-tile overhead study) for ncu."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
def rnd(m, n):
    d = dempty(m, n); d.t.normal_(); return d
A, B, C = rnd(16384, 256), rnd(256, 16384), rnd(16384, 16384)
for _ in range(3):
    dv.gemm("N", "N", 1.0, A, B, 0.0, C)
torch.cuda.synchronize()
