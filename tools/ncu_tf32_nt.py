"""One C5-shaped 3xTF32 GEMM (NT 32768^2 x 512, beta=1: the fp32 WY update) for ncu."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
def rnd(m, n):
    d = dempty(m, n, dtype=torch.float32); d.t.normal_(); return d
A, B, C = rnd(32768, 512), rnd(32768, 512), rnd(32768, 32768)
for _ in range(3):
    dv.sgemm_tf32x3("N", "T", 1.0, A, B, 1.0, C)
torch.cuda.synchronize()
