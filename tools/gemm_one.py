import sys; sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
M = N = 16384; K = 256
C = dempty(M, N); C.t.normal_()
A = dempty(M, K); A.t.normal_()
B = dempty(N, K); B.t.normal_()
for beta in (0.0, 1.0):
    dv.gemm("N", "T", -1.0, A, B, beta, C)
torch.cuda.synchronize()
