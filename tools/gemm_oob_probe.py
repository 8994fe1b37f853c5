"""DMMA GEMM: does C = beta C + alpha A B write outside the M x N view?"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

D = lambda d: d.tensor().T
for (M, N, K, ta, tb, beta) in [(20001, 44, 256, "N", "N", 1.0), (20001, 44, 256, "N", "N", 0.0),
                                (20001, 300, 256, "N", "N", 1.0), (9001, 44, 256, "N", "N", 1.0),
                                (20001, 44, 256, "N", "T", 1.0), (20003, 200, 512, "N", "N", 1.0)]:
    big = dempty(2 * M, N)
    big.t.normal_()
    C = big.sub(0, 0, M, N)
    A = dempty(K if ta == "T" else M, M if ta == "T" else K); A.t.normal_()
    B = dempty(N if tb == "T" else K, K if tb == "T" else N); B.t.normal_()
    before = D(big)[M:, :N].clone()
    dv.gemm(ta, tb, -1.0, A, B, beta, C)
    torch.cuda.synchronize()
    diff = D(big)[M:, :N] != before
    print(f"M={M} N={N} K={K} {ta}{tb} beta={beta}: {int(diff.sum())} entries below the view changed"
          + (f" (rows {M + int(diff.any(1).nonzero().min())}..{M + int(diff.any(1).nonzero().max())})" if diff.any() else ""),
          flush=True)
