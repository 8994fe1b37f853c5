"""Sweep: no DMMA GEMM variant writes outside its C view (odd/even M and N,
all op combinations, beta 0/1, C views at row offsets 0/1 inside a taller,
wider buffer; split-K, re-staged and TMA-store paths)."""
import itertools
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

V = lambda d: d.tensor().T
bad = 0
for (M, N, K), (ta, tb), beta, off in itertools.product(
        [(20001, 300, 256), (20000, 301, 256), (4097, 4095, 64), (301, 20001, 512), (129, 131, 4097),
         (40001, 129, 16)],
        [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")], (0.0, 1.0), (0, 1)):
    big = dempty(M + off + 40, N + 3)
    big.t.normal_()
    C = big.sub(off, 1, M, N)
    A = dempty(K if ta == "T" else M, M if ta == "T" else K); A.t.normal_()
    B = dempty(N if tb == "T" else K, K if tb == "T" else N); B.t.normal_()
    before = V(big)[:big.rows, :big.cols].clone()
    dv.gemm(ta, tb, 1.0, A, B, beta, C)
    torch.cuda.synchronize()
    after = V(big)[:big.rows, :big.cols]
    mask = torch.ones_like(after, dtype=torch.bool)
    mask[off:off + M, 1:1 + N] = False
    n_out = int((after != before)[mask].sum())
    if n_out:
        bad += 1
        print(f"OOB: M={M} N={N} K={K} {ta}{tb} beta={beta} off={off}: {n_out} entries outside the view", flush=True)
print("cases with writes outside the view:", bad)
