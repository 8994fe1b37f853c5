"""DMMA GEMM with sub-matrix operands at odd row offsets (8-byte aligned) vs
torch fp64, over sizes that take the split-K / re-staged / direct-store paths."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

torch.manual_seed(0)


def sub_of(rows, cols, off):
    big = dempty(rows + off, cols)
    big.t.normal_()
    return big.sub(off, 0, rows, cols)


def dense(d):
    return d.tensor().T.clone()


worst = 0.0
for (m, n, k) in [(4096, 4096, 4096), (18725, 4096, 4096), (4096, 4096, 18725), (300, 96, 700), (4096, 256, 256)]:
    for ta, tb in [("N", "N"), ("T", "N"), ("N", "T")]:
        for offs in [(0, 0, 1), (1, 0, 0), (0, 1, 0), (1, 1, 1), (3, 0, 1)]:
            for beta in (0.0, 1.0):
                A = sub_of(k if ta == "T" else m, m if ta == "T" else k, offs[0])
                B = sub_of(n if tb == "T" else k, k if tb == "T" else n, offs[1])
                C = sub_of(m, n, offs[2])
                a, b, c0 = dense(A), dense(B), dense(C)
                ref = -1.0 * ((a.T if ta == "T" else a) @ (b.T if tb == "T" else b)) + beta * c0
                dv.gemm(ta, tb, -1.0, A, B, beta, C)
                err = ((dense(C) - ref).abs().max() / ref.abs().max()).item()
                worst = max(worst, err)
                if err > 1e-12:
                    print(f"BAD m={m} n={n} k={k} {ta}{tb} offs={offs} beta={beta}: rel err {err:.2e}", flush=True)
print("worst", worst)
