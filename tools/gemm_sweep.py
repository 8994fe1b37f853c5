"""K / beta sweep of the DMMA GEMM (TFLOP/s, CUDA events)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

def rnd(m, n):
    d = dempty(m, n); d.t.normal_(); return d

def t_of(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps

M = N = 16384
C = rnd(M, N)
for ta, tb in [("N", "T"), ("N", "N")]:
    for K in [64, 128, 256, 512, 1024, 2048]:
        A = rnd(K, M) if ta == "T" else rnd(M, K)
        B = rnd(N, K) if tb == "T" else rnd(K, N)
        for beta in [0.0, 1.0]:
            t = t_of(lambda: dv.gemm(ta, tb, -1.0, A, B, beta, C))
            print(f"{ta}{tb} M=N={M} K={K:5d} beta={beta}: {t*1e3:8.3f} ms {2*M*N*K/t/1e12:6.2f} TF/s", flush=True)
        del A, B
