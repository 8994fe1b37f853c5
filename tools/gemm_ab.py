"""A/B of GEMM epilogue variants on the K=256/512 update shapes (TFLOP/s,
CUDA events).  Run once per environment setting, e.g.
UTV_GEMM_TSTORE0=1 python tools/gemm_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_13402_b200.device as dv  # noqa: E402
from paper_2106_13402_b200._lib import dempty  # noqa: E402


def rnd(m, n):
    d = dempty(m, n)
    d.t.normal_()
    return d


def t_of(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("UTV_")) or "default"
M = N = 16384
C = rnd(M, N)
for ta, tb in [("N", "T"), ("N", "N"), ("T", "N")]:
    for K in [256, 512, 2048]:
        A = rnd(K, M) if ta == "T" else rnd(M, K)
        B = rnd(N, K) if tb == "T" else rnd(K, N)
        for beta in [0.0, 1.0]:
            t = t_of(lambda: dv.gemm(ta, tb, -1.0, A, B, beta, C))
            print(f"[{tag}] {ta}{tb} M=N={M} K={K:5d} beta={beta}: {t*1e3:8.3f} ms {2*M*N*K/t/1e12:6.2f} TF/s",
                  flush=True)
        del A, B
# split-K shapes (sampling / W = Y^T B)
for ta, tb, m, n, k in [("T", "N", 256, 16384, 16384), ("N", "N", 16384, 256, 16384),
                        ("T", "N", 256, 8192, 8192), ("T", "N", 256, 4096, 12288)]:
    A = rnd(k, m) if ta == "T" else rnd(m, k)
    B = rnd(n, k) if tb == "T" else rnd(k, n)
    Cs = rnd(m, n)
    t = t_of(lambda: dv.gemm(ta, tb, 1.0, A, B, 0.0, Cs))
    print(f"[{tag}] splitK {ta}{tb} {m}x{n}x{k}: {t*1e3:8.3f} ms {2*m*n*k/t/1e12:6.2f} TF/s", flush=True)
