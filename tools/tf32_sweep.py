"""3xTF32 tcgen05 GEMM throughput (useful FLOP/s, CUDA events) on C5-like shapes."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

def rnd(m, n):
    d = dempty(m, n, dtype=torch.float32); d.t.normal_(); return d

def t_of(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps

for (ta, tb, m, n, k, beta) in [("N", "N", 8192, 8192, 8192, 0.0), ("T", "N", 8192, 8192, 8192, 0.0),
                                ("N", "T", 8192, 8192, 8192, 0.0), ("T", "T", 8192, 8192, 8192, 0.0),
                                ("T", "T", 32768, 512, 32768, 0.0), ("N", "N", 32768, 512, 32768, 0.0),
                                ("N", "T", 32768, 32768, 512, 1.0), ("N", "N", 32768, 32768, 512, 1.0)]:
    A = rnd(k, m) if ta == "T" else rnd(m, k)
    B = rnd(n, k) if tb == "T" else rnd(k, n)
    C = rnd(m, n)
    t = t_of(lambda: dv.sgemm_tf32x3(ta, tb, 1.0, A, B, beta, C))
    print(f"{ta}{tb} {m}x{n}x{k} beta={beta}: {t*1e3:8.3f} ms {2*m*n*k/t/1e12:7.1f} TF/s (useful)", flush=True)
    del A, B, C
