"""Per-tile time of the K=256 DMMA GEMM vs grid size (UTV_GEMM_CTAS set by the caller):
contention between SMs shows up as a longer per-tile time at full grid."""
import os, sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
def rnd(m, n):
    d = dempty(m, n); d.t.normal_(); return d
M = N = 16384
cap = int(os.environ.get("UTV_GEMM_CTAS", "148") or 148)
C = rnd(M, N)
for K in [256, 1024]:
    A, B = rnd(M, K), rnd(K, N)
    for beta in [0.0, 1.0]:
        f = lambda: dv.gemm("N", "N", 1.0, A, B, beta, C)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        tiles = (M // 128) * (N // 128)
        print(f"cap={cap:3d} K={K:5d} beta={beta}: {ms:8.3f} ms, {2*M*N*K/ms/1e9:6.2f} TF/s, "
              f"{ms*1e3/(tiles/cap):6.2f} us per tile per CTA, {2*M*N*K/ms/1e9/cap*148:6.2f} TF/s scaled to 148")
