"""Time geqrf of n x n (and powerURV) for look-ahead tuning."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
for n in [8192, 16384]:
    A = dempty(n, n); A.t.normal_()
    B = dempty(n, n)
    def f():
        B.t.copy_(A.t); dv.geqrf(B)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize()
    print(n, e0.elapsed_time(e1), "ms", flush=True)
    del A, B
