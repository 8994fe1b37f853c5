"""Device time of randUTV basic (b=256, q=2) for A/B of pipeline knobs."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty, deye
for n in [int(x) for x in (sys.argv[1:] or ["8192", "16384"])]:
    b, q = 256, 2
    T0 = dempty(n, n); T0.t.normal_()
    steps = -(-n // b)
    G = dempty(b, sum(n - i * b for i in range(steps - 1))); G.t.normal_()
    run = dv.RandUtvRun(n, n, b, q)
    T = dempty(n, n); U = deye(n); V = deye(n)
    def f():
        T.t.copy_(T0.t); U.t.zero_(); U.t.fill_diagonal_(1.0); V.t.zero_(); V.t.fill_diagonal_(1.0)
        run.run(T, U, V, G)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"randUTV n={n}: {min(ts):.1f} ms  checksum {float(T.t.diagonal().abs().sum()):.12e}", flush=True)
    del T0, G, run, T, U, V
