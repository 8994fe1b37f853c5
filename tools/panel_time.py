"""Panel QR (single <=256-wide geqrf) device time vs rows and CTA budget."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
for m in [16384, 8192, 4096, 2048]:
    A = dempty(m, 256); A.t.normal_()
    B = dempty(m, 256)
    def f():
        B.t.copy_(A.t); dv.geqrf(B)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"ctas={os.environ.get('UTV_PANEL_CTAS', 'all')} rows={m} {min(ts):.3f} ms", flush=True)
