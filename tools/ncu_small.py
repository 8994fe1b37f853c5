"""Representative panel-QR leaf and Jacobi launches for ncu captures."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
what = sys.argv[1] if len(sys.argv) > 1 else "qr"
if what == "qr":
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    A = dempty(rows, 256); A.t.normal_()
    for _ in range(2):
        B = dempty(rows, 256); B.t.copy_(A.t); dv.geqrf(B)
else:
    A = dempty(256, 256); A.t.normal_(); A.t.triu_()
    for _ in range(2):
        dv.gesvj(A)
torch.cuda.synchronize()
