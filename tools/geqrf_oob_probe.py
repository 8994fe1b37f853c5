"""Does geqrf on the top rows of a buffer write below its sub-matrix?"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

D = lambda d: d.tensor().T
for (half, n) in [(20001, 300), (20000, 300), (20001, 256), (20001, 257), (9001, 300), (37449, 300)]:
    big = dempty(2 * half, n)
    big.t.normal_(generator=torch.Generator(device="cuda").manual_seed(half))
    before = D(big)[half:2 * half, :n].clone()
    dv.geqrf(big.sub(0, 0, half, n))
    torch.cuda.synchronize()
    diff = (D(big)[half:2 * half, :n] != before)
    if diff.any():
        rows = diff.any(dim=1).nonzero().flatten()
        cols = diff.any(dim=0).nonzero().flatten()
        print(f"{half}x{n}: {int(diff.sum())} entries below the view changed: rows {half + int(rows.min())}.."
              f"{half + int(rows.max())}, cols {int(cols.min())}..{int(cols.max())}", flush=True)
    else:
        print(f"{half}x{n}: clean", flush=True)
