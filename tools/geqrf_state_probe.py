"""Which earlier call corrupts a following geqrf (odd row offset, 20001 x 300)?"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

D = lambda d: d.tensor().T


def qr_err(sub):
    m, n = sub.rows, sub.cols
    A = D(sub)[:m, :n].clone()
    Y, T = dv.geqrf(sub)
    Yd, Td, Rd = D(Y)[:m, :n], D(T)[:n, :n], torch.triu(D(sub)[:n, :n])
    E = torch.zeros(m, n, device="cuda", dtype=torch.float64)
    E[:n, :n] = torch.eye(n, device="cuda", dtype=torch.float64)
    Q = E - Yd @ (Td @ Yd[:n, :].T)
    return (Q @ Rd - A).abs().max().item() / A.abs().max().item()


def fresh(rows, n, off, seed):
    big = dempty(rows + off, n)
    big.t.normal_(generator=torch.Generator(device="cuda").manual_seed(seed))
    return big.sub(off, 0, rows, n)


target = lambda: fresh(20001, 300, 20001, 7)
print("alone                         ", f"{qr_err(target()):.1e}")
for label, pre in [("after even 20001x300 geqrf ", lambda: fresh(20001, 300, 0, 1)),
                   ("after odd 20001x300 geqrf  ", lambda: fresh(20001, 300, 1, 2)),
                   ("after even 9001x300 geqrf  ", lambda: fresh(9001, 300, 0, 3)),
                   ("after even 20001x256 geqrf ", lambda: fresh(20001, 256, 0, 4)),
                   ("after even 20000x300 geqrf ", lambda: fresh(20000, 300, 0, 5))]:
    e0 = qr_err(pre())
    torch.cuda.synchronize()
    print(label, f"pre {e0:.1e}  target {qr_err(target()):.1e}", flush=True)
