"""geqrf's compact-WY factor checked by its defining property on the device:
Q = I - Y T Y^T, thin Q R = A and Q^T Q = I (torch fp64)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty


def dense(d):
    return d.tensor().T


for (m, n) in [(9001, 300), (37448, 4096), (37449, 4096), (74898, 300), (74898, 1024), (20000, 600), (20001, 600)]:
    a = dempty(m, n)
    a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(m + n))
    A = dense(a)[:m, :n].clone()
    r = dempty(m, n)
    r.t[:, :m].copy_(a.t[:, :m])
    Y, T = dv.geqrf(r)
    Yd, Td, Rd = dense(Y)[:m, :n], dense(T)[:n, :n], torch.triu(dense(r)[:n, :n])
    E = torch.zeros(m, n, device="cuda", dtype=torch.float64)
    E[:n, :n] = torch.eye(n, device="cuda", dtype=torch.float64)
    Q = E - Yd @ (Td @ Yd[:n, :].T)
    rec = (Q @ Rd - A).abs().max().item() / A.abs().max().item()
    orth = (Q.T @ Q - torch.eye(n, device="cuda", dtype=torch.float64)).abs().max().item()
    print(f"geqrf {m}x{n}: thin Q R = A to {rec:.1e}, orth {orth:.1e}", flush=True)
    del a, r, Y, T, Q, E
    torch.cuda.empty_cache()
