"""geqrf on a sub-matrix view at a row offset: thin Q R = A on the device."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

D = lambda d: d.tensor().T
for (m, n, off, total) in [(2000, 300, 1, None), (9001, 300, 1, None), (20001, 300, 1, None),
                           (37449, 300, 1, None), (37449, 300, 37449, 74898), (37449, 300, 2, None),
                           (37449, 256, 1, None), (37449, 512, 1, None)]:
    rows = total or (m + off)
    big = dempty(rows, n)
    big.t.normal_(generator=torch.Generator(device="cuda").manual_seed(m + off))
    sub = big.sub(off, 0, m, n)
    A = D(sub)[:m, :n].clone()
    Y, T = dv.geqrf(sub)
    Yd, Td, Rd = D(Y)[:m, :n], D(T)[:n, :n], torch.triu(D(sub)[:n, :n])
    E = torch.zeros(m, n, device="cuda", dtype=torch.float64)
    E[:n, :n] = torch.eye(n, device="cuda", dtype=torch.float64)
    Q = E - Yd @ (Td @ Yd[:n, :].T)
    rec = (Q @ Rd - A).abs().max().item() / A.abs().max().item()
    orth = (Q.T @ Q - E[:n]).abs().max().item()
    print(f"geqrf {m}x{n} at row offset {off} (ld {big.ld}): QR=A {rec:.1e}, orth {orth:.1e}", flush=True)


def check(sub, A, Y, T, label):
    m, n = sub.rows, sub.cols
    Yd, Td, Rd = D(Y)[:m, :n], D(T)[:n, :n], torch.triu(D(sub)[:n, :n])
    E = torch.zeros(m, n, device="cuda", dtype=torch.float64)
    E[:n, :n] = torch.eye(n, device="cuda", dtype=torch.float64)
    Q = E - Yd @ (Td @ Yd[:n, :].T)
    print(f"{label}: QR=A {(Q @ Rd - A).abs().max().item() / A.abs().max().item():.1e}", flush=True)


for (half, n) in [(37449, 300), (601, 300), (9001, 300), (20001, 300)]:
    big = dempty(2 * half, n)
    big.t.normal_(generator=torch.Generator(device="cuda").manual_seed(half))
    s0, s1 = big.sub(0, 0, half, n), big.sub(half, 0, half, n)
    A0, A1 = D(s0)[:half, :n].clone(), D(s1)[:half, :n].clone()
    Y0, T0 = dv.geqrf(s0)
    Y1, T1 = dv.geqrf(s1)
    check(s0, A0, Y0, T0, f"consecutive halves {half}x{n}: first")
    check(s1, A1, Y1, T1, f"consecutive halves {half}x{n}: second")
    # second half alone
    big.t.normal_(generator=torch.Generator(device="cuda").manual_seed(half))
    A1 = D(s1)[:half, :n].clone()
    Y1, T1 = dv.geqrf(s1)
    check(s1, A1, Y1, T1, f"second half alone {half}x{n}")
