"""TSQR / geqrf accuracy with odd row offsets at C4-like sizes (device-side checks)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty
from paper_2106_13402_b200.sharded import tsqr, Comm, DeviceOps


def dense(d):
    return d.tensor().T


def recon(m, n, chunk):
    a = dempty(m, n)
    a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(40))
    q, r = tsqr(a, Comm(), DeviceOps(), chunk_rows=chunk)
    Q, R, A = dense(q)[:m, :n], dense(r)[:n, :n], dense(a)[:m, :n]
    orth = (Q.T @ Q - torch.eye(n, device="cuda", dtype=torch.float64)).abs().max().item()
    rec = ((Q @ R) - A).abs().max().item() / A.abs().max().item()
    print(f"tsqr {m}x{n} chunk {chunk}: orth {orth:.1e} recon {rec:.1e}", flush=True)


def geqrf_offset(m, n, off):
    big = dempty(m + off, n)
    big.t.normal_(generator=torch.Generator(device="cuda").manual_seed(41))
    ref = dempty(m, n)
    ref.t[:, :m].copy_(big.t[:, off:off + m])
    dv.geqrf(ref)
    sub = big.sub(off, 0, m, n)
    dv.geqrf(sub)
    d = (torch.diagonal(dense(sub)[:n, :n]) - torch.diagonal(dense(ref)[:n, :n])).abs().max().item()
    print(f"geqrf {m}x{n} at row offset {off}: max |diag R - diag R(offset 0)| {d:.1e}", flush=True)


for n in (300, 1024, 4096):
    recon(74898, n, 37449)
for off in (0, 1, 2):
    geqrf_offset(37449, 4096, off)
geqrf_offset(37448, 4096, 1)
