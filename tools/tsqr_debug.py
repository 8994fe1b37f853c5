"""Step-by-step check of the TSQR tree (sharded.tsqr) at a failing size."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2106_13402_b200._lib import dempty
from paper_2106_13402_b200.sharded import DeviceOps, _row_chunks, q_times_top

m = int(sys.argv[1]) if len(sys.argv) > 1 else 74898
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 37449
ops = DeviceOps()
I = lambda k: torch.eye(k, device="cuda", dtype=torch.float64)
D = lambda d: d.tensor().T
a = dempty(m, n)
a.t.normal_(generator=torch.Generator(device="cuda").manual_seed(40))
A = D(a)[:m, :n].clone()
chunks = _row_chunks(m, n, cap)
print("chunks", chunks)
work = ops.copy(a)
leaves = []
for (r0, nr) in chunks:
    blk = ops.sub(work, r0, 0, nr, n)
    y, t = ops.geqrf(blk)
    leaves.append((y, t))
    Rc = torch.triu(D(blk)[:n, :n])
    E = torch.zeros(nr, n, device="cuda", dtype=torch.float64); E[:n] = I(n)
    Yd, Td = D(y)[:nr, :n], D(t)[:n, :n]
    Qc = E - Yd @ (Td @ Yd[:n].T)
    print(f"leaf r0={r0} nr={nr}: QR=A {((Qc @ Rc) - A[r0:r0 + nr]).abs().max().item():.1e}; "
          f"below-diag of R block {D(blk)[:n, :n].tril(-1).abs().max().item():.1e}; "
          f"rows n.. of blk {D(blk)[n:nr, :n].abs().max().item() if nr > n else 0:.1e}")
nch = len(chunks)
stk = ops.empty(nch * n, n)
for c, (r0, _) in enumerate(chunks):
    ops.lacpy(ops.sub(work, r0, 0, n, n), ops.sub(stk, c * n, 0, n, n))
S0 = D(stk)[:nch * n, :n].clone()
ys, ts = ops.geqrf(stk)
R = torch.triu(D(stk)[:n, :n])
f = ops.empty(nch * n, n)
e = ops.eye(n)
q_times_top(ys, ts, e, f, ops)
F = D(f)[:nch * n, :n]
print(f"stack: F R = S {((F @ R) - S0).abs().max().item():.1e}, orth {(F.T @ F - I(n)).abs().max().item():.1e}")
for c, (r0, nr) in enumerate(chunks):
    out = ops.empty(nr, n)
    y, t = leaves[c]
    top = ops.sub(f, c * n, 0, n, n)
    q_times_top(y, t, top, out, ops)
    Qc = D(out)[:nr, :n]
    print(f"chunk {c}: Q_c R = A_c {((Qc @ R) - A[r0:r0 + nr]).abs().max().item():.1e}")
