"""Two tall geqrf calls on two streams concurrently vs one call of twice the rows.
usage: python tools/tall_qr_conc.py [rows_each] [cols]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

r = int(sys.argv[1]) if len(sys.argv) > 1 else 37449
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
A = [dempty(r, n) for _ in range(2)]
for a in A:
    a.t.normal_()
B = [dempty(r, n) for _ in range(2)]
s2 = [torch.cuda.Stream(), torch.cuda.Stream()]
main = torch.cuda.current_stream()


def one_seq():
    for a, b in zip(A, B):
        b.t.copy_(a.t)
        dv.geqrf(b)


def one_conc():
    for a, b in zip(A, B):
        b.t.copy_(a.t)
    ev = torch.cuda.Event()
    ev.record(main)
    outs = []
    for s, b in zip(s2, B):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            outs.append(dv.geqrf(b))
    for s in s2:
        main.wait_stream(s)
    return outs


for name, f in [("sequential", one_seq), ("concurrent", one_conc)]:
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
    print(f"{name}: 2 x geqrf {r}x{n}: {e0.elapsed_time(e1):.1f} ms", flush=True)
