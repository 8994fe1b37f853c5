"""powerURV per-phase device times (UTV_PHASES=1 makes libutvb200 print them)."""
import os, sys
os.environ["UTV_PHASES"] = "1"
sys.path.insert(0, ".")
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = int(sys.argv[2]) if len(sys.argv) > 2 else 2
A = dempty(n, n); A.t.normal_()
G = dempty(n, n); G.t.normal_()
run = dv.PowerUrvRun(n, n, q)
for rep in range(2):
    print(f"--- rep {rep}", file=sys.stderr, flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run.run(A, G); e1.record(); torch.cuda.synchronize()
    print(f"powerURV n={n} q={q}: {e0.elapsed_time(e1):.1f} ms", file=sys.stderr, flush=True)
