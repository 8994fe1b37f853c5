"""Per-launch timeline of one tall geqrf (C4's TSQR leaf): category busy
times and the slowest GEMM launches by shape.
usage: UTV_PROF_DUMP=gpurun_out/tall.csv python tools/tall_qr_prof.py [rows] [cols]"""
import collections
import os
import sys

sys.path.insert(0, ".")
import torch

import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200 import _lib
from paper_2106_13402_b200._lib import dempty

m = int(sys.argv[1]) if len(sys.argv) > 1 else 74898
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
A = dempty(m, n)
A.t.normal_()
B = dempty(m, n)
for rep in range(2):
    B.t.copy_(A.t)
    torch.cuda.synchronize()
    dump = os.environ.get("UTV_PROF_DUMP")
    if dump and os.path.exists(dump):
        os.remove(dump)
    _lib.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dv.geqrf(B)
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.profile_end()
ms = e0.elapsed_time(e1)
fl = 2.0 * m * n * n - 2.0 / 3.0 * n ** 3
print(f"geqrf {m}x{n}: {ms:.1f} ms, {fl / ms / 1e9:.1f} TF/s (Householder flops)")
for k, v in prof.items():
    if v["ms"] > 0:
        print(f"  {k:14s} {v['ms']:8.1f} ms  {v.get('flops', 0) / max(v['ms'], 1e-9) / 1e9:6.1f} TF/s")

cats = list(_lib.PROF_CATEGORIES)
dump = os.environ.get("UTV_PROF_DUMP")
if dump:
    rows = []
    for line in open(dump):
        c, t0, t1, f, st = line.strip().split(",")
        rows.append((cats[int(c)], float(t0), float(t1), float(f), st))
    by = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for c, t0, t1, f, st in rows:
        k = (c, f"{f:.4g}", st)
        by[k][0] += t1 - t0
        by[k][1] += 1
        by[k][2] += f
    print("top launch groups (category, flops per launch, stream): total ms, count, TF/s")
    for k, (t, cnt, f) in sorted(by.items(), key=lambda kv: -kv[1][0])[:40]:
        print(f"  {k[0]:12s} {k[1]:>10s} {k[2]:>14s} {t:8.2f} ms x{cnt:3d} {f / max(t, 1e-9) / 1e9:6.1f}")
    print("first launches in time order: category, start, ms, GF, TF/s, stream")
    for c, t0, t1, f, st in sorted(rows, key=lambda r: r[1])[:60]:
        print(f"  {c:12s} {t0:9.3f} {t1 - t0:8.3f} {f / 1e9:9.1f} {f / max(t1 - t0, 1e-9) / 1e9:6.1f} {st}")
