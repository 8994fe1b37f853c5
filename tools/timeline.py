"""Kernel timeline of one call (UTV_PROF_DUMP) -> idle gaps, per-stream busy, per-category time.
Usage: python tools/timeline.py geqrf 16384 | purv 16384 | rutv 8192"""
import os, sys, collections
sys.path.insert(0, ".")
what, n = sys.argv[1], int(sys.argv[2])
path = f"gpurun_out/timeline_{what}_{n}.csv"
if os.path.exists(path): os.remove(path)
import torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200 import _lib
from paper_2106_13402_b200._lib import dempty, deye
if what == "rutv32":
    import bench
    A = bench.make_rank_deficient_f32(n, 2000, 50)
else:
    A = dempty(n, n); A.t.normal_()
if what == "rutv32":
    b = 512; steps = -(-n // b)
    G = dempty(b, sum(n - i * b for i in range(steps - 1)), dtype=torch.float32); G.t.normal_()
    run = dv.RandUtvRun32(n, n, b, 2)
    T = dempty(n, n, dtype=torch.float32); U = dempty(n, n, dtype=torch.float32); V = dempty(n, n, dtype=torch.float32)
    def f():
        T.t.copy_(A.t); U.t.zero_(); U.t[:, :n].fill_diagonal_(1.0); V.t.zero_(); V.t[:, :n].fill_diagonal_(1.0)
        run.run(T, U, V, G)
elif what == "geqrf":
    B = dempty(n, n)
    def f(): B.t.copy_(A.t); dv.geqrf(B)
elif what == "purv":
    G = dempty(n, n); G.t.normal_(); run = dv.PowerUrvRun(n, n, 2)
    def f(): run.run(A, G)
else:
    b = 256; steps = -(-n // b)
    G = dempty(b, sum(n - i * b for i in range(steps - 1))); G.t.normal_()
    run = dv.RandUtvRun(n, n, b, 2); T = dempty(n, n); U = deye(n); V = deye(n)
    def f(): T.t.copy_(A.t); run.run(T, U, V, G)
f(); torch.cuda.synchronize()
os.environ["UTV_PROF_DUMP"] = path
_lib.profile_begin(); f(); prof = _lib.profile_end()
names = _lib.PROF_CATEGORIES
rows = [l.strip().split(",") for l in open(path)]
ev = sorted((float(r[1]), float(r[2]), int(r[0]), r[4]) for r in rows)
t0, t1 = ev[0][0], max(e[1] for e in ev)
# union of all kernel intervals -> idle time
busy, cs, ce = 0.0, -1, -1
for s, e, c, st in ev:
    if s > ce:
        busy += max(0, ce - cs); cs, ce = s, e
    else:
        ce = max(ce, e)
busy += ce - cs
print(f"{what} n={n}: span {t1 - t0:.2f} ms, any-kernel busy {busy:.2f} ms, idle {t1 - t0 - busy:.2f} ms")
for k, v in prof.items():
    if v["count"]:
        print(f"  {k:14s} launches {v['count']:5d}  sum {v['ms']:9.2f} ms  busy {v['busy_ms']:9.2f} ms  "
              f"{v['flops'] / max(v['busy_ms'], 1e-9) / 1e9:7.2f} TF/s(busy)")
per_stream = collections.defaultdict(float)
for s, e, c, st in ev: per_stream[st] += e - s
for st, v in per_stream.items(): print(f"  stream {st}: {v:.2f} ms of launches")
# per stream and category
psc = collections.defaultdict(float)
for s_, e_, c_, st_ in ev: psc[(st_, names[c_])] += e_ - s_
for (st_, c_), v in sorted(psc.items()): print(f"    {st_} {c_:14s} {v:9.2f} ms")
# critical-path stalls of the main stream: idle gaps of the stream "(nil)"
# that end within 50 us of a side-stream kernel's end (the main stream was
# waiting on that event)
main = sorted((s, e, names[c]) for s, e, c, st in ev if st == "(nil)")
side = sorted((e, names[c], st) for s, e, c, st in ev if st != "(nil)")
stall = collections.defaultdict(float)
gaps, cnt = 0.0, collections.Counter()
for (s0, e0, _), (s1, e1, _) in zip(main, main[1:]):
    g = s1 - e0
    if g <= 0.005:
        continue
    gaps += g
    last = [x for x in side if e0 - 1e-3 <= x[0] <= s1 + 1e-3]
    key = last[-1][1] if last else "none"
    stall[key] += g
    cnt[key] += 1
print(f"  main-stream idle gaps > 5 us: {gaps:.2f} ms")
for k, v in sorted(stall.items(), key=lambda kv: -kv[1]):
    print(f"    ended by {k:14s} {v:9.2f} ms over {cnt[k]} gaps")
