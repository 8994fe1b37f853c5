"""Quick device timings of the kernels and drivers (CUDA events)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dempty, deye
from paper_2106_13402_b200 import randutv as ru

def ev_time(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)

def rnd(m, n):
    d = dempty(m, n); d.t.normal_(); return d

out = {}
which = sys.argv[1:] or ["gemm", "qr", "svd", "rutv"]
if "gemm" in which:
    for (ta, tb, m, n, k) in [("N","N",8192,8192,8192), ("T","N",8192,8192,8192), ("N","T",8192,8192,8192), ("T","T",8192,8192,8192),
                              ("T","T",16384,256,16384), ("N","N",16384,256,16384), ("T","N",16384,256,16384),
                              ("N","T",16384,16384,256), ("N","N",16384,256,256), ("T","N",256,16384,16384), ("T","N",4096,256,4096)]:
        A = rnd(k, m) if ta == "T" else rnd(m, k)
        B = rnd(n, k) if tb == "T" else rnd(k, n)
        C = rnd(m, n)
        t = ev_time(lambda: dv.gemm(ta, tb, 1.0, A, B, 1.0, C))
        out[f"gemm_{ta}{tb}_{m}x{n}x{k}"] = dict(s=t, tflops=2*m*n*k/t/1e12); print(f"gemm_{ta}{tb}_{m}x{n}x{k}", out[f"gemm_{ta}{tb}_{m}x{n}x{k}"], flush=True)
        del A, B, C
if "qr" in which:
    for (m, n) in [(16384, 256), (8192, 256), (2048, 256), (4096, 4096), (8192, 8192)]:
        A = rnd(m, n)
        def f():
            B = dempty(m, n); B.t.copy_(A.t); dv.geqrf(B)
        t = ev_time(f, 2)
        out[f"geqrf_{m}x{n}"] = dict(s=t, tflops=(2*m*n*n - 2*n**3/3)/t/1e12); print(m, n, out[f"geqrf_{m}x{n}"], flush=True)
if "svd" in which:
    for n in [64, 128, 256]:
        A = rnd(n, n); A.t.triu_()
        t = ev_time(lambda: dv.gesvj(A))
        sig, U, V, st = dv.gesvj(A)
        out[f"gesvj_{n}"] = dict(s=t, sweeps=int(st.cpu().item())); print(n, out[f"gesvj_{n}"], flush=True)
if "rutv" in which:
    for (n, b, q) in [(2048, 128, 1), (4096, 256, 2), (8192, 256, 2)]:
        T0 = rnd(n, n)
        steps = -(-n // b)
        G = rnd(b, sum(n - i*b for i in range(steps - 1)))
        run = dv.RandUtvRun(n, n, b, q)
        def f():
            T = dempty(n, n); T.t.copy_(T0.t); U = deye(n); V = deye(n)
            run.run(T, U, V, G)
        t = ev_time(f, 2)
        out[f"randutv_{n}_b{b}_q{q}"] = dict(s=t, sweeps=run.status.cpu().tolist()[:4]); print(n, b, q, out[f"randutv_{n}_b{b}_q{q}"], flush=True)
if "qrcp" in which:
    for n in [1024, 4096, 8192, 16384]:
        A = rnd(n, n)
        def f():
            B = dempty(n, n); B.t.copy_(A.t); dv.geqp3(B)
        t = ev_time(f, 2)
        by = sum(16.0 * (n - j) * (n - j - 1) for j in range(n))
        out[f"geqp3_{n}"] = dict(s=t, gbs=by / t / 1e9); print("geqp3", n, out[f"geqp3_{n}"], flush=True)
        del A
print(json.dumps(out, indent=1))
