"""Benchmark: powerURV (q=2) + randUTV basic (b=256, q=2) on a 16384^2 fp64
matrix on one B200 (BASELINE.json metric: "powerURV & randUTV seconds at
n=16384 fp64; FP64 TFLOP/s vs B200 peak").

One *step* = one randUTV(b=256, q=2) factorisation + one powerURV(q=2)
factorisation of the same synthetic matrix, inputs resident in HBM.
value = algorithmic FP64 FLOPs of both (SURVEY.md §8d model) / seconds.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload auto|headline|c2|c4|c5]

--gpus N > 1 without WORLD_SIZE in the environment re-launches this script
under torchrun (N ranks, 127.0.0.1 rendezvous, NCCL_DEBUG=INFO unless set).
With N > 1 ranks the primary line is the ROW-SHARDED C4 powerURV
(524288 x 4096, q=1, strong scaling: the rows are split over the ranks,
collectives inside libutvb200 over NCCL); the headline runs as independent
replicas in a nested secondary object (randUTV does not shard).
At N = 1 the headline is the primary line and a 1-GPU C4 run is nested as
the scaling base.
--impl reference times the GENUINE reference package (oracle/_ref, an
unmodified copy of utvkit made by oracle/build_ref.py; the numpy port
oracle/utv_oracle.py if the copy is absent) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1   # measured DMMA m8n8k4 peak on this pool's B200 (profiles/fp64_peak_r01.json)
# DRAM traffic of the representative WY-update launch (NT 16384x16384x256,
# beta=1), one `ncu --set full` capture: read + write bytes per launch vs the
# algorithmic bytes (A, B 32 MiB each + C read and written, 2 GiB each).
GEMM_TRAFFIC = {"bytes": 2.811756e9 + 2.102741e9, "algorithmic_bytes": 2 * 8 * 16384 * 256 + 2 * 8 * 16384 ** 2,
                "launch": "dgemm NT M=N=16384 K=256 beta=1 (compact-WY trailing update)",
                "source": "profiles/r02_ncu_gemm_nt_16384x16384x256_epilogue.txt"}
FP64_PEAK_SRC = "measured: tools/fp64_peak.cu DMMA m8n8k4, 148 SMs @1965 MHz (profiles/fp64_peak_r01.json)"
# dense TF32 tcgen05 peak (M=128, N=128 - K10's MMA shape), measured by
# tools/tf32_peak.cu (profiles/tf32_peak_r02.json); 3xTF32 does 3 MMAs per
# useful product, so the useful-FLOP roofline of K10 is a third of it
TF32_PEAK_TFLOPS = 1061.5
TF32_PEAK_SRC = ("measured: tools/tf32_peak.cu tcgen05.mma.cta_group::1.kind::tf32 M=128 N=128, "
                 "148 SMs @1965 MHz (profiles/tf32_peak_r02.json); useful peak = 1/3 (3xTF32)")


# ---------------------------------------------------------------------------
# FLOP models
# ---------------------------------------------------------------------------

def randutv_flops(m, n, b, q):
    """GEMM-phase algorithmic FLOPs of randUTV basic."""
    s = -(-n // b)
    f = 0.0
    for i in range(1, s):
        lo = (i - 1) * b
        kr, kc = m - lo, n - lo
        r = kc - b
        f += (2 + 4 * q) * kr * kc * b                      # sampling
        f += 4 * m * kc * b + 2 * m * b * b                 # T right
        f += 4 * n * kc * b + 2 * n * b * b                 # V right
        f += 4 * m * kr * b + 2 * m * b * b                 # U right
        f += 4 * kr * r * b + 2 * r * b * b                 # T left
        f += 2 * m * b * b + 2 * n * b * b + 2 * b * b * r + 2 * lo * b * b  # rotations
    lo = (s - 1) * b
    kr, kc = m - lo, n - lo
    f += 2 * m * kr * kr + 2 * n * kc * kc + 2 * lo * kc * kc
    return f


def powerurv_flops(m, n, q):
    """Algorithmic FLOPs of powerURV: q(8mn^2 + 4n^3/3) + 4mn^2 - 2n^3/3."""
    return q * (8.0 * m * n * n + 4.0 * n ** 3 / 3) + 4.0 * m * n * n - 2.0 * n ** 3 / 3


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_threads():
    return os.cpu_count() or 1


def _reference_impl():
    """(module, kind): the genuine reference copy (oracle/_ref) or the port."""
    from oracle import build_ref
    if build_ref.available():
        return build_ref.load(), "reference"
    from oracle import utv_oracle
    return None, "port"


def _ref_time_purv(uk, n, q=2, seed=0):
    a = np.random.default_rng(seed).standard_normal((n, n))
    if uk is None:
        from oracle import utv_oracle as orc
        g = orc.draw_gaussian(orc.gaussian_stream(2), n, n)
        t0 = time.perf_counter()
        orc.power_urv(a, q, g)
        return time.perf_counter() - t0
    t0 = time.perf_counter()
    uk.power_urv(a, q, uk.RngStream(2))                  # reference powerurv.py:75-79
    return time.perf_counter() - t0


def _ref_time_rutv(uk, n, b=256, q=2, seed=0):
    a = np.random.default_rng(seed).standard_normal((n, n))
    if uk is None:
        from oracle import utv_oracle as orc
        blocks = orc.randutv_sample_blocks(orc.gaussian_stream(3), n, n, b)
        t0 = time.perf_counter()
        orc.randutv_basic(a, b, q, blocks)
        return time.perf_counter() - t0
    t0 = time.perf_counter()
    uk.randutv_basic(a, b, q, uk.RngStream(3))           # reference randutv.py:228-235
    return time.perf_counter() - t0


#: bounded sample of the headline workload timed on the host cores
REF_RUTV_N, REF_PURV_N = 1536, 512


def cpu_sample_run(uk=None, kind=None, rutv_n=REF_RUTV_N, purv_n=REF_PURV_N, b=256, q=2):
    """One sample step of the reference on the host: randUTV(rutv_n) + powerURV(purv_n)."""
    if kind is None:
        uk, kind = _reference_impl()
    tr = _ref_time_rutv(uk, rutv_n, b, q)
    tp = _ref_time_purv(uk, purv_n, q)
    fl = randutv_flops(rutv_n, rutv_n, b, q) + powerurv_flops(purv_n, purv_n, q)
    src = ("oracle/_ref/utvkit (unmodified reference copy)" if kind == "reference"
           else "oracle/utv_oracle.py (numpy port)")
    return dict(seconds=tr + tp, flops=fl, rutv_s=tr, purv_s=tp, kind=kind,
                sample=f"randUTV b={b} q={q} n={rutv_n} + powerURV q={q} n={purv_n} on i.i.d. "
                       f"N(0,1) input (runtime is data-independent, PAPER.md:843); {src}, "
                       f"numpy {np.__version__}, OpenBLAS on all host threads")


def _fit_power_law(ns, ts):
    """t = c n^alpha by least squares in log-log space."""
    x, y = np.log(np.asarray(ns, float)), np.log(np.asarray(ts, float))
    alpha, logc = np.polyfit(x, y, 1)
    return float(np.exp(logc)), float(alpha)


def _ref_time_tall(uk, n, aspect=128, q=1, seed=0):
    """Reference power_urv_from_sample (powerurv.py:41-72) on a tall m = aspect*n matrix."""
    m = aspect * n
    a = np.random.default_rng(seed).standard_normal((m, n))
    if uk is None:
        from oracle import utv_oracle as orc
        g = orc.draw_gaussian(orc.gaussian_stream(4), n, n)
        t0 = time.perf_counter()
        orc.power_urv(a, q, g)
        return time.perf_counter() - t0
    g = np.asfortranarray(uk.RngStream(4).standard_normal(n, n))
    t0 = time.perf_counter()
    uk.power_urv_from_sample(a, q, g)
    return time.perf_counter() - t0


def _ladder_line(args, kind, metric, config, full_flops, sample_flops, timed, ladder_fits, extra):
    """Reference-arm JSON line: value = full-size FLOPs / extrapolated seconds."""
    t_full = sum(c * x ** al for (c, al, x) in ladder_fits)
    val = full_flops / t_full / 1e12
    tot = sum(timed)
    sample_val = sample_flops * len(timed) / tot / 1e12
    line = {
        "impl": "reference", "metric": metric, "value": val, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(timed), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "value_kind": "extrapolated to the full config from a measured ladder (t = c n^alpha fit "
                      "per algorithm, see 'ladder'); full-size CPU runs take hours to days",
        "sample_value": sample_val, "extrapolated_seconds": t_full,
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": kind,
                         "sample_value": sample_val},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    return line


def run_reference(args, wl="headline"):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return                                   # rank 0 alone runs the CPU arm
    uk, kind = _reference_impl()
    src = ("oracle/_ref/utvkit (unmodified reference copy)" if kind == "reference"
           else "oracle/utv_oracle.py (numpy port)")
    if wl == "c5":
        print(json.dumps({"impl": "reference", "unavailable": "the reference is fp64-only "
                          "(check_matrix casts to float64, matrix.py:42): no fp32 CPU path"}), flush=True)
        return
    if wl == "c4":
        m, n = args.c4_rows, args.c4_cols
        for _ in range(args.warmup):
            _ref_time_tall(uk, 64)
        timed = [_ref_time_tall(uk, 128) for _ in range(args.steps)]
        lad = {128: float(np.median(timed)), 192: _ref_time_tall(uk, 192), 256: _ref_time_tall(uk, 256)}
        c, al = _fit_power_law(list(lad), list(lad.values()))
        line = _ladder_line(
            args, kind, C4_METRIC,
            {"workload": f"C4 powerURV q=1 on {m}x{n} fp64 (reference: one process, host cores)"},
            powerurv_flops(m, n, 1), powerurv_flops(128 * 128, 128, 1), timed, [(c, al, n)],
            {"ladder": {"tall m=128n, q=1, n -> s": {k: round(v, 3) for k, v in lad.items()},
                        "fit": f"t = {c:.3g} n^{al:.2f}"},
             "sample": f"power_urv_from_sample q=1 on 16384x128 i.i.d. N(0,1); {src}"})
        print(json.dumps(line), flush=True)
        return
    if wl == "c2":
        n, q = 8192, 2
        for _ in range(args.warmup):
            _ref_time_purv(uk, 256, q)
        timed = [_ref_time_purv(uk, 384, q) for _ in range(args.steps)]
        lad = {256: _ref_time_purv(uk, 256, q), 384: float(np.median(timed)), 512: _ref_time_purv(uk, 512, q)}
        c, al = _fit_power_law(list(lad), list(lad.values()))
        line = _ladder_line(
            args, kind, C2_METRIC, {"workload": f"C2 powerURV q={q} on {n}x{n} fp64"},
            powerurv_flops(n, n, q), powerurv_flops(384, 384, q), timed, [(c, al, n)],
            {"ladder": {"powerURV q=2, n -> s": {k: round(v, 3) for k, v in lad.items()},
                        "fit": f"t = {c:.3g} n^{al:.2f}"},
             "sample": f"power_urv q=2 on 384x384 i.i.d. N(0,1); {src}"})
        print(json.dumps(line), flush=True)
        return
    n, b, q = args.n, args.b, args.q
    for _ in range(args.warmup):
        cpu_sample_run(uk, kind, rutv_n=768, purv_n=256, b=b, q=q)
    timed, tr, tp = [], [], []
    sample = None
    for _ in range(args.steps):
        r = cpu_sample_run(uk, kind, b=b, q=q)
        timed.append(r["seconds"])
        tr.append(r["rutv_s"])
        tp.append(r["purv_s"])
        sample = r["sample"]
    # ladder: two more sizes per algorithm, fitted t = c n^alpha,
    # extrapolated to the headline n (labelled as such; the full-size CPU runs
    # take ~35 min (randUTV) and days (powerURV) on these hosts)
    lad_r = {1024: _ref_time_rutv(uk, 1024, b, q), REF_RUTV_N: float(np.median(tr)),
             2048: _ref_time_rutv(uk, 2048, b, q)}
    lad_p = {384: _ref_time_purv(uk, 384, q), REF_PURV_N: float(np.median(tp)),
             768: _ref_time_purv(uk, 768, q)}
    cr, ar = _fit_power_law(list(lad_r), list(lad_r.values()))
    cp, apw = _fit_power_law(list(lad_p), list(lad_p.values()))
    c1 = _ref_time_rutv(uk, 2000, 128, 1)       # C1 (BASELINE configs[0]) timed directly
    line = _ladder_line(
        args, kind, METRIC, config_dict(args, 1),
        randutv_flops(n, n, b, q) + powerurv_flops(n, n, q),
        randutv_flops(REF_RUTV_N, REF_RUTV_N, b, q) + powerurv_flops(REF_PURV_N, REF_PURV_N, q),
        timed, [(cr, ar, n), (cp, apw, n)],
        {"ladder": {"randUTV b=256 q=2, n -> s": {k: round(v, 3) for k, v in lad_r.items()},
                    "randUTV fit": f"t = {cr:.3g} n^{ar:.2f} -> {cr * n ** ar:.0f} s at n={n}",
                    "powerURV q=2, n -> s": {k: round(v, 3) for k, v in lad_p.items()},
                    "powerURV fit": f"t = {cp:.3g} n^{apw:.2f} -> {cp * n ** apw:.0f} s at n={n}"},
         "sample": sample,
         "c1_seconds": c1,
         "c1": "randUTV b=128 q=1 on 2000x2000 (BASELINE configs[0]), measured directly"})
    print(json.dumps(line), flush=True)


METRIC = "powerURV(q=2)+randUTV(b=256,q=2) fp64 n=16384: FP64 TFLOP/s (algorithmic, SURVEY §8d)"


def config_dict(args, ws=None):
    ws = args.gpus if ws is None else ws
    return {"workload": f"powerURV q={args.q} + randUTV basic b={args.b} q={args.q} on "
                        f"{args.n}x{args.n} fp64 (BASELINE configs C3 + powerURV n=16384 target)",
            "n": args.n, "b": args.b, "q": args.q,
            "matrix": "A = Q1 diag(d) Q2^T, d_i = max(exp(-((i-1)/(n/4))^2), 1e-5) (Gaussian decay)",
            "l2_policy": "inputs (2 GiB/matrix) larger than the 126 MB L2; no explicit flush",
            "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def make_decay_matrix(n, seed):
    """Synthetic A = Q1 diag(d) Q2^T generated on the device with our own QR."""
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dempty
    gen = torch.Generator(device="cuda").manual_seed(seed)
    qs = []
    for _ in range(2):
        g = dempty(n, n)
        g.t.normal_(generator=gen)
        Y, T = dv.geqrf(g)
        qs.append(dv.orgqr(Y, T, n))
        del g, Y, T
    i = torch.arange(n, device="cuda", dtype=torch.float64)
    d = torch.clamp(torch.exp(-(i / (n / 4.0)) ** 2), min=1e-5)
    q1, q2 = qs
    q1.t[:, :n].mul_(d[:, None])                        # Q1 diag(d): scale columns
    a = dv.gemm("N", "T", 1.0, q1, q2)
    return a


def _init_dist(ws, local):
    import torch
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def _sync_all(ws):
    import torch
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
        torch.cuda.synchronize()


def _max_over_ranks(ws, x):
    if ws == 1:
        return x
    import torch
    tt = torch.tensor([x], device="cuda", dtype=torch.float64)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


def _lib_copy(src, dst):
    from paper_2106_13402_b200 import _lib
    _lib.check(_lib.load().utv_dlacpy(src.rows, src.cols, src.ptr, src.ld, dst.ptr, dst.ld,
                                      _lib.stream_ptr()), "utv_dlacpy")


def _lib_eye(m):
    from paper_2106_13402_b200 import _lib
    _lib.check(_lib.load().utv_dlaset(b"A", m.rows, m.cols, 0.0, 1.0, m.ptr, m.ld,
                                      _lib.stream_ptr()), "utv_dlaset")


def _panel_columns(n, b, q):
    """Householder columns factored by the panel kernel per headline step:
    randUTV 2 b-wide panels per regular step, powerURV (2q+1) n-wide QRs."""
    return 2 * b * (-(-n // b) - 1) + (2 * q + 1) * n


def kernel_entries(prof, step_s, n, b, q, sweeps):
    """Per-kernel figures of the non-GEMM kernels (panel QR
    algorithmic GB/s and us/column, Jacobi ms/call and sweeps, split-K share)."""
    pq, jr, jf, sk = prof["panel_qr"], prof["jacobi_rounds"], prof["jacobi_finish"], prof["splitk_reduce"]
    cols = _panel_columns(n, b, q)
    out = {
        "panel_qr": {"ms_per_step": pq["ms"], "launches": pq["count"],
                     "us_per_column": 1e3 * pq["ms"] / cols if cols else None,
                     "algorithmic_GBps": pq["bytes"] / (pq["ms"] / 1e3) / 1e9 if pq["ms"] else None,
                     "bytes_model": "8*3*rows*cols per panel (read A, write R and Y)",
                     "share_of_step": pq["ms"] / 1e3 / step_s},
        "jacobi": {"ms_per_step": jr["ms"] + jf["ms"], "calls": jr["count"],
                   "ms_per_call": (jr["ms"] + jf["ms"]) / max(jr["count"], 1),
                   "sweeps_mean": float(np.mean(sweeps)) if len(sweeps) else None,
                   "sweeps_max": int(np.max(sweeps)) if len(sweeps) else None},
        "splitk_reduce": {"ms_per_step": sk["ms"], "launches": sk["count"],
                          "share_of_step": sk["ms"] / 1e3 / step_s},
        "note": "panel_qr / jacobi ms are event intervals on their launching streams inside "
                "the step: the Jacobi SVDs run on a side stream sharing SMs with the GEMMs, "
                "so see 'isolated' for the kernels timed alone",
    }
    return out


def isolated_kernels(n_panel=16384, b=256, reps=3):
    """The two latency-bound kernels timed alone (CUDA events, after warm-up):
    one fused panel QR of an n_panel x b panel, and one b x b Jacobi SVD of a
    graded upper triangle (the R of a panel QR of a decaying matrix, what
    randUTV hands the SVD)."""
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dempty, dfrom_numpy

    def ev_time(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    rng = np.random.default_rng(0)
    p0 = dfrom_numpy(rng.standard_normal((n_panel, b)) * np.logspace(0, -5, b))
    work = dempty(n_panel, b)

    def panel():
        dv.lacpy(p0, work)
        dv.geqrf(work)
    t_panel = ev_time(panel)
    t_copy = ev_time(lambda: dv.lacpy(p0, work))
    dv.lacpy(p0, work)
    dv.geqrf(work)
    r = dempty(b, b)
    dv.lacpy(work.sub(0, 0, b, b), r)
    t_jac = ev_time(lambda: dv.gesvj(r))
    sweeps = int(dv.gesvj(r)[3].cpu().item())
    ms_panel = t_panel - t_copy
    return {"panel_qr": {"shape": f"{n_panel}x{b}", "call": "utv_dgeqrf (panel kernel + T)", "ms": ms_panel,
                         "us_per_column": 1e3 * ms_panel / b,
                         "algorithmic_GBps": 8.0 * 3 * n_panel * b / (ms_panel / 1e3) / 1e9},
            "jacobi": {"shape": f"{b}x{b} graded triangle", "ms_per_call": t_jac, "sweeps": sweeps}}


def run_ours(args, nested=False):
    import torch
    ws, rank, local = dist_env()
    _init_dist(ws, local)
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import dempty

    n, b, q = args.n, args.b, args.q
    steps, warmup = (1, 1) if nested else (args.steps, args.warmup)
    A = make_decay_matrix(n, seed=30 + rank)
    # Gaussian samples exactly as the reference draws them (host PCG64)
    rng = pk.RngStream(3)
    blocks = pk.randutv.draw_sample_blocks(rng, n, n, b)
    Gr = dv.stage_randutv_blocks(blocks, b)
    del blocks
    gp_host = pk.gaussian(n, n, pk.RngStream(2))
    Gp = _lib.dfrom_numpy(gp_host)
    del gp_host
    torch.cuda.synchronize()

    rrun = dv.RandUtvRun(n, n, b, q)
    prun = dv.PowerUrvRun(n, n, q)
    T = dempty(n, n)
    U = dempty(n, n)
    V = dempty(n, n)

    def rutv_step():
        _lib_copy(A, T)                 # randUTV works in place on T (randutv.py:114)
        _lib_eye(U)
        _lib_eye(V)
        rrun.run(T, U, V, Gr)

    def step():
        rutv_step()
        prun.run(A, Gp)

    for _ in range(warmup):
        step()
    _sync_all(ws)

    # per-algorithm split (untimed) + roofline inputs of the dominant kernel
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    _lib.profile_begin()
    e0.record()
    rutv_step()
    e1.record()
    prun.run(A, Gp)
    e2.record()
    prof = _lib.profile_end()
    rutv_s = e0.elapsed_time(e1) / 1e3
    purv_s = e1.elapsed_time(e2) / 1e3
    sweeps = rrun.status.cpu().numpy()
    _sync_all(ws)

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)
    _sync_all(ws)
    launches0 = _lib.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        step()
    t1.record()
    _sync_all(ws)
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    secs = _max_over_ranks(ws, t0.elapsed_time(t1) / 1e3)
    per_step = secs / steps
    f_rutv = randutv_flops(n, n, b, q)
    f_purv = powerurv_flops(n, n, q)
    flops = f_rutv + f_purv
    value = ws * flops / per_step / 1e12

    # ---- e2e through the public API (host numpy in, host numpy out) ----
    e2e = None
    if not args.no_e2e and not nested:
        a_host = A.to_numpy()
        a_host = np.asfortranarray(a_host)
        del T, U, V

        def e2e_step():
            fr = pk.randutv_basic(a_host, b, q, pk.RngStream(3))
            fp = pk.power_urv(a_host, q, pk.RngStream(2))
            del fr, fp

        # one untimed call (pinned rings, host thread pools, device buffers
        # in the caching allocator), then E2E_STEPS timed calls, wall clock
        e2e_step()
        torch.cuda.synchronize()
        e2e_steps = max(1, min(steps, 2))
        te = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = _max_over_ranks(ws, (time.perf_counter() - te) / e2e_steps)
        h2d = 8 * (2 * n * n + sum(k * b for k in range(n, b, -b)) + n * n)
        d2h = 8 * (3 * n * n + 5 * n * n) + 8 * (-(-n // b)) * 2
        e2e = {"value": ws * flops / e2e_s / 1e12, "unit": "TFLOP/s", "seconds": e2e_s,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": e2e_steps, "warmup": 1,
               "includes": "host PCG64 draws of G (reference RNG), H2D of A and G, device "
                           "factorisations, D2H of U,T,V and Uq,R,Vq (numpy results)"}

    g = prof["dgemm_dmma"]
    # GEMM flops over the union of GEMM launch intervals (all streams): the
    # side-stream U/V transforms run concurrently with main-stream GEMMs on a
    # CTA budget, so summing per-launch durations would double-count SM time
    gemm_busy_s = (g["busy_ms"] or g["ms"]) / 1e3
    gemm_tflops = g["flops"] / gemm_busy_s / 1e12 if gemm_busy_s > 0 else 0.0
    phase = {k: round(v["ms"], 3) for k, v in prof.items()}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu and not nested:
        r = cpu_sample_run()
        cpu = {"value": r["flops"] / r["seconds"] / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(),
               "kind": r["kind"], "sample": r["sample"], "seconds": r["seconds"]}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": steps,
        "warmup": warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated Gaussian-decay A; G from the reference PCG64 stream)",
        "config": config_dict(args, ws),
        "seconds": {"randutv": rutv_s, "powerurv": purv_s, "step": per_step},
        "tflops": {"randutv": f_rutv / rutv_s / 1e12, "powerurv": f_purv / purv_s / 1e12,
                   "algorithmic_over_peak": value / ws / FP64_PEAK_TFLOPS,
                   "note": "algorithmic_over_peak divides SURVEY §8d FLOPs (powerURV executes "
                           "~8n^3/3 fewer per round, csrc/powerurv.cu) by the peak; it is not a "
                           "utilisation figure - roofline.frac is"},
        "roofline": {"bound": "tensor", "kernel": "dgemm_tma_kernel (DMMA.8x8x4)",
                     "achieved": gemm_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": gemm_tflops / FP64_PEAK_TFLOPS, "traffic": GEMM_TRAFFIC["bytes"],
                     "traffic_note": GEMM_TRAFFIC,
                     "peak_source": FP64_PEAK_SRC,
                     "share_of_step": gemm_busy_s / (rutv_s + purv_s),
                     "achieved_method": "DMMA GEMM algorithmic flops / union of GEMM launch "
                                        "intervals over all streams (CUDA events, live)",
                     "sum_of_launch_ms": g["ms"],
                     "launches_per_step": g["count"]},
        "kernels": dict(kernel_entries(prof, rutv_s + purv_s, n, b, q, sweeps),
                        isolated=isolated_kernels(n, b) if not nested else None),
        "phase_ms": phase,
        "jacobi_sweeps": {"mean": float(np.mean(sweeps)), "max": int(np.max(sweeps))},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    del A, Gr, Gp, rrun, prun
    torch.cuda.empty_cache()
    if nested:
        return line
    if ws == 1 and not args.no_c4:
        line["c4"] = run_c4(args, nested=True)        # the 1-GPU base of the C4 scaling curve
    if rank == 0:
        print(json.dumps(line), flush=True)
    _finish_dist(ws)


def _finish_dist(ws):
    if ws > 1:
        import torch
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# C2: powerURV q=2 on 8192^2 (BASELINE configs[1])
# ---------------------------------------------------------------------------

C2_METRIC = "powerURV q=2 fp64 8192^2: FP64 TFLOP/s (algorithmic, SURVEY §8d)"


def run_c2(args):
    import torch
    ws, rank, local = dist_env()
    _init_dist(ws, local)
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200 import _lib
    n, q = 8192, 2
    A = make_decay_matrix(n, seed=20 + rank)
    Gp = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(2)))
    prun = dv.PowerUrvRun(n, n, q)
    for _ in range(args.warmup):
        prun.run(A, Gp)
    _sync_all(ws)
    _lib.profile_begin()
    prun.run(A, Gp)
    prof = _lib.profile_end()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        prun.run(A, Gp)
    t1.record()
    _sync_all(ws)
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    per = _max_over_ranks(ws, t0.elapsed_time(t1) / 1e3) / args.steps
    flops = powerurv_flops(n, n, q)
    g = prof["dgemm_dmma"]
    gb = (g["busy_ms"] or g["ms"]) / 1e3
    line = {"metric": C2_METRIC, "value": ws * flops / per / 1e12, "unit": "TFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated Gaussian-decay A, seed 20; G = RngStream(2))",
            "config": {"workload": f"C2 powerURV q={q} on {n}x{n} fp64",
                       "l2_policy": "inputs (512 MiB) larger than the 126 MB L2; no explicit flush",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "roofline": {"bound": "tensor", "kernel": "dgemm_tma_kernel (DMMA.8x8x4)",
                         "achieved": g["flops"] / gb / 1e12 if gb else 0.0, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": g["flops"] / gb / 1e12 / FP64_PEAK_TFLOPS if gb else 0.0,
                         "traffic": None, "share_of_step": gb / per},
            "phase_ms": {k: round(v["ms"], 3) for k, v in prof.items()},
            "gpu_launches": int(launches), "clocks": clk, "e2e": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    _finish_dist(ws)


# ---------------------------------------------------------------------------
# C4: row-sharded powerURV on a tall matrix (strong scaling over ranks)
# ---------------------------------------------------------------------------

C4_METRIC = "row-sharded powerURV q=1, 524288x4096 fp64: FP64 TFLOP/s (algorithmic, SURVEY §8d)"


def run_c4(args, nested=False):
    """C4 through the product path: utv_powerurv_sharded_f64 on every rank
    (collectives inside libutvb200: NCCL over the ranks' GPUs at N > 1)."""
    import torch
    ws, rank, local = dist_env()
    _init_dist(ws, local)
    from paper_2106_13402_b200 import sharded
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import dempty
    comm = sharded.NativeComm.nccl() if ws > 1 else sharded.NativeComm.local_group(1)[0]
    m, n, q = args.c4_rows, args.c4_cols, 1
    steps, warmup = (1, 1) if nested else (args.steps, args.warmup)
    rows = [m // ws + (1 if r < m % ws else 0) for r in range(ws)]
    gen = torch.Generator(device="cuda").manual_seed(40 + rank)
    a = dempty(rows[rank], n)
    a.t.normal_(generator=gen)                     # i.i.d. N(0,1) rows (PAPER.md:843 timing input)
    g = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(4)))
    torch.cuda.synchronize()

    def step():
        return sharded.power_urv_sharded_native(a, g, q, comm, chunk_rows=args.c4_chunk or None)

    for _ in range(warmup):
        out = step()
        del out
    _sync_all(ws)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        out = step()
        del out
    t1.record()
    _sync_all(ws)
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    per = _max_over_ranks(ws, t0.elapsed_time(t1) / 1e3) / steps
    flops = powerurv_flops(m, n, q)
    line = {"metric": C4_METRIC, "value": flops / per / 1e12, "unit": "TFLOP/s", "n_gpus": ws,
            "steps": steps, "warmup": warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device N(0,1) rows per rank; G from the reference PCG64 stream)",
            "config": {"workload": f"C4 powerURV q={q} on {m}x{n} fp64, row-sharded over {ws} rank(s)",
                       "rows_per_rank": rows, "tsqr_leaf_rows": args.c4_chunk or "panel limit",
                       "parallelism": f"row shards x{ws} (utv_powerurv_sharded_f64: NCCL allgather "
                                      f"+ allreduce + broadcast inside libutvb200)" if ws > 1
                                      else "1 GPU (utv_powerurv_sharded_f64, 1-rank communicator)",
                       "l2_policy": "inputs (16 GiB / ranks) larger than L2"},
            "frac_of_fp64_peak": flops / per / 1e12 / ws / FP64_PEAK_TFLOPS,
            "gpu_launches": int(launches), "clocks": clk, "e2e": None, "cpu_baseline": None}
    comm.close()
    del a, g
    torch.cuda.empty_cache()
    if nested:
        return line
    if ws > 1 and not args.no_replicas:
        line["headline_replicas"] = run_ours(args, nested=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    _finish_dist(ws)


# ---------------------------------------------------------------------------
# C5: fp32 randUTV (3xTF32 tensor cores) on a rank-deficient 32768^2 matrix
# ---------------------------------------------------------------------------

C5_METRIC = "randUTV b=512 q=2 fp32 (3xTF32 tcgen05), 32768^2 rank 2000: useful TFLOP/s (SURVEY §8d)"


def make_rank_deficient_f32(n, r, seed):
    """A = U_r diag(d) V_r^T, d_i = 10^(-3(i-1)/(r-1)), built on
    the device with our own QR / GEMM kernels, returned as fp32."""
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dempty
    gen = torch.Generator(device="cuda").manual_seed(seed)
    qs = []
    for _ in range(2):
        g = dempty(n, r)
        g.t.normal_(generator=gen)
        Y, T = dv.geqrf(g)
        qs.append(dv.orgqr(Y, T, r))
        del g, Y, T
    i = torch.arange(r, device="cuda", dtype=torch.float64)
    d = 10.0 ** (-3.0 * i / max(r - 1, 1))
    q1, q2 = qs
    q1.t[:r, :n].mul_(d[:, None])
    a64 = dv.gemm("N", "T", 1.0, q1, q2)
    del q1, q2, qs
    a = dempty(n, n, dtype=torch.float32)
    a.t[:, :n].copy_(a64.t[:, :n])
    del a64
    torch.cuda.empty_cache()
    return a


def run_c5(args):
    import torch
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import dempty
    from paper_2106_13402_b200.randutv import _eye32
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, b, q, r = args.c5_n, 512, 2, args.c5_rank
    A = make_rank_deficient_f32(n, r, 50 + rank)
    blocks = pk.randutv.draw_sample_blocks(pk.RngStream(5), n, n, b)
    G = dv.stage_randutv_blocks(blocks, b, dtype=torch.float32)
    del blocks
    run = dv.RandUtvRun32(n, n, b, q)
    T = dempty(n, n, dtype=torch.float32)
    U, V = _eye32(n), _eye32(n)
    lib = _lib.load()

    def eye32(m):
        _lib.check(lib.utv_slaset(b"A", m.rows, m.cols, 0.0, 1.0, m.ptr, m.ld, _lib.stream_ptr()),
                   "utv_slaset")

    def step():
        T.t.copy_(A.t)
        eye32(U)
        eye32(V)
        run.run(T, U, V, G)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _lib.profile_begin()
    step()
    prof = _lib.profile_end()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    secs = t0.elapsed_time(t1) / 1e3
    if ws > 1:
        tt = torch.tensor([secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        secs = float(tt.item())
    per = secs / args.steps
    flops = randutv_flops(n, n, b, q)
    g = prof["sgemm_tf32x3"]
    line = {"metric": C5_METRIC, "value": ws * flops / per / 1e12, "unit": "TFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xTF32)",
            "data": "synthetic rank-deficient (device-generated U_r diag(d) V_r^T; G from the reference PCG64 stream)",
            "config": {"workload": f"C5 randUTV b={b} q={q} fp32 on {n}x{n}, rank {r}",
                       "l2_policy": "inputs (4 GiB) larger than L2",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "roofline": {"bound": "tensor",
                         "kernel": "sgemm_tf32x3_kernel (tcgen05.mma kind::tf32, 3 products)",
                         "achieved": g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0,
                         "peak": TF32_PEAK_TFLOPS / 3, "unit": "TFLOP/s (useful)",
                         "frac": (g["flops"] / (g["ms"] / 1e3) / 1e12) / (TF32_PEAK_TFLOPS / 3)
                         if g["ms"] > 0 else 0.0,
                         "peak_source": TF32_PEAK_SRC, "traffic": None,
                         "share_of_step": g["ms"] / 1e3 / per},
            "phase_ms": {k: round(v["ms"], 3) for k, v in prof.items()},
            "gpu_launches": int(launches), "clocks": clk, "e2e": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def _spawn_ranks(n):
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--q", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="N=1: skip the nested 1-GPU C4 run")
    ap.add_argument("--no-replicas", action="store_true", help="N>1: skip the nested headline replicas")
    ap.add_argument("--workload", choices=["auto", "headline", "c2", "c4", "c5"], default="auto",
                    help="auto = headline at N=1, row-sharded C4 at N>1; "
                         "headline = BASELINE metric (n=16384 powerURV + randUTV); "
                         "c2 = powerURV q=2 8192^2 (BASELINE configs[1]); "
                         "c4 = row-sharded tall powerURV (BASELINE configs[3]); "
                         "c5 = fp32 3xTF32 randUTV (BASELINE configs[4])")
    ap.add_argument("--c5-n", type=int, default=32768)
    ap.add_argument("--c5-rank", type=int, default=2000)
    ap.add_argument("--c4-rows", type=int, default=524288)
    ap.add_argument("--c4-cols", type=int, default=4096)
    ap.add_argument("--c4-chunk", type=int, default=0,
                    help="TSQR leaf rows (0 = the panel kernel's limit, 75776)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args.gpus))
    os.environ.setdefault("NCCL_DEBUG", "INFO")       # rank count visible in the NCCL log
    ws = dist_env()[0]
    wl = args.workload if args.workload != "auto" else ("headline" if ws == 1 else "c4")
    if args.impl == "reference":
        run_reference(args, wl)
    elif wl == "c4":
        run_c4(args)
    elif wl == "c5":
        run_c5(args)
    elif wl == "c2":
        run_c2(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
