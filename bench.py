"""Benchmark: powerURV (q=2) + randUTV basic (b=256, q=2) on a 16384^2 fp64
matrix on one B200 (BASELINE.json metric: "powerURV & randUTV seconds at
n=16384 fp64; FP64 TFLOP/s vs B200 peak").

One *step* = one randUTV(b=256, q=2) factorisation + one powerURV(q=2)
factorisation of the same synthetic matrix, inputs resident in HBM.
value = algorithmic FP64 FLOPs of both (SURVEY.md §8d model) / seconds.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): randUTV does not shard -> every rank runs an
independent replica ("replicas only"; scaling "weak"), timed max over ranks.
--impl reference times the reference algorithm on the host cores (the CPU
oracle port, oracle/utv_oracle.py) on a bounded sample of the workload.
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
GEMM_TRAFFIC = {"bytes": 2.821095e9 + 2.106140e9, "algorithmic_bytes": 2 * 8 * 16384 * 256 + 2 * 8 * 16384 ** 2,
                "launch": "dgemm NT M=N=16384 K=256 beta=1 (compact-WY trailing update)",
                "source": "profiles/r01_ncu_gemm_nt_16384x16384x256_v4.txt"}
FP64_PEAK_SRC = "measured: tools/fp64_peak.cu DMMA m8n8k4, 148 SMs @1965 MHz (profiles/fp64_peak_r01.json)"


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


def cpu_sample_run(rutv_n=1536, purv_n=512, b=256, q=2, seed=0):
    """Reference algorithm (CPU oracle port) on a bounded sample; returns dict."""
    from oracle import utv_oracle as orc
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((rutv_n, rutv_n))
    blocks = orc.randutv_sample_blocks(orc.gaussian_stream(3), rutv_n, rutv_n, b)
    t0 = time.perf_counter()
    orc.randutv_basic(a, b, q, blocks)
    t1 = time.perf_counter()
    ap = rng.standard_normal((purv_n, purv_n))
    g = orc.draw_gaussian(orc.gaussian_stream(2), purv_n, purv_n)
    t2 = time.perf_counter()
    orc.power_urv(ap, q, g)
    t3 = time.perf_counter()
    fl = randutv_flops(rutv_n, rutv_n, b, q) + powerurv_flops(purv_n, purv_n, q)
    return dict(seconds=(t1 - t0) + (t3 - t2), flops=fl, rutv_s=t1 - t0, purv_s=t3 - t2,
                sample=f"randUTV b={b} q={q} n={rutv_n} + powerURV q={q} n={purv_n}, "
                       f"oracle/utv_oracle.py (numpy {np.__version__}, OpenBLAS threads)")


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    for _ in range(args.warmup):
        cpu_sample_run()
    tot_s, tot_f = 0.0, 0.0
    sample = None
    for _ in range(args.steps):
        r = cpu_sample_run()
        tot_s += r["seconds"]
        tot_f += r["flops"]
        sample = r["sample"]
    val = tot_f / tot_s / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


METRIC = "powerURV(q=2)+randUTV(b=256,q=2) fp64 n=16384: FP64 TFLOP/s (algorithmic, SURVEY §8d)"


def config_dict(args):
    return {"workload": f"powerURV q={args.q} + randUTV basic b={args.b} q={args.q} on "
                        f"{args.n}x{args.n} fp64 (BASELINE configs C3 + powerURV n=16384 target)",
            "n": args.n, "b": args.b, "q": args.q,
            "matrix": "A = Q1 diag(d) Q2^T, d_i = max(exp(-((i-1)/(n/4))^2), 1e-5) (Gaussian decay)",
            "l2_policy": "inputs (2 GiB/matrix) larger than the 126 MB L2; no explicit flush",
            "parallelism": f"replicas x{args.gpus}" if args.gpus > 1 else "1 GPU"}


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


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_13402_b200 as pk
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import deye, dempty

    n, b, q = args.n, args.b, args.q
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
    eye_idx = torch.arange(n, device="cuda")

    def step():
        T.t.copy_(A.t)
        U.t.zero_()
        U.t[eye_idx, eye_idx] = 1.0
        V.t.zero_()
        V.t[eye_idx, eye_idx] = 1.0
        rrun.run(T, U, V, Gr)
        prun.run(A, Gp)

    def sync_all():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    sync_all()

    # per-algorithm split (untimed) + roofline inputs of the dominant kernel
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    _lib.profile_begin()
    e0.record()
    T.t.copy_(A.t); U.t.zero_(); U.t[eye_idx, eye_idx] = 1.0; V.t.zero_(); V.t[eye_idx, eye_idx] = 1.0
    rrun.run(T, U, V, Gr)
    e1.record()
    prun.run(A, Gp)
    e2.record()
    prof = _lib.profile_end()
    rutv_s = e0.elapsed_time(e1) / 1e3
    purv_s = e1.elapsed_time(e2) / 1e3
    sweeps = rrun.status.cpu().numpy()
    sync_all()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)
    sync_all()
    launches0 = _lib.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    sync_all()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    secs = t0.elapsed_time(t1) / 1e3
    if ws > 1:
        tt = torch.tensor([secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        secs = float(tt.item())
    per_step = secs / args.steps
    f_rutv = randutv_flops(n, n, b, q)
    f_purv = powerurv_flops(n, n, q)
    flops = f_rutv + f_purv
    value = ws * flops / per_step / 1e12

    # ---- e2e through the public API (host numpy in, host numpy out) ----
    e2e = None
    if not args.no_e2e:
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
        e2e_steps = max(1, min(args.steps, 2))
        te = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - te) / e2e_steps
        if ws > 1:
            tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(tt.item())
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
    if rank == 0 and not args.no_cpu:
        r = cpu_sample_run()
        cpu = {"value": r["flops"] / r["seconds"] / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(),
               "kind": "port", "sample": r["sample"], "seconds": r["seconds"]}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated Gaussian-decay A; G from the reference PCG64 stream)",
        "config": config_dict(args),
        "seconds": {"randutv": rutv_s, "powerurv": purv_s, "step": per_step},
        "tflops": {"randutv": f_rutv / rutv_s / 1e12, "powerurv": f_purv / purv_s / 1e12,
                   "frac_of_fp64_peak": value / ws / FP64_PEAK_TFLOPS},
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
        "phase_ms": phase,
        "jacobi_sweeps": {"mean": float(np.mean(sweeps)), "max": int(np.max(sweeps))},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# C4: row-sharded powerURV on a tall matrix (strong scaling over ranks)
# ---------------------------------------------------------------------------

C4_METRIC = "row-sharded powerURV q=1, 524288x4096 fp64: FP64 TFLOP/s (algorithmic, SURVEY §8d)"


def run_c4(args):
    import torch
    ws, rank, local = dist_env()
    from paper_2106_13402_b200 import sharded
    import paper_2106_13402_b200 as pk
    from paper_2106_13402_b200 import _lib
    from paper_2106_13402_b200._lib import dempty
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = sharded.TorchComm()
    else:
        comm = sharded.Comm()
    m, n, q = args.c4_rows, args.c4_cols, 1
    rows = [m // ws + (1 if r < m % ws else 0) for r in range(ws)]
    gen = torch.Generator(device="cuda").manual_seed(40 + rank)
    a = dempty(rows[rank], n)
    a.t.normal_(generator=gen)                     # i.i.d. N(0,1) rows (PAPER.md:843 timing input)
    g = _lib.dfrom_numpy(pk.gaussian(n, n, pk.RngStream(4)))
    torch.cuda.synchronize()

    def step():
        return sharded.power_urv_sharded(a, g, q, comm)

    def sync_all():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        out = step()
        del out
    sync_all()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        out = step()
        del out
    t1.record()
    sync_all()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    secs = t0.elapsed_time(t1) / 1e3
    if ws > 1:
        tt = torch.tensor([secs], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        secs = float(tt.item())
    per = secs / args.steps
    flops = powerurv_flops(m, n, q)
    line = {"metric": C4_METRIC, "value": flops / per / 1e12, "unit": "TFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device N(0,1) rows per rank; G from the reference PCG64 stream)",
            "config": {"workload": f"C4 powerURV q={q} on {m}x{n} fp64, row-sharded over {ws} rank(s)",
                       "rows_per_rank": rows, "parallelism": f"row shards x{ws} (NCCL allreduce + TSQR)",
                       "l2_policy": "inputs (16 GiB / ranks) larger than L2"},
            "frac_of_fp64_peak": flops / per / 1e12 / ws / FP64_PEAK_TFLOPS,
            "gpu_launches": int(launches), "clocks": clk, "e2e": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


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
    idx = torch.arange(n, device="cuda")

    def step():
        T.t.copy_(A.t)
        U.t.zero_(); U.t[idx, idx] = 1.0
        V.t.zero_(); V.t[idx, idx] = 1.0
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
            "roofline": {"kernel": "sgemm_tf32x3_kernel (tcgen05.mma kind::tf32, 3 products)",
                         "achieved_useful_tflops": g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0,
                         "share_of_step": g["ms"] / 1e3 / per},
            "phase_ms": {k: round(v["ms"], 3) for k, v in prof.items()},
            "gpu_launches": int(launches), "clocks": clk, "e2e": None, "cpu_baseline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


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
    ap.add_argument("--workload", choices=["headline", "c4", "c5"], default="headline",
                    help="headline = BASELINE metric (n=16384 powerURV + randUTV); "
                         "c4 = row-sharded tall powerURV (BASELINE configs[3]); "
                         "c5 = fp32 3xTF32 randUTV (BASELINE configs[4])")
    ap.add_argument("--c5-n", type=int, default=32768)
    ap.add_argument("--c5-rank", type=int, default=2000)
    ap.add_argument("--c4-rows", type=int, default=524288)
    ap.add_argument("--c4-cols", type=int, default=4096)
    args = ap.parse_args()
    if args.workload == "c4" and args.impl != "reference":
        run_c4(args)
    elif args.workload == "c5" and args.impl != "reference":
        run_c5(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
