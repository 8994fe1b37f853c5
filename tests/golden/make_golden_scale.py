"""Golden vectors at (near) config scale, made by running the REFERENCE itself.

Run once in the build container (where /root/reference exists; ~30 min of
CPU on 8 cores):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_scale.py [case ...]

Each case is run TWICE through the reference: on A and on A with a 1-ulp
perturbation of every entry (A * (1 + eps) elementwise, rounded).  The
per-entry difference of the two runs is the reference's own rounding-noise
envelope at that size; the GPU parity tests (tests/test_gpu_scale.py) gate
against max(1e-10-relative, that envelope), so the envelope is measured, not
hard-coded.

The inputs are regenerated bit for bit on the GPU box (no /root/reference
there): A = PCG64(seed).standard_normal((m, n)) (numpy, C order) times an
exact power-of-two column scaling 2**-floor(steps*j/n), so nothing depends
on libm.  Only small summaries are committed: diag(T) / diag(R), the
Frobenius trailing curve e_k (bench.trailing_fro_curve, bench.py:63-72),
the first columns of U and V, and a checksum of A.

Cases (BASELINE configs they stand in for):
  rutv8192  randutv_basic(A, b=256, q=2, RngStream(3))  8192^2   (C3 at half size)
  purv2048  power_urv(A, q=2, RngStream(2))              2048^2   (C2; the reference
            needs ~40 min at 4096 and days at 8192)
  tall16k   power_urv_from_sample(A, q=1, G)              16384x256 (C4 shape family)
  tall32k   power_urv_from_sample(A, q=1, G)              32768x512 (C4 shape family)
"""

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (kind, m, n, params, seed_a, seed_g, steps)
    "rutv8192": ("randutv", 8192, 8192, dict(b=256, q=2), 30, 3, 20),
    "purv2048": ("powerurv", 2048, 2048, dict(q=2), 20, 2, 20),
    "tall16k": ("powerurv_g", 16384, 256, dict(q=1), 40, 4, 12),
    "tall32k": ("powerurv_g", 32768, 512, dict(q=1), 41, 4, 12),
}


def make_input(m, n, seed, steps):
    """Shared with tests/test_gpu_scale.py (regenerated there bit for bit)."""
    a = np.random.Generator(np.random.PCG64(seed)).standard_normal((m, n))
    scale = np.ldexp(1.0, -(np.arange(n) * steps // n))
    return np.asfortranarray(a * scale)


def checksum(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def perturb(a):
    eps = np.finfo(np.float64).eps
    return np.asfortranarray(a * (1.0 + eps))


def run_case(uk, name):
    kind, m, n, prm, sa, sg, steps = CASES[name]
    a = make_input(m, n, sa, steps)
    out = {}
    for tag, x in (("", a), ("_p", perturb(a))):
        t0 = time.time()
        if kind == "randutv":
            f = uk.randutv_basic(x, prm["b"], prm["q"], uk.RngStream(sg))
            t = f.T
            u, v = f.U, f.V
        elif kind == "powerurv":
            f = uk.power_urv(x, prm["q"], uk.RngStream(sg))
            t = f.R
            u, v = uk.materialize_q(f.Uq, 4), uk.materialize_q(f.Vq, 4)
        else:
            g = uk.RngStream(sg).standard_normal(n, n)
            f = uk.power_urv_from_sample(x, prm["q"], np.asfortranarray(g))
            t = f.R
            u, v = uk.materialize_q(f.Uq, 4), uk.materialize_q(f.Vq, 4)
        dt = time.time() - t0
        print(f"{name}{tag}: {dt:.1f} s", flush=True)
        out["diag" + tag] = np.diag(t).copy()
        out["efro" + tag] = ukb.trailing_fro_curve(t)
        out["U4" + tag] = np.array(u[:, :4])
        out["V4" + tag] = np.array(v[:, :4])
        out["secs" + tag] = dt
    np.savez_compressed(os.path.join(OUT, f"scale_{name}.npz"), kind=kind, m=m, n=n,
                        seed_a=sa, seed_g=sg, steps=steps, sha_a=checksum(a),
                        params=repr(prm), **out,
                        call=f"{kind} {prm} on make_input({m},{n},{sa},{steps}); "
                             f"_p = same on A*(1+eps)")
    print("wrote", name, flush=True)


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import utvkit as uk  # noqa: E402  (reference, read-only)
    global ukb
    from utvkit import bench as ukb  # noqa: E402
    names = sys.argv[1:] or list(CASES)
    for name in names:
        run_case(uk, name)


if __name__ == "__main__":
    main()
