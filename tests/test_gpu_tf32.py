"""GPU parity of the 3xTF32 tcgen05 GEMM (K10, fp32 variant of the WY/sampling
GEMMs): against a float64 numpy product of the same fp32 inputs, tolerance at
fp32 level (the tolerance a plain TF32 product would miss by ~100x)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 32), (1, 1, 1), (130, 70, 45), (512, 384, 1000), (1000, 257, 64), (2048, 512, 4096)]


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_sgemm_tf32x3_fp32_accuracy(ta, tb, shape):
    import torch
    import paper_2106_13402_b200.device as dv
    from paper_2106_13402_b200._lib import dfrom_numpy
    m, n, k = shape
    rng = np.random.default_rng(m + 3 * n + 7 * k + 2 * ta + tb)
    A = rng.standard_normal((k, m) if ta else (m, k)).astype(np.float32)
    B = rng.standard_normal((n, k) if tb else (k, n)).astype(np.float32)
    C0 = rng.standard_normal((m, n)).astype(np.float32)
    ref = (1.25 * ((A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64))
           - 0.5 * C0.astype(np.float64))
    C = dfrom_numpy(C0, dtype=torch.float32)
    dv.sgemm_tf32x3("T" if ta else "N", "T" if tb else "N", 1.25, dfrom_numpy(A, dtype=torch.float32),
                    dfrom_numpy(B, dtype=torch.float32), -0.5, C)
    torch.cuda.synchronize()
    out = C.to_numpy().astype(np.float64)
    # standard fp32 forward-error bound of a length-k dot product,
    # |err| <= c k u (|A||B|)_ij (u = 2^-24; the tensor-core accumulator does
    # not round to nearest, so the bound is the worst-case linear one); a
    # plain TF32 product (u = 2^-11) misses it by ~4 orders of magnitude
    u = 2.0 ** -24
    absab = np.abs(A.T if ta else A).astype(np.float64) @ np.abs(B.T if tb else B).astype(np.float64)
    bound = 2 * (k + 2) * u * (1.25 * absab + 0.5 * np.abs(C0)) + 1e-30
    assert np.all(np.abs(out - ref) <= bound), np.max(np.abs(out - ref) / bound)
