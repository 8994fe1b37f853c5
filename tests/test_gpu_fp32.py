"""GPU tests of the fp32 randUTV variant (BASELINE C5: 3xTF32 tcgen05 GEMMs,
fp32 storage) on rank-deficient inputs, judged as SURVEY §8c prescribes for
fp32 (there is no fp32 oracle): e_k against Eckart-Young from the known
spectrum and against the fp64 oracle, normalised reconstruction and
orthogonality at the 1e-4 (fp32) level; diag(T) informational only."""
import numpy as np
import pytest

from oracle import utv_oracle as orc

pytestmark = pytest.mark.gpu


def _rank_deficient(n, r, seed):
    gen = orc.gaussian_stream(seed)
    u = orc.random_orthogonal_fast(n, gen)[:, :r]
    v = orc.random_orthogonal_fast(n, gen)[:, :r]
    d = 10.0 ** (-3.0 * np.arange(r) / max(r - 1, 1))
    return np.asfortranarray((u * d) @ v.T), d


@pytest.mark.parametrize("n,r,b,q", [(512, 60, 64, 2), (1024, 250, 128, 2), (1024, 300, 256, 1)])
def test_randutv_fp32_rank_deficient(n, r, b, q):
    import paper_2106_13402_b200 as pk
    a, d = _rank_deficient(n, r, 50 + n)
    f = pk.randutv_basic(a, b, q, pk.RngStream(5), record_trailing=True, dtype=np.float32)
    assert f.T.dtype == np.float32 and f.U.dtype == np.float32
    U, T, V = (x.astype(np.float64) for x in (f.U, f.T, f.V))
    anorm = np.linalg.norm(a)
    # normalised reconstruction and orthogonality (fp32 level)
    assert np.linalg.norm(a - U @ T @ V.T) / anorm < 1e-4   # BASELINE fp32 tolerance
    assert np.abs(U.T @ U - np.eye(n)).max() < 1e-4
    assert np.abs(V.T @ V - np.eye(n)).max() < 1e-4
    # e_k vs Eckart-Young (tail of the known spectrum) and vs the fp64 oracle
    ek = pk.trailing_fro_curve(T)            # e_k = ||T[k:, k:]||_F, k = 1, 2, ...
    tail = np.sqrt(np.concatenate([np.cumsum((d ** 2)[::-1])[::-1], np.zeros(n + 1)]))
    ey = tail[1: len(ek) + 1]                 # Eckart-Young optimum for rank k
    assert np.all(ek >= ey - 1e-5 * anorm)
    # fp32 unstabilised sampling loses directions below ~eps32^(1/(2q+1)) of
    # a block's top singular value (SURVEY §7 hard part 6): e_k stays within a
    # small factor of the optimum (SPEC's powerURV bound is 2 sigma_{k+1})
    assert np.mean(ek[: r] <= 2.0 * ey[: r] + 1e-5 * anorm) >= 0.9
    assert np.all(ek[: r] <= 4.0 * ey[: r] + 1e-5 * anorm)
    # past the numerical rank everything is fp32 noise
    assert ek[r + b] < 1e-5 * anorm
    assert np.abs(np.diag(T)[r + b:]).max() < 1e-5 * d[0]
