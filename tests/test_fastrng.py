"""The parallel host Gaussian generator (csrc/rng_host.cu via fastrng) must
reproduce numpy's Generator(PCG64(seed)).standard_normal bit for bit — the
reference's G (matrix.py:16-33) — and leave the generator in the same state.
CPU only (host code in libutvb200.so)."""
import numpy as np
import pytest

from paper_2106_13402_b200 import fastrng


def test_native_generator_enabled():
    assert fastrng.enabled()


@pytest.mark.parametrize("seed", [0, 3, 2 ** 63 + 11])
@pytest.mark.parametrize("shape", [(1, 1), (513, 257), (2048, 1024), (4096, 2500)])
def test_bit_identical_to_numpy(seed, shape):
    ref = np.random.Generator(np.random.PCG64(seed))
    mine = np.random.Generator(np.random.PCG64(seed))
    want = ref.standard_normal(shape)
    got = fastrng.standard_normal(mine, shape)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert mine.bit_generator.state == ref.bit_generator.state
    # the stream continues identically
    assert np.array_equal(mine.standard_normal(5000), ref.standard_normal(5000))


def test_blocked_draws_equal_bulk_draw():
    """randUTV draws one block per step (randutv.py:189): blockwise == bulk."""
    ref = np.random.Generator(np.random.PCG64(31))
    bulk = ref.standard_normal(3 * 300_000)
    mine = np.random.Generator(np.random.PCG64(31))
    parts = [fastrng.standard_normal(mine, (300_000,)) for _ in range(3)]
    assert np.array_equal(np.concatenate(parts), bulk)


def test_rngstream_uses_same_stream():
    import paper_2106_13402_b200 as pk
    a = pk.RngStream(9).standard_normal(1200, 700)
    b = np.random.Generator(np.random.PCG64(9)).standard_normal((1200, 700))
    assert np.array_equal(a, b)
