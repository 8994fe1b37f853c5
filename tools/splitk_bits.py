"""Write the outputs of split-K GEMM shapes to an .npz (used by
tests/test_gpu_kernels.py to compare the fused split-K epilogue with the
separate reduce kernel, UTV_SPLITK_FUSE_MAX=0, bit for bit)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2106_13402_b200.device as dv  # noqa: E402
from paper_2106_13402_b200._lib import dfrom_numpy  # noqa: E402

SHAPES = [("T", "N", 256, 8192, 8192, 0.0), ("N", "N", 12000, 256, 12000, 1.0),
          ("T", "N", 256, 16384, 4096, -1.0), ("N", "T", 3000, 256, 9000, 0.5)]


def main(out):
    res = {}
    for i, (ta, tb, m, n, k, beta) in enumerate(SHAPES):
        rng = np.random.default_rng(i)
        a = rng.standard_normal((k, m) if ta == "T" else (m, k))
        b = rng.standard_normal((n, k) if tb == "T" else (k, n))
        c = dfrom_numpy(rng.standard_normal((m, n)))
        dv.gemm(ta, tb, 1.25, dfrom_numpy(a), dfrom_numpy(b), beta, c)
        res[f"c{i}"] = c.to_numpy()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
