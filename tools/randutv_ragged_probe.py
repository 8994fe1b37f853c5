import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2106_13402_b200 as pk
from oracle import utv_oracle as orc
for (m, n, b) in [(1003, 513, 256), (1003, 512, 256), (1003, 514, 256), (1004, 513, 256), (600, 257, 128)]:
    a, d = orc.decay_matrix(n, 1e-5, seed=m + b, m=m)
    ref = orc.randutv_basic(a, b, 2, orc.randutv_sample_blocks(orc.gaussian_stream(b), m, n, b))
    f = pk.randutv_basic(a, b, 2, pk.RngStream(b))
    dt = np.abs(np.diag(f.T) - np.diag(ref["T"]))
    tol = 1e-10 * np.abs(np.diag(ref["T"])) + 16 * orc.EPS * d[0]
    bad = np.nonzero(dt > tol)[0]
    print(m, n, b, "bad idx", bad[:10], "diffs", dt[bad[:5]], "ref", np.diag(ref["T"])[bad[:5]], "ours", np.diag(f.T)[bad[:5]], flush=True)
