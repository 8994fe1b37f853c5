import sys; sys.path.insert(0, ".")
import numpy as np, torch, json
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200 import _lib
from paper_2106_13402_b200._lib import dempty, dfrom_numpy
rng = np.random.default_rng(0)
for kind in ("graded", "gauss", "purv"):
    if kind == "graded":
        a = rng.standard_normal((16384, 256)) * np.logspace(0, -5, 256)
        p = dfrom_numpy(a); dv.geqrf(p); r = dempty(256, 256); dv.lacpy(p.sub(0, 0, 256, 256), r)
    else:
        r = dfrom_numpy(rng.standard_normal((256, 256)))
    for tr in (None, False):
        dv.gesvj(r, tr); torch.cuda.synchronize()
        _lib.profile_begin()
        for _ in range(5): out = dv.gesvj(r, tr)
        torch.cuda.synchronize()
        prof = _lib.profile_end()
        print(kind, tr, {k: round(v["ms"] / 5, 4) for k, v in prof.items() if v["count"]}, "sweeps", int(out[3].cpu()))
