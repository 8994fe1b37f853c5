import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2106_13402_b200.device as dv
from paper_2106_13402_b200._lib import dfrom_numpy
rng = np.random.default_rng(0)
for n, kind in [(512, "graded"), (512, "rankdef"), (256, "gauss_decay"), (512, "gauss")]:
    if kind == "graded":
        d = 10.0 ** (-3.0 * np.arange(n) / (n - 1))
    elif kind == "rankdef":
        d = np.concatenate([10.0 ** (-3.0 * np.arange(300) / 299), 1e-7 * np.ones(n - 300)])
    elif kind == "gauss_decay":
        d = np.maximum(np.exp(-(np.arange(n) / (n / 4)) ** 2), 1e-5)
    else:
        d = np.ones(n)
    q1, _ = np.linalg.qr(rng.standard_normal((n, n))); q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (q1 * d) @ q2.T
    # like randUTV: R of a QR of a sampled panel (A times a Gaussian-ish rotation) -> graded upper triangular
    _, r = np.linalg.qr(a @ q2)
    for name, m in [("R", r), ("R^T", r.T.copy())]:
        sig, U, V, st = dv.gesvj(dfrom_numpy(np.asfortranarray(m)))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dv.gesvj(dfrom_numpy(np.asfortranarray(m))); e1.record(); torch.cuda.synchronize()
        print(n, kind, name, "sweeps", int(st.item()), f"{e0.elapsed_time(e1):.2f} ms", flush=True)
