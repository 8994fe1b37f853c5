"""Generate golden vectors by running the REFERENCE package (utvkit) itself.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes small .npz fixtures next to this script.  The GPU box never reads
/root/reference; it only reads these committed fixtures.  Each fixture
records the reference call that produced it (``call`` key).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import utvkit as uk  # noqa: E402  (reference, read-only)

    def save(name, **kw):
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **kw)
        print("wrote", path, os.path.getsize(path), "bytes")

    # ---- hqr_full (qr.py:71-100) -----------------------------------------
    cases = {}
    rng = np.random.default_rng(11)
    cases["eye4"] = np.eye(4)
    cases["col34"] = np.array([[3.0], [4.0]])
    cases["rand100x60"] = rng.standard_normal((100, 60))
    rd = rng.standard_normal((40, 24))
    rd[:, 5] = 0.0                      # exactly zero column -> skip rule
    rd[:, 9] = rd[:, 2] * 2.0           # dependent column
    rd[:, 17:] = 0.0                    # trailing zero block
    cases["rankdef40x24"] = rd
    e1 = np.zeros((6, 3)); e1[0, 0] = 2.0; e1[1, 1] = -1.0; e1[:, 2] = 1.0
    cases["collinear6x3"] = e1          # sigma == 0 columns -> skip rule
    neg = rng.standard_normal((33, 33))
    neg[0, 0] = -abs(neg[0, 0]) * 10
    cases["square33"] = neg
    for key, a in cases.items():
        q, r = uk.hqr_full(a)
        save("hqr_" + key, A=a, Y=q.Y, Twy=q.Twy, R=r, call="hqr_full(A)")

    # ---- apply_q / materialize_q (qr.py:103-131) ------------------------
    a = rng.standard_normal((50, 30))
    q, _ = uk.hqr_full(a)
    bl = rng.standard_normal((50, 7))
    br = rng.standard_normal((9, 50))
    save("applyq_50x30", A=a, BL=bl, BR=br,
         left=uk.apply_q(q, bl, "left", False),
         left_t=uk.apply_q(q, bl, "left", True),
         right=uk.apply_q(q, br, "right", False),
         right_t=uk.apply_q(q, br, "right", True),
         Q=uk.materialize_q(q), Q30=uk.materialize_q(q, 30),
         call="apply_q / materialize_q on hqr_full(A)")

    # ---- svd_dense (svd.py:37-58) -------------------------------------
    svd_cases = {
        "diag321": np.diag([3.0, 2.0, 1.0]),
        "rand20": rng.standard_normal((20, 20)),
        "rank1": np.outer(rng.standard_normal(12), rng.standard_normal(12)),
        "zero5": np.zeros((5, 5)),
        "upper64": np.triu(rng.standard_normal((64, 64))),
        "tall30x8": rng.standard_normal((30, 8)),
    }
    for key, a in svd_cases.items():
        s = uk.svd_dense(a, mode="full")
        save("svd_" + key, A=a, U=s.U, sigma=s.sigma, V=s.V, call="svd_dense(A,'full')")

    # ---- power_urv_from_sample (powerurv.py:41-72) ----------------------
    purv = [("gauss120x80_q1", 120, 80, 1, 21), ("gauss96_q2", 96, 96, 2, 22),
            ("gauss64x48_q0", 64, 48, 0, 23), ("tall200x40_q2", 200, 40, 2, 24)]
    for key, m, n, qq, seed in purv:
        st = uk.RngStream(seed)
        a = uk.gaussian(m, n, st)
        g = uk.gaussian(n, n, st)
        f = uk.power_urv_from_sample(a, qq, g)
        save("purv_" + key, A=a, G=g, q=qq, Uy=f.Uq.Y, Ut=f.Uq.Twy, R=f.R,
             Vy=f.Vq.Y, Vt=f.Vq.Twy, call=f"power_urv_from_sample(A,{qq},G)")
    # power_urv with an RngStream: G is gaussian(n, n, rng) (powerurv.py:75-79)
    a, _ = uk.gen_fast_decay(80, 1e-5, uk.RngStream(5))
    f = uk.power_urv(a, 2, uk.RngStream(6))
    save("purv_fast80_q2_seed6", A=a, seed=6, q=2, Uy=f.Uq.Y, Ut=f.Uq.Twy,
         R=f.R, Vy=f.Vq.Y, Vt=f.Vq.Twy, call="power_urv(A,2,RngStream(6))")

    # ---- randutv_basic (randutv.py:110-193, 228-235) --------------------
    rutv = []
    st = uk.RngStream(31)
    rutv.append(("gauss150x100_b30_q1", uk.gaussian(150, 100, st), 30, 1, 32))
    rutv.append(("gauss300_b64_q1", uk.gaussian(300, 300, uk.RngStream(33)), 64, 1, 34))
    rutv.append(("tall300x260_b64_q2", uk.gaussian(300, 260, uk.RngStream(35)), 64, 2, 36))
    fd, _ = uk.gen_fast_decay(200, 1e-5, uk.RngStream(37))
    rutv.append(("fast200_b50_q2", fd, 50, 2, 38))
    rutv.append(("single64_b64_q1", uk.gaussian(64, 64, uk.RngStream(39)), 64, 1, 40))
    rutv.append(("gauss97_b16_q0", uk.gaussian(97, 97, uk.RngStream(41)), 16, 0, 42))
    rk = uk.gaussian(120, 30, uk.RngStream(43)) @ uk.gaussian(30, 120, uk.RngStream(44))
    rutv.append(("rank30_120_b32_q1", rk, 32, 1, 45))
    for key, a, b, qq, seed in rutv:
        f = uk.randutv_basic(a, b, qq, uk.RngStream(seed), record_trailing=True)
        save("rutv_" + key, A=a, b=b, q=qq, seed=seed, U=f.U, T=f.T, V=f.V,
             errors=np.array(f.errors), trailing=np.array(f.trailing_fro),
             steps=f.steps_done, efro=uk.bench.trailing_fro_curve(f.T),
             call=f"randutv_basic(A,{b},{qq},RngStream({seed}),record_trailing=True)")

    boosted(uk, save)


def boosted(uk=None, save=None):
    """randutv_boosted / randutv_partial (randutv.py:130-139, 196-264)."""
    if uk is None:
        sys.dont_write_bytecode = True
        sys.path.insert(0, REF)
        import utvkit as uk  # noqa: E402

        def save(name, **kw):
            path = os.path.join(OUT, name + ".npz")
            np.savez_compressed(path, **kw)
            print("wrote", path, os.path.getsize(path), "bytes")
    cases = []
    cases.append(("gauss150x100_b30_q1_p30", uk.gaussian(150, 100, uk.RngStream(51)), 30, 1, 30, 52, None, None))
    fd, _ = uk.gen_fast_decay(200, 1e-5, uk.RngStream(53))
    cases.append(("fast200_b50_q2_p20", fd, 50, 2, 20, 54, None, None))
    cases.append(("tall300x260_b64_q2_p64", uk.gaussian(300, 260, uk.RngStream(55)), 64, 2, 64, 56, None, None))
    cases.append(("gauss160_b32_q1_p0", uk.gaussian(160, 160, uk.RngStream(57)), 32, 1, 0, 58, None, None))
    cases.append(("gauss96_b40_q1_p16", uk.gaussian(96, 96, uk.RngStream(59)), 40, 1, 16, 60, None, None))
    cases.append(("partial_rank_tall300x260_b64_q1_p16", uk.gaussian(300, 260, uk.RngStream(61)), 64, 1, 16, 62, None, 100))
    cases.append(("partial_tol_fast200_b32_q2_p8", fd, 32, 2, 8, 63, 1e-3, None))
    for key, a, b, qq, pp, seed, tol, mr in cases:
        rng = uk.RngStream(seed)
        if key.startswith("partial"):
            f = uk.randutv_partial(a, b, qq, pp, rng, tol_fro=tol, max_rank=mr, record_trailing=True)
            call = f"randutv_partial(A,{b},{qq},{pp},RngStream({seed}),tol_fro={tol},max_rank={mr},record_trailing=True)"
        else:
            f = uk.randutv_boosted(a, b, qq, pp, rng, record_trailing=True)
            call = f"randutv_boosted(A,{b},{qq},{pp},RngStream({seed}),record_trailing=True)"
        nxt = rng.standard_normal(1, 1)[0, 0]      # rng consumption parity
        save("boost_" + key, A=a, b=b, q=qq, p=pp, seed=seed, tol=np.nan if tol is None else tol,
             max_rank=-1 if mr is None else mr, U=f.U, T=f.T, V=f.V, errors=np.array(f.errors),
             trailing=np.array(f.trailing_fro), steps=f.steps_done,
             efro=uk.bench.trailing_fro_curve(f.T), next_normal=nxt, call=call)


def matgen():
    """Reference generators (matgen.py) at small sizes."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import utvkit as uk  # noqa: E402
    a, d = uk.gen_fast_decay(64, 1e-3, uk.RngStream(71))
    b, e = uk.gen_s_shaped(48, uk.RngStream(72))
    q = uk.matgen.random_orthogonal(40, uk.RngStream(73))
    np.savez_compressed(os.path.join(OUT, "matgen_small.npz"), fast=a, fast_d=d, s=b, s_d=e,
                        bie=uk.gen_bie(20), kahan=uk.gen_kahan(12), kahan_th=uk.gen_kahan(9, 0.7),
                        orth=q, gauss=uk.gen_gaussian(10, uk.RngStream(74)),
                        call="gen_fast_decay(64,1e-3,RngStream(71)); gen_s_shaped(48,RngStream(72)); "
                             "random_orthogonal(40,RngStream(73)); gen_bie(20); gen_kahan(12); "
                             "gen_kahan(9,0.7); gen_gaussian(10,RngStream(74))")
    print("wrote matgen_small.npz")


def hqrcp():
    """Reference hqrcp (qr.py:152-204) on pivot-sensitive inputs."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import utvkit as uk  # noqa: E402
    rng = np.random.default_rng(91)
    cases = {}
    cases["gauss120x80"] = rng.standard_normal((120, 80))
    cases["wide60x90"] = rng.standard_normal((60, 90))
    cases["kahan100"] = uk.gen_kahan(100, 1.2)
    cases["fast100"] = uk.gen_fast_decay(100, 1e-9, uk.RngStream(92))[0]
    rd = rng.standard_normal((80, 60))
    rd[:, 3] = 0.0                          # zero column
    rd[:, 7] = rd[:, 1]                     # exact duplicate -> tie, leftmost wins
    rd[:, 11] = -rd[:, 1]
    rd[:, 20] = rd[:, 2] + 1e-9 * rd[:, 5]  # near-dependent -> downdate recompute
    rd[:, 40:] = rd[:, :20] @ rng.standard_normal((20, 20))  # rank 40ish
    cases["rankdef80x60"] = rd
    cases["equalcols30x12"] = np.ones((30, 12))
    cases["one1x1"] = np.array([[-2.5]])
    cases["row1x5"] = rng.standard_normal((1, 5))
    cases["col5x1"] = rng.standard_normal((5, 1))
    cases["zero6x4"] = np.zeros((6, 4))
    for name, a in cases.items():
        f = uk.hqrcp(a)
        np.savez_compressed(os.path.join(OUT, f"qrcp_{name}.npz"), a=a, Y=f.q.Y, Twy=f.q.Twy, R=f.R,
                            perm=f.perm, call="hqrcp(a)")
        print("wrote", name)


def rsvd():
    """Reference rsvd / projector_gap (rsvd.py:31-78) for SPEC acceptance 2:
    shared-G powerURV vs RSVD on a Gaussian 60x40 for every (ell, q)."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import utvkit as uk  # noqa: E402
    rng = uk.RngStream(81)
    a = uk.gen_gaussian(60, rng)[:, :40].copy(order="F")
    g = uk.gaussian(40, 40, rng)
    out = dict(A=a, G=g, ells=np.array([1, 5, 10, 20, 40]), qs=np.array([0, 1, 2]))
    for q in (0, 1, 2):
        urv = uk.power_urv_from_sample(a, q, g)
        for ell in (1, 5, 10, 20, 40):
            rs = uk.rsvd(a, g, ell, q)
            out[f"U_rsvd_q{q}_l{ell}"] = rs.U_rsvd
            out[f"sigma_q{q}_l{ell}"] = rs.sigma
            out[f"gap_q{q}_l{ell}"] = uk.projector_gap(uk.materialize_q(urv.Uq, ell), rs.U_rsvd, a)
    np.savez_compressed(os.path.join(OUT, "rsvd_gauss60x40.npz"),
                        call="rsvd(A,G,ell,q); projector_gap(materialize_q(power_urv_from_sample(A,q,G).Uq,ell),"
                             " U_rsvd, A)", **out)
    print("wrote rsvd_gauss60x40.npz")


def spec_acc5():
    """SPEC acceptance 5 as the reference computes it (the REF_ACC5 table in
    tests/test_gpu_spec.py): max_k e_k/sigma_{k+1} - 1 (spectral) of
    randutv_boosted(q=2, p=b) and randutv_basic(q=2), n=400, b=50, on
    gen_fast_decay(400, 1e-5, RngStream(200 + 10 s)), s = 0..4."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import utvkit as uk  # noqa: E402

    def curve(t):
        r = min(t.shape)
        return np.array([np.linalg.svd(t[k:r, k:], compute_uv=False)[0] if k < r else 0.0
                         for k in range(1, t.shape[1])])
    for s in range(5):
        seed = 200 + 10 * s
        a, sig = uk.gen_fast_decay(400, 1e-5, uk.RngStream(seed))
        opt = np.sort(sig)[::-1][1:]
        cb = curve(uk.randutv_boosted(a, 50, 2, 50, uk.RngStream(seed + 1)).T)
        cs = curve(uk.randutv_basic(a, 50, 2, uk.RngStream(seed + 1)).T)
        print(f"({np.max(cb / opt - 1)!r}, {np.max(cs / opt - 1)!r}),")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "spec_acc5":
        spec_acc5()
    elif len(sys.argv) > 1 and sys.argv[1] == "rsvd":
        rsvd()
    elif len(sys.argv) > 1 and sys.argv[1] == "hqrcp":
        hqrcp()
    elif len(sys.argv) > 1 and sys.argv[1] == "boosted":
        boosted()
    elif len(sys.argv) > 1 and sys.argv[1] == "matgen":
        matgen()
    else:
        main()
