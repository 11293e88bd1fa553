import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import callers_oracle as co
import oracle
g = np.random.default_rng(5)
core = g.standard_normal((4, 3, 2))
Us = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in ((20, 4), (15, 3), (12, 2))]
L = g.standard_normal((60, 3)) @ g.standard_normal((3, 40))
# replay the oracle IALM to get the 3rd partial-SVD input
Ws = []
orig = co._shrink_spectrum
def spy(psvd, M, sv, mu):
    Ws.append((M.copy(), sv))
    return orig(psvd, M, sv, mu)
co._shrink_spectrum = spy
co.ialm_rpca(L, dict(svd_engine="flipflop", max_iter=3))
W, sv = Ws[2]
np.save(os.path.join(os.path.dirname(os.path.abspath(__file__)), "W_fail.npy"), W)
print("sv", sv, "W", W.shape)
if len(sys.argv) > 1:
    import paper_1803_01982_b200 as ffb
    for mode in ("trqrcp", "srqr", "ff"):
        prm = ffb.SketchParams(k=sv, l=39, b=32, p=5)
        try:
            if mode == "trqrcp":
                f = ffb.trqrcp(W, prm); print(mode, "ok finite R", np.isfinite(f.R).all(), "Y", np.isfinite(f.Y).all() if hasattr(f,'Y') else None)
                o = oracle.trqrcp(W, oracle.resolve(60, 40, sv, 39, 32, 5))
                print("  perm equal", np.array_equal(f.perm, o.perm), np.abs(f.R - o.R).max())
            elif mode == "srqr":
                r = ffb.srqr(W, prm); print(mode, "ok", r.cert)
            else:
                ap = ffb.flip_flop_srqr(W, sv, l=39); print(mode, "ok", ap.s)
        except Exception as e:
            print(mode, type(e).__name__, e)
    print("oracle", oracle.flip_flop(W, sv, l=39).s)
