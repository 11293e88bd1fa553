import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import nuclear as N
g = np.random.default_rng(5)
core = g.standard_normal((4, 3, 2))
Us = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in ((20, 4), (15, 3), (12, 2))]
L = g.standard_normal((60, 3)) @ g.standard_normal((3, 40))
orig = N._shrink_spectrum
def spy(psvd, W, sv, mu):
    print("iter: sv", sv, "mu", mu, "W finite", bool(torch.isfinite(W).all()), "W max", float(W.abs().max()))
    try:
        X, k = orig(psvd, W, sv, mu)
    except Exception as e:
        Wn = W.cpu().numpy()
        np.save("/tmp/W_fail.npy", Wn)
        print("FAIL", e, "sv", sv)
        import oracle
        o = oracle.flip_flop(Wn, sv, l=min(sv + 60, 39))
        print("oracle s", o.s[:6])
        raise
    print("   keep", k, "X finite", bool(torch.isfinite(X).all()))
    return X, k
N._shrink_spectrum = spy
try:
    st = N.ialm_rpca(L, N.IalmParams(svd_engine="flipflop", max_iter=10))
    print(st.iterations, st.rank, st.residuals[-1])
except Exception as e:
    print("ERR", e)
