import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1803_01982_b200 as ffb
import oracle
g = np.random.default_rng(5)
core = g.standard_normal((4, 3, 2))
Us = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in ((20, 4), (15, 3), (12, 2))]
L = g.standard_normal((60, 3)) @ g.standard_normal((3, 40))
for l in (5, 10, 20, 39):
    prm = ffb.SketchParams(k=min(10, l), l=l, b=32, p=5)
    try:
        f = ffb.trqrcp(L, prm)
        print("l", l, "trqrcp ok", np.isfinite(f.R).all(), np.abs(np.diag(f.R[:, :l])).min())
    except Exception as e:
        print("l", l, "trqrcp", type(e).__name__, e)
    try:
        r = ffb.srqr(L, prm)
        print("   srqr ok", r.cert)
    except Exception as e:
        print("   srqr", type(e).__name__, e)
    try:
        ap = ffb.flip_flop_srqr(L, min(10, l), l=l)
        print("   ff ok", ap.s[:5])
    except Exception as e:
        print("   ff", type(e).__name__, e)
    o = oracle.flip_flop(L, min(10, l), l=l)
    print("   oracle", o.s[:5])
