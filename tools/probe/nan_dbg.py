import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
import paper_1803_01982_b200 as ffb
from golden_io import load
c = load("cfg5_small")
ap = ffb.flip_flop_srqr(c["A"], c["k"], l=c["l"], b=c["b"], p=c["p"], seed=c["seed"])
print("warm ok")
A = np.random.default_rng(0).standard_normal((60, 40)); A[3, 5] = np.nan
for name, f in (("trqrcp", lambda: ffb.trqrcp(A, ffb.SketchParams(k=5, l=8))),
                ("srqr", lambda: ffb.srqr(A, ffb.SketchParams(k=5, l=8))),
                ("ff", lambda: ffb.flip_flop_srqr(A, 5, l=8))):
    try:
        f(); print(name, "no error")
    except Exception as e:
        print(name, type(e).__name__, str(e)[:150])
