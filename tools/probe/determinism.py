"""Bitwise determinism sweep: random fuzz cases, each run R times in one process."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import numpy as np
from test_gpu_fuzz import _case
import paper_1803_01982_b200 as ffb

S0 = int(sys.argv[1]); N = int(sys.argv[2]); R = int(sys.argv[3])
bad = 0
for sd in range(S0, S0 + N):
    A, k, l, b, p, g, s = _case(np.random.default_rng(sd))
    outs = []
    for _ in range(R):
        try:
            ap = ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=s)
            outs.append((np.asarray(ap.meta["srqr"].fact.R).copy(), np.asarray(ap.s).copy(), np.asarray(ap.u).copy()))
        except ffb.CertificationError:
            outs.append(None)
        except Exception as e:
            outs.append(type(e).__name__)
    ref = outs[0]
    for o in outs[1:]:
        same = (o is None and ref is None) or (isinstance(o, str) and o == ref) or (
            isinstance(o, tuple) and isinstance(ref, tuple) and all(np.array_equal(x, y) for x, y in zip(o, ref)))
        if not same:
            bad += 1
            print("NONDET seed", sd, A.shape, k, l, b, p, g, flush=True)
            break
print("determinism:", N, "cases x", R, "->", bad, "nondeterministic")
