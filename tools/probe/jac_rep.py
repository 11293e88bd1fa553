"""Repeat one fuzz case R times; report sweeps, bitwise spread of sigma, failures."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import numpy as np
from test_gpu_fuzz import _case
import paper_1803_01982_b200 as ffb

A, k, l, b, p, g, s = _case(np.random.default_rng(777 + int(sys.argv[1])))
R = int(sys.argv[2])
first = None
for it in range(R):
    print("CALL", it, file=sys.stderr, flush=True)
    try:
        ap = ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=s)
    except Exception as e:
        print("it", it, "ERR", e, flush=True); continue
    sg = np.asarray(ap.s); R_ = np.asarray(ap.meta["srqr"].fact.R)
    if first is None:
        first = (sg, R_)
    print("it", it, "sweeps", ap.meta.get("svd_sweeps"), "ds", float(np.max(np.abs(sg - first[0]))),
          "dR", float(np.max(np.abs(R_ - first[1]))), flush=True)
