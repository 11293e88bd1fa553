"""Repeat fuzz case 15 (rank-45 input, l=95) and print the Jacobi off-norm per sweep."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
from test_gpu_fuzz import _case
import paper_1803_01982_b200 as ffb

A, k, l, b, p, g, s = _case(np.random.default_rng(777 + int(sys.argv[1]) if len(sys.argv) > 1 else 792))
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    try:
        ap = ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=s)
        print("it", it, "sweeps", ap.meta.get("svd_sweeps"), flush=True)
    except Exception as e:
        print("it", it, "ERR", e, flush=True)
