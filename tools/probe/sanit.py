"""Small calls for compute-sanitizer (racecheck / memcheck / synccheck)."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import numpy as np
from test_gpu_fuzz import _case
import paper_1803_01982_b200 as ffb

rs = np.random.default_rng(1)
A = rs.standard_normal((300, 200))
ffb.flip_flop_srqr(A, 20, l=64, b=32, p=5)
A, k, l, b, p, g, s = _case(np.random.default_rng(777 + 15))
ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=s)
ffb.rsisvd(rs.standard_normal((300, 200)), 10)
print("sanit done")
