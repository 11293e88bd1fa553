"""Replay the test_gpu_fuzz case sequence R times in one process (intermittency hunt)."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import numpy as np
from test_gpu_fuzz import _case
import paper_1803_01982_b200 as ffb

R = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cases = [_case(np.random.default_rng(777 + s)) for s in range(16)]
ref15 = None
for rep in range(R):
    for i, (A, k, l, b, p, g, s) in enumerate(cases):
        if i == 15:
            print("CASE15", flush=True); sys.stderr.flush()
        try:
            ap = ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=s)
        except ffb.CertificationError:
            continue
        except Exception as e:
            print("rep", rep, "case", i, "ERR", e, flush=True)
            continue
        if i == 15:
            sg = np.asarray(ap.s)
            if ref15 is None:
                ref15 = sg
            print("rep", rep, "sweeps", ap.meta.get("svd_sweeps"), "ds", float(np.max(np.abs(sg - ref15))), flush=True)
