"""Run a fixed case list and save (R, s, u, v) so two builds / knob settings can
be compared bitwise: python ab_bitwise.py out.npz ; then compare a.npz b.npz."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import numpy as np

if sys.argv[1] == "compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("compared", len(a.files), "arrays;", len(bad), "differ", bad[:10])
    for k in bad[:5]:
        print(k, float(np.max(np.abs(a[k] - b[k]))))
    sys.exit(0)
from test_gpu_fuzz import _case
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads

out = {}
cases = [_case(np.random.default_rng(777 + s)) for s in range(16)]
cases += [_case(np.random.default_rng(5000 + s)) for s in range(24)]
cases.append((np.eye(300, 200), 20, 60, 32, 5, 2.0, 0))
cases.append((workloads.numpy_matrix("cfg1"), 50, 60, 32, 10, 2.0, 0))
for i, (A, k, l, b, p, g, s) in enumerate(cases):
    try:
        ap = ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=s)
    except ffb.CertificationError:
        continue
    out[f"R{i}"] = np.asarray(ap.meta["srqr"].fact.R)
    out[f"s{i}"] = np.asarray(ap.s)
    out[f"u{i}"] = np.asarray(ap.u)
    out[f"v{i}"] = np.asarray(ap.v)
np.savez(sys.argv[1], **out)
print("saved", len(out))
