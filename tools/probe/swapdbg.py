import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
import paper_1803_01982_b200 as ffb
from test_gpu_param_sweep import _matrix
A = _matrix(400, 300, "noisy", 7)
for g in (2.0, 1.3):
    try:
        r = ffb.srqr(A, ffb.SketchParams(k=25, l=35, b=32, p=5, g=g, d=3, seed=7))
        print(g, r.cert)
    except ffb.CertificationError as e:
        print(g, "cert error", e.result.cert)
for tg in (False, True):
    try:
        ap = ffb.flip_flop_srqr(A, 25, l=35, b=32, p=5, g=1.3, d=3, seed=7, trace_gaps=tg)
        print("ff trace", tg, ap.meta["srqr"].cert)
    except ffb.CertificationError as e:
        print("ff trace", tg, "cert error", e.result.cert)
    try:
        r = ffb.srqr(A, ffb.SketchParams(k=25, l=35, b=32, p=5, g=1.3, d=3, seed=7))
        print("srqr again", r.cert.swaps)
    except ffb.CertificationError as e:
        print("srqr again cert error")
