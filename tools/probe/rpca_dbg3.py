import sys, os, shutil
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1803_01982_b200 import _capi
if len(sys.argv) > 1:
    _capi.LIB_PATH = os.path.join(ROOT, "tools/probe_bin/libffb200_old.so")
    _capi.load(_capi.LIB_PATH)
import paper_1803_01982_b200 as ffb
W = np.load(os.path.join(ROOT, "tools/probe/W_fail.npy"))
for l in (6, 8, 12, 20, 39):
    try:
        f = ffb.trqrcp(W, ffb.SketchParams(k=4, l=l, b=32, p=5)); print(l, "trqrcp ok")
    except Exception as e:
        print(l, "trqrcp", type(e).__name__, e)
