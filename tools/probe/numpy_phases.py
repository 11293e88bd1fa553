"""Phase split of the numpy-in / numpy-out call (cfg2): cProfile top entries."""
import cProfile, pstats, os, sys, time, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads, engine

w = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = workloads.CONFIGS[w]
An = np.asfortranarray(workloads.torch_matrix(w, seed=0).cpu().numpy())
for _ in range(2):
    ffb.flip_flop_srqr(An, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
engine._omega_cache_clear() if hasattr(engine, "_omega_cache_clear") else None
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(3):
    r = ffb.flip_flop_srqr(An, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
pr.disable()
print(f"{(time.perf_counter() - t0) / 3 * 1e3:.1f} ms/call")
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(28)
print("\n".join(l[:150] for l in s.getvalue().splitlines()[4:50]))
