"""Wall time of the numpy-in / numpy-out call (the reference-facing signature) vs pinned torch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads

w = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = workloads.CONFIGS[w]
A = workloads.torch_matrix(w, seed=0)
An = np.asfortranarray(A.cpu().numpy())
Ac = np.ascontiguousarray(An)
for lab, X in (("numpy F-order", An), ("numpy C-order", Ac)):
    ffb.flip_flop_srqr(X, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
    t0 = time.perf_counter()
    for _ in range(3):
        r = ffb.flip_flop_srqr(X, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
        _ = (np.asarray(r.u).sum(), np.asarray(r.v).sum(), np.asarray(r.s).sum())
    print(f"{lab}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms/call", flush=True)
t0 = time.perf_counter()
d = torch.from_numpy(An.T).to("cuda"); torch.cuda.synchronize()
print(f"pageable H2D alone: {(time.perf_counter() - t0) * 1e3:.1f} ms")
