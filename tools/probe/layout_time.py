"""Device-resident flip-flop time for column-major vs row-major A (same values)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads

for w in sys.argv[1:] or ["cfg2"]:
    cfg = workloads.CONFIGS[w]
    A = workloads.torch_matrix(w, seed=0)
    Ac = A if A.stride(0) == 1 else A.t().contiguous().t()
    Ar = Ac.contiguous()
    for lab, X in (("col-major", Ac), ("row-major", Ar)):
        for _ in range(3):
            r = ffb.flip_flop_srqr(X, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            r = ffb.flip_flop_srqr(X, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
        e1.record()
        torch.cuda.synchronize()
        print(f"{w} {lab} strides={tuple(X.stride())}: {e0.elapsed_time(e1) / 10:.3f} ms  sigma_k={float(r.s[-1]):.6e}", flush=True)
