"""e2e pipelining probe: calls over S streams on pinned host inputs (cfg2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import batch, workloads
A = workloads.torch_matrix("cfg2", seed=0)
m, n = A.shape
Ah = torch.empty((n, m), dtype=torch.float64, pin_memory=True); Ah.copy_(A.t()); Ahc = Ah.t()
del A
k, l, b, p = 256, 272, 64, 16
def run(S, N):
    outs = [(torch.empty((k, m), dtype=torch.float64, pin_memory=True).t(),
             torch.empty((k, n), dtype=torch.float64, pin_memory=True).t()) for _ in range(N)]
    def one(i):
        r = ffb.flip_flop_srqr(Ahc, k, l=l, b=b, p=p, seed=0)
        outs[i][0].copy_(r.u, non_blocking=True); outs[i][1].copy_(r.v, non_blocking=True)
        return i
    batch.run_streams(list(range(S)), one, n_streams=S)
    torch.cuda.synchronize(); t = time.perf_counter()
    batch.run_streams(list(range(N)), one, n_streams=S)
    torch.cuda.synchronize(); return (time.perf_counter() - t) / N * 1e3
for S, N in ((3, 12), (3, 12), (2, 12), (3, 24), (2, 8)):
    print(f"streams={S} calls={N}: {run(S, N):.2f} ms/step", flush=True)
