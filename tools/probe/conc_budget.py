"""Throughput of 12 resident cfg2 factorizations on 3 streams (batch.run_streams)
per SM budget, several repeats each: is the rate stable?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import batch, workloads

w = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = workloads.CONFIGS[w]
A = workloads.torch_matrix(w, seed=0)

def cstep(i):
    return ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0).s

for ns, budgets in ((3, (49, 46, 44, 40, 36)), (2, (74, 70, 64)), (4, (37, 34, 30))):
    for b in budgets:
        rates = []
        for rep in range(4):
            batch.run_streams(list(range(ns)), cstep, n_streams=ns, budget=b)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            batch.run_streams(list(range(12)), cstep, n_streams=ns, budget=b)
            torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            rates.append(12e3 / e0.elapsed_time(e1))
        print(f"{w} streams={ns} budget={b}: " + " ".join(f"{r:.1f}" for r in rates), flush=True)
