"""cfg5-shaped batch: Python stream pool (batch.run_streams) vs one
ffb_run_batched call (batch.NativeBatch, C++ threads), same problems."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1803_01982_b200 as ffb  # noqa: E402
from paper_1803_01982_b200 import batch, engine, workloads  # noqa: E402

cfg = workloads.CONFIGS["cfg5"]
probs = [workloads.torch_matrix("cfg5", seed=i) for i in range(64)]
engine.prefetch_omega([(cfg.b + cfg.p, cfg.m, i) for i in range(64)], threads=8)
for T in (8, 12, 16):
    nb = batch.NativeBatch(probs, cfg.k, cfg.l, cfg.b, cfg.p, seeds=list(range(64)), threads=T)
    nb.run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        out = nb.run()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    ref = ffb.flip_flop_srqr(probs[5], cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=5)
    same = torch.equal(out[5]["s"], ref.s)
    print(f"native threads={T}: {dt*1e3:.1f} ms per 64 -> {64/dt:.0f} fact/s; s bitwise == single call: {same}", flush=True)
def solve(i):
    return ffb.flip_flop_srqr(probs[i], cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=i)
batch.run_streams(list(range(64)), solve, n_streams=8)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    batch.run_streams(list(range(64)), solve, n_streams=8)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 3
print(f"python run_streams 8: {dt*1e3:.1f} ms per 64 -> {64/dt:.0f} fact/s", flush=True)
