"""Host -> HBM rate of engine._upload_bytes on a pageable numpy array (cfg2's A,
537 MB): python tools/probe/upload_rate.py  (env FFB_STAGE_WORKERS / FFB_STAGE_CHUNK_MB)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1803_01982_b200 import engine

n = 8192
a = np.random.default_rng(0).standard_normal((n, n))
dev = torch.device("cuda", 0)
for _ in range(2):
    t = engine._upload_bytes(torch, a, dev)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    t = engine._upload_bytes(torch, a, dev)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
best = min(ts)
print(f"workers={engine._copy_pool()._max_workers} chunk={engine._STAGE_CHUNK >> 20}MB: {best * 1e3:.1f} ms, {a.nbytes / best / 1e9:.1f} GB/s (cores {os.cpu_count()})")
# pure pinned DMA for reference
p = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
p.numpy()[:] = a.reshape(-1)
d = torch.empty(a.size, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(p, non_blocking=True); torch.cuda.synchronize()
print(f"pinned DMA: {(time.perf_counter() - t0) * 1e3:.1f} ms")
t0 = time.perf_counter(); p.numpy()[:] = a.reshape(-1); print(f"one-thread host copy: {(time.perf_counter() - t0) * 1e3:.1f} ms")
