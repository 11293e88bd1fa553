"""cfg3 e2e pipeline diagnosis: allocator activity and per-call time vs stream count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads, batch

w = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = workloads.CONFIGS[w]
A = workloads.torch_matrix(w, seed=0)
m, n = A.shape
A_host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
A_host.copy_(A.t())
Ah = A_host.t()
del A
torch.cuda.synchronize()
# raw H2D bandwidth
d = torch.empty_like(A_host, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(A_host, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"H2D {A_host.numel()*8/1e9:.2f} GB in {e0.elapsed_time(e1):.2f} ms = {A_host.numel()*8/e0.elapsed_time(e1)/1e6:.1f} GB/s")
del d

def piped(i):
    r = ffb.flip_flop_srqr(Ah, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
    u = r.u.to("cpu", non_blocking=True)
    return i

for ns in (1, 2, 3, 4):
    batch.run_streams(list(range(ns)), piped, n_streams=ns)
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    batch.run_streams(list(range(12)), piped, n_streams=ns)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 12 * 1e3
    s1 = torch.cuda.memory_stats()
    print(f"streams={ns}: {dt:.2f} ms/fact, cudaMalloc calls {s1['num_device_alloc'] - s0['num_device_alloc']}, frees {s1['num_device_free'] - s0['num_device_free']}, retries {s1['num_alloc_retries'] - s0['num_alloc_retries']}", flush=True)
