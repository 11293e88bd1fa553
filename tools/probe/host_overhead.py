"""Where does the host time of one Python-API call go (cfg3)?"""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads

w = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = workloads.CONFIGS[w]
A = workloads.torch_matrix(w, seed=0)
for _ in range(2):
    ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(5):
    ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
e1.record(); torch.cuda.synchronize()
print(f"wall {(time.perf_counter()-t0)/5*1e3:.2f} ms/call, device span {e0.elapsed_time(e1)/5:.2f} ms/call")
s1 = torch.cuda.Stream()
for label, ctx in (("side stream", torch.cuda.stream(s1)), ("default again", torch.cuda.stream(torch.cuda.default_stream()))):
    with ctx:
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
            torch.cuda.synchronize()
            print(f"{label} rep {rep}: wall {(time.perf_counter()-t0)/5*1e3:.2f} ms/call", flush=True)
