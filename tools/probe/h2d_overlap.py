"""Does an 800 MB pinned H2D copy overlap a running factorization on another stream?"""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads

w = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = workloads.CONFIGS[w]
A = workloads.torch_matrix(w, seed=0)
m, n = A.shape
H = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
H.copy_(A.t())
D = torch.empty_like(H, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
torch.cuda.synchronize()

def compute(N, out):
    with torch.cuda.stream(s1):
        t0 = time.perf_counter()
        for _ in range(N):
            ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) / N * 1e3)

def copies(N, out):
    with torch.cuda.stream(s2):
        t0 = time.perf_counter()
        for _ in range(N):
            D.copy_(H, non_blocking=True)
            s2.synchronize()
        out.append((time.perf_counter() - t0) / N * 1e3)

a, b = [], []
compute(4, a); copies(4, b)
print(f"alone: compute {a[0]:.2f} ms/fact, H2D {b[0]:.2f} ms/copy")
a, b = [], []
t1 = threading.Thread(target=compute, args=(6, a)); t2 = threading.Thread(target=copies, args=(8, b))
t1.start(); t2.start(); t1.join(); t2.join()
print(f"together: compute {a[0]:.2f} ms/fact, H2D {b[0]:.2f} ms/copy")
