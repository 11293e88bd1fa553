"""Per-kernel device time of ONE factorization run under an SM budget (the
conditions of a batch worker thread): python tools/probe/budget_split.py cfg5 18"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1803_01982_b200 as ffb  # noqa: E402
from paper_1803_01982_b200 import _capi, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 18
cfg = workloads.CONFIGS[name]
A = workloads.torch_matrix(name, seed=0)
lib = _capi.load()
for b in (0, budget):
    lib.ffb_set_thread_sm_budget(b)

    def step():
        return ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    times, counts = bench.profile_kernels(step)
    fam = {}
    for k, v in times.items():
        f = bench.kernel_family(k)
        fam[f] = fam.get(f, 0.0) + v
    print(f"{name} budget={b}: {e0.elapsed_time(e1) / 5:.3f} ms/factorization, kernel sum {sum(times.values()):.3f} ms")
    for f, v in sorted(fam.items(), key=lambda kv: -kv[1])[:int(os.environ.get("TOPN", "8"))]:
        print(f"   {v:7.3f} ms  {f}")
