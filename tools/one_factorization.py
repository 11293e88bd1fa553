"""Run W warm-up + 1 profiled flip_flop_srqr on a BASELINE workload (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_01982_b200 as ffb  # noqa: E402
from paper_1803_01982_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.workload]
A = workloads.torch_matrix(a.workload, seed=0) if a.workload != "cfg4" else \
    workloads.torch_tensor_unfoldings(seed=0)[0]
for _ in range(a.warmup):
    r = ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
torch.cuda.synchronize()
# ncu --profile-from-start off: only the measured factorizations are captured
torch.cuda.profiler.start()
torch.cuda.nvtx.range_push("factor")
for _ in range(a.reps):
    r = ffb.flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.profiler.stop()
print("kernels per factorization:", r.meta["kernels"], "swaps:", r.meta["srqr"].cert.swaps, "svd_sweeps:", r.meta.get("svd_sweeps"))
