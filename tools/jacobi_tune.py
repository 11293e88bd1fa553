"""Time the flip-flop on cfg2 for Jacobi knob settings (env vars read per launch)."""
import os, subprocess, sys, json
res = {}
for bs in ("8", "16"):
    for inner in ("1", "2", "3"):
        env = dict(os.environ, FFB_JACOBI_BS=bs, FFB_JACOBI_INNER=inner)
        out = subprocess.run([sys.executable, "-c", """
import torch, time
import paper_1803_01982_b200 as ffb
from paper_1803_01982_b200 import workloads
A = workloads.torch_matrix('cfg2', seed=0)
for _ in range(2): r = ffb.flip_flop_srqr(A, 256, l=272, b=64, p=16, seed=0)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(3): r = ffb.flip_flop_srqr(A, 256, l=272, b=64, p=16, seed=0)
torch.cuda.synchronize(); print((time.perf_counter()-t)/3*1e3, r.meta['svd_sweeps'], float(r.s[-1]))
"""], env=env, capture_output=True, text=True)
        res[f"bs{bs}_inner{inner}"] = out.stdout.strip() or out.stderr[-300:]
print(json.dumps(res, indent=1))
