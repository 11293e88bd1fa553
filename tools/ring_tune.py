"""Column-ring Jacobi geometry sweep (run under gpurun): time ffb_small_svd per l
for lane-group widths G and cluster sizes C, and the block kernel beside it.
usage: python tools/ring_tune.py [l ...]"""
import os
import subprocess
import sys

ls = [int(x) for x in sys.argv[1:]] or [50, 60, 100, 144]
here = os.path.dirname(os.path.abspath(__file__))
for l in ls:
    cases = [("block", {"FFB_JACOBI_BLOCK": "1"})]
    for g in ("4", "8", "16", "32"):
        for c in ("1", "2", "4", "8", "16"):
            cases.append((f"ring G={g} C={c}", {"FFB_RING_G": g, "FFB_RING_C": c, "FFB_RING_MAXL": "448"}))
    for name, env in cases:
        out = subprocess.run([sys.executable, os.path.join(here, "jacobi_bench.py"), str(l)],
                             env=dict(os.environ, FFB_JACOBI_PROF="1", **env), capture_output=True, text=True)
        ring = [x for x in out.stderr.splitlines() if x.startswith("jacobi ring")]
        res = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-200:]
        tag = ring[-1].split(":")[0].replace("jacobi ring ", "") if ring else "block kernel"
        if name.startswith("ring") and not ring:
            continue   # geometry did not fit: the block kernel ran
        print(f"{name:18s} | {tag:40s} | {res}", flush=True)
