"""Calibrate the CPU baseline: the reference itself (ffsrqr, numba backend,
/root/reference/pkg/src) against the numpy oracle port (oracle/) on the same
host, the same matrices and the same thread count.

Runs only where /root/reference exists (the build container); writes
profiles/r04_cpu_calibration.json.  The GPU box's bench `cpu_baseline` /
`--impl reference` arm is the port; this file states its relation to the
reference.

usage: NUMBA_CACHE_DIR=/tmp/numba_cache python tools/calibrate_cpu.py [cfg1 cfg5 cfg2]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import oracle  # noqa: E402
from paper_1803_01982_b200 import workloads  # noqa: E402


def main(names):
    import ffsrqr
    from ffsrqr import backend
    from ffsrqr.svd import flip_flop_srqr

    try:
        from threadpoolctl import threadpool_info
        blas = [{k: d.get(k) for k in ("internal_api", "num_threads", "version")} for d in threadpool_info()]
    except Exception:  # pragma: no cover
        blas = None
    out = {"host_cores": len(os.sched_getaffinity(0)), "blas": blas,
           "reference_backend": getattr(backend, "BACKEND", None) or getattr(backend, "NAME", None),
           "reference_version": getattr(ffsrqr, "__version__", None), "configs": {}}
    path = os.path.join(ROOT, "profiles", "r04_cpu_calibration.json")
    for name in names:
        cfg = workloads.CONFIGS[name]
        t0 = time.perf_counter()
        A = np.asfortranarray(workloads.numpy_matrix(name, seed=0))
        gen = time.perf_counter() - t0
        # JIT warm-up of the numba kernels on a small problem first
        flip_flop_srqr(A[:200, :150].copy(), 10, l=12, b=cfg.b, p=cfg.p, seed=0)
        reps = 3 if name != "cfg2" else 1
        tr, tp = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = flip_flop_srqr(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
            tr.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            o = oracle.flip_flop(A, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
            tp.append(time.perf_counter() - t0)
        rel = float(np.max(np.abs(r.s - o.s) / r.s))
        out["configs"][name] = {"m": cfg.m, "n": cfg.n, "k": cfg.k, "l": cfg.l, "b": cfg.b, "p": cfg.p,
                                "reference_s": min(tr), "port_s": min(tp),
                                "port_over_reference": min(tp) / min(tr), "reps": reps,
                                "sigma_max_rel_diff": rel, "matrix_gen_s": gen}
        print(name, out["configs"][name], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg5", "cfg2"])
