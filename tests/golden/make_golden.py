"""Generate golden fixtures by running the REFERENCE package (build container only).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Imports ``ffsrqr`` from ``/root/reference/pkg/src`` (read-only; absent on the
GPU box, which only reads the committed ``.npz`` files).  Each case stores its
input (or the recipe + sha256 of the input bytes), the parameters, and the
reference outputs:

* from a separate ``srqr(A, params)`` call: the true ``R`` (the reference's
  ``flip_flop_srqr`` overwrites ``meta['srqr'].fact.R`` via a view,
  ``ffsrqr/svd.py:67-68``), ``perm``, ``q_ext``, ``rtilde`` and the certificate;
* from ``flip_flop_srqr``: ``u, s, v`` and ``diag_L = diag(meta R[:l,:l])``
  (which, because of that aliasing, is the partial-LQ diagonal);
* from ``_trqrcp_state``: per-block pivot arrangements via ``_block_pivots``.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import ffsrqr  # noqa: E402
from ffsrqr import sketch as rsketch  # noqa: E402
from ffsrqr.errors import CertificationError  # noqa: E402
from ffsrqr.generators import gen_type1, kahan  # noqa: E402
from ffsrqr.sketch import SketchParams  # noqa: E402
from ffsrqr.srqr import srqr as ref_srqr  # noqa: E402
from ffsrqr.svd import flip_flop_srqr  # noqa: E402

from paper_1803_01982_b200 import workloads  # noqa: E402


def sha(A):
    return hashlib.sha256(np.ascontiguousarray(A, dtype=np.float64).tobytes()).hexdigest()


def block_orders(A, prm):
    """Replay the reference TRQRCP and record each block's pivot arrangement."""
    orig = rsketch._block_pivots
    rec = []

    def spy(B, j0, bb):
        out = orig(B, j0, bb)
        rec.append(np.array(out))
        return out

    rsketch._block_pivots = spy
    try:
        rsketch._trqrcp_state(A, prm)
    finally:
        rsketch._block_pivots = orig
    return rec


def run_case(name, A, k, l=None, b=32, p=5, g=2.0, seed=0, store_A=True, recipe=None,
             store_uv=True, flipflop=True):
    m, n = A.shape
    bb, pp = b, p
    if bb + pp > m:  # flip_flop clamp (svd.py:53-55) applied to srqr too for consistency
        bb = max(1, m - pp)
        pp = m - bb
    prm = SketchParams(k=k, l=l, b=bb, p=pp, g=g, seed=seed).resolve(m, n)
    out = dict(m=m, n=n, k=k, l=prm.l, b=prm.b, p=prm.p, g=g, d=prm.d, seed=seed,
               sha256=sha(A), recipe=json.dumps(recipe or {}))
    if store_A:
        out["A"] = A
    t = time.perf_counter()
    status = "ok"
    try:
        res = ref_srqr(A, prm)
    except CertificationError as exc:
        res = exc.result
        status = "CertificationError"
    out["srqr_status"] = status
    out["srqr_seconds"] = time.perf_counter() - t
    out["perm"] = res.fact.perm
    out["R"] = res.fact.R
    out["q_ext"] = res.q_ext if store_uv else res.q_ext[:, :0]
    out["rtilde"] = res.rtilde
    c = res.cert
    out["cert"] = np.array([c.alpha, c.g1, c.g2, c.swaps, c.tau_bound, c.tau_hat_bound,
                            res.r22_norm_estimate])
    orders = block_orders(A, prm)
    out["n_blocks"] = len(orders)
    for i, o in enumerate(orders):
        out[f"block_order_{i}"] = o
    if flipflop and status == "ok":
        t = time.perf_counter()
        ap = flip_flop_srqr(A, k, l=l, b=b, p=p, g=g, seed=seed)
        out["ff_seconds"] = time.perf_counter() - t
        out["s"] = ap.s
        out["diag_L"] = np.diag(ap.meta["srqr"].fact.R[:, : ap.meta["srqr"].fact.k]).copy()
        out["flop_count"] = ap.flop_count
        if store_uv:
            out["u"] = ap.u
            out["v"] = ap.v
        else:
            w = workloads.philox(12345, 777)
            xu = w.standard_normal(m)
            xv = w.standard_normal(n)
            out["u_proj_abs"] = np.abs(ap.u.T @ xu)
            out["v_proj_abs"] = np.abs(ap.v.T @ xv)
            out["u_colnorm"] = np.linalg.norm(ap.u, axis=0)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: m={m} n={n} k={k} l={prm.l} b={prm.b} p={prm.p} status={status} "
          f"swaps={int(c.swaps)} blocks={len(orders)} srqr={out['srqr_seconds']:.2f}s")


def main():
    g = np.random.default_rng
    run_case("rand90x70", g(100).standard_normal((90, 70)), 24, l=24, b=8, p=4)
    run_case("type1_120x90", gen_type1(120, 90, 40, seed=1), 12, l=17)
    run_case("type1_300", gen_type1(300, 300, 100, seed=3), 20, l=25)
    run_case("kahan96_l20", kahan(96, 1.2), 20, l=20, b=8, p=4)
    run_case("kahan96_l60", kahan(96, 1.2), 60, l=60, b=8, p=4)
    run_case("lowrank60x40", g(4).standard_normal((60, 10)) @ g(4).standard_normal((10, 40)),
             10, l=10, b=8, p=4, seed=1)
    run_case("certfail60x50", g(3).standard_normal((60, 50)), 8, l=8, b=8, p=4,
             g=1.0 + 1e-12, flipflop=False)
    run_case("identity8", np.eye(8), 3)
    run_case("tall600x300", g(7).standard_normal((600, 300)) @ np.diag(np.geomspace(1, 1e-4, 300)),
             40, l=45, b=16, p=6, seed=5)
    run_case("wide100x900", g(8).standard_normal((100, 900)), 20, l=25, b=8, p=4, seed=2)
    A1 = workloads.numpy_matrix("cfg1")
    run_case("cfg1", A1, 50, l=60, b=32, p=10, store_A=False, store_uv=False,
             recipe={"generator": "workloads.numpy_matrix", "cfg": "cfg1", "seed": 0})
    run_case("cfg1_g1p2", A1, 50, l=60, b=32, p=10, g=1.2, store_A=False, store_uv=False,
             recipe={"generator": "workloads.numpy_matrix", "cfg": "cfg1", "seed": 0})
    A5 = workloads.numpy_matrix("cfg5", seed=3, m=1024, n=512)
    run_case("cfg5_small", A5, 64, l=72, b=32, p=16, seed=3, store_A=False, store_uv=False,
             recipe={"generator": "workloads.numpy_matrix", "cfg": "cfg5", "seed": 3,
                     "m": 1024, "n": 512})
    with open(os.path.join(HERE, "VERSION.txt"), "w") as f:
        f.write(f"reference ffsrqr {ffsrqr.__version__} backend={ffsrqr.BACKEND} "
                f"numpy={np.__version__}\n")


if __name__ == "__main__":
    main()
