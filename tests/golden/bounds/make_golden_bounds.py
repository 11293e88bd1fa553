"""Golden vectors for check_theorem_bounds (ffsrqr/svd.py:174-255), made by
running the REFERENCE in the build container (it is absent on the GPU box).

The reference's flip_flop_srqr clobbers meta["srqr"].fact.R (svd.py:67-68),
so the report is formed on an ApproxSvd whose meta["srqr"] is the result of
a separate reference srqr() call with identical parameters: the same
factorization, with its true R.  Cases follow the reference's own tests
(tests/test_svd.py:80-101, tests/test_acceptance.py:101-110).

Run: python tests/golden/bounds/make_golden_bounds.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from ffsrqr.generators import gen_type1  # noqa: E402
from ffsrqr.sketch import SketchParams  # noqa: E402
from ffsrqr.srqr import srqr as ref_srqr  # noqa: E402
from ffsrqr.svd import ApproxSvd, check_theorem_bounds, flip_flop_srqr  # noqa: E402


def case(name, A, k, l, seed):
    ap = flip_flop_srqr(A, k, l=l, seed=seed)
    prm = ap.meta["params"]
    res = ref_srqr(A, SketchParams(k=prm.k, l=prm.l, b=prm.b, p=prm.p, epsilon=prm.epsilon,
                                   g=prm.g, d=prm.d, seed=prm.seed).resolve(*A.shape))
    ap2 = ApproxSvd(u=ap.u, s=ap.s, v=ap.v, meta={"srqr": res})
    rep = check_theorem_bounds(A, ap2)
    d = rep.detail
    np.savez(os.path.join(HERE, name + ".npz"), A=A, k=k, l=l, seed=seed,
             tau=rep.tau, tau_hat=rep.tau_hat, degenerate=rep.degenerate, all_ok=rep.all_ok,
             flags=np.array([rep.aux_lower_ok, rep.sv_lower_ok, rep.sv_upper_ok,
                             rep.aux_residual_ok, rep.residual_ok]),
             r22_2=d.get("r22_2", 0.0), r22_12=d.get("r22_12", 0.0), resid2=d.get("resid2", 0.0),
             g1=d.get("g1", 0.0), g2=d.get("g2", 0.0), sigma_exact=rep.sigma_exact)
    print(name, rep.all_ok, rep.degenerate, rep.tau, rep.tau_hat)


if __name__ == "__main__":
    case("bounds_type1_120_s0", gen_type1(120, 120, 50, seed=0), 10, 15, 0)
    case("bounds_type1_100_s7", gen_type1(100, 100, 40, seed=7), 10, 15, 1)
    case("bounds_type1_300_s3", gen_type1(300, 300, 100, seed=3), 20, 25, 3)
    g = np.random.default_rng(8)
    case("bounds_degenerate", g.standard_normal((40, 6)) @ g.standard_normal((6, 30)), 4, 6, 0)
