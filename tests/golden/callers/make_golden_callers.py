"""Golden fixtures for the callers around the hot path, produced by running the
REFERENCE package (build container only):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/callers/make_golden_callers.py

* ``rsisvd_*``: ffsrqr.svd.rsisvd (svd.py:101-133) -> u, s, v;
* ``hosvd_*`` / ``sthosvd_*``: ffsrqr.tensor.hosvd / st_hosvd (tensor.py:104-145)
  with the built-in "flipflop" and "rsisvd" engines -> core, factors;
* ``ialm_*``: ffsrqr.nuclear.ialm_rpca / ialm_mc (nuclear.py:105-191) with the
  flip-flop and RSISVD partial SVDs -> low_rank, sparse, residual/rank history.

Inputs are small seeded numpy draws stored in the fixtures themselves.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from ffsrqr import nuclear, svd, tensor  # noqa: E402


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **kw)
    print(name, {k: getattr(v, "shape", v) for k, v in kw.items() if k != "A"})


def lowrank(rs, m, n, r, decay=0.7):
    U, _ = np.linalg.qr(rs.standard_normal((m, r)))
    V, _ = np.linalg.qr(rs.standard_normal((n, r)))
    return (U * decay ** np.arange(r)) @ V.T


def main():
    rs = np.random.default_rng(20240501)
    # ---- RSISVD
    for name, (m, n, k, p, q, seed) in {
        "rsisvd_tall": (300, 200, 20, 5, 2, 3),
        "rsisvd_wide": (120, 400, 10, 5, 1, 0),
        "rsisvd_q0": (256, 160, 16, 8, 0, 7),
    }.items():
        A = lowrank(rs, m, n, min(m, n) // 2, 0.93) + 1e-6 * rs.standard_normal((m, n))
        ap = svd.rsisvd(A, k, p=p, q=q, seed=seed)
        save(name, A=A, k=k, p=p, q=q, seed=seed, u=ap.u, s=ap.s, v=ap.v, flop_count=ap.flop_count)
    # ---- Tucker
    core = rs.standard_normal((5, 4, 3))
    Us = [np.linalg.qr(rs.standard_normal((s, r)))[0] for s, r in ((30, 5), (24, 4), (20, 3))]
    X = np.einsum("abc,ia,jb,kc->ijk", core, *Us) + 1e-6 * rs.standard_normal((30, 24, 20))
    X = np.asfortranarray(X)
    for eng in ("flipflop", "rsisvd"):
        d = tensor.hosvd(X, (5, 4, 3), engine=eng, seed=2)
        save(f"hosvd_{eng}", X=X, ranks=np.array([5, 4, 3]), seed=2, core=d.core,
             f0=d.factors[0], f1=d.factors[1], f2=d.factors[2])
        d = tensor.st_hosvd(X, (5, 4, 3), engine=eng, seed=2)
        save(f"sthosvd_{eng}", X=X, ranks=np.array([5, 4, 3]), seed=2, core=d.core,
             f0=d.factors[0], f1=d.factors[1], f2=d.factors[2], order=np.array(d.meta["order"]))
    # ---- IALM
    L = lowrank(rs, 80, 60, 4, 0.8) * 10.0
    S = np.where(rs.random((80, 60)) < 0.05, rs.standard_normal((80, 60)) * 5.0, 0.0)
    mask = rs.random((80, 60)) < 0.6
    for eng in ("flipflop", "rsisvd"):
        prm = nuclear.IalmParams(svd_engine=eng, max_iter=25, seed=1)
        st = nuclear.ialm_rpca(L + S, prm)
        save(f"ialm_rpca_{eng}", M=L + S, engine=eng, max_iter=25, seed=1, low_rank=st.low_rank,
             sparse=st.sparse, rank=st.rank, iterations=st.iterations,
             residuals=np.array(st.residuals), ranks=np.array(st.ranks), mus=np.array(st.mus))
        st = nuclear.ialm_mc(L, mask, prm)
        save(f"ialm_mc_{eng}", M=L, mask=mask, engine=eng, max_iter=25, seed=1,
             low_rank=st.low_rank, sparse=st.sparse, rank=st.rank, iterations=st.iterations,
             residuals=np.array(st.residuals), ranks=np.array(st.ranks), mus=np.array(st.mus))


if __name__ == "__main__":
    main()
