"""CPU oracle for the callers around the hot path — TEST INFRASTRUCTURE ONLY.

numpy restatements of the reference's RSISVD baseline, Tucker (HOSVD /
ST-HOSVD) and nuclear-norm (IALM RPCA / matrix completion) drivers, each
citing the reference file:line it follows (``/root/reference/pkg/src/ffsrqr``).
They use this package's flip-flop oracle (``ffsrqr_oracle.flip_flop``) as the
low-rank engine, exactly like the reference binds ``svd.flip_flop_srqr``.

Pinning: ``tests/golden/callers/make_golden_callers.py`` runs the reference
itself on small seeded inputs; ``tests/test_oracle_callers.py`` checks these
restatements against those fixtures.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .ffsrqr_oracle import OracleError, flip_flop, gaussian

STREAM_RSISVD = 2_000_000   # ffsrqr/rng.py:13


@dataclass
class OracleSvd:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    meta: dict = field(default_factory=dict)


def rsisvd(A, k, p=5, q=2, seed=0):
    """ffsrqr/svd.py:101-133: randomized subspace iteration, q power steps."""
    A = np.asarray(A, dtype=float)
    m, n = A.shape
    if not 1 <= k <= min(m, n):
        raise OracleError("DimensionError", f"rsisvd needs 1 <= k <= min(m,n); got k={k}")
    if p < 0 or q < 0:
        raise OracleError("DimensionError", "rsisvd needs p >= 0 and q >= 0")
    r = min(k + p, min(m, n))
    omega = gaussian(n, r, seed, STREAM_RSISVD)
    Q, _ = np.linalg.qr(A @ omega)
    for _ in range(q):
        Q, _ = np.linalg.qr(A.T @ Q)
        Q, _ = np.linalg.qr(A @ Q)
    B = Q.T @ A
    Ub, s, Vt = np.linalg.svd(B, full_matrices=False)
    return OracleSvd(u=Q @ Ub[:, :k], s=s[:k].copy(), v=Vt[:k].T.copy(),
                     meta={"method": "rsisvd", "q": q, "p": p, "sv_all": s.copy()})


# ---------------------------------------------------------------- Tucker

def unfold(X, mode):
    """ffsrqr/tensor.py:21-27 (columns: remaining modes, Fortran order)."""
    return np.reshape(np.moveaxis(np.asarray(X), mode, 0), (X.shape[mode], -1), order="F")


def fold(M, mode, shape):
    """ffsrqr/tensor.py:30-38."""
    shape = tuple(shape)
    lead = (shape[mode],) + shape[:mode] + shape[mode + 1:]
    return np.moveaxis(np.reshape(M, lead, order="F"), 0, mode)


def nmode_product(X, U, mode):
    """ffsrqr/tensor.py:41-52: contract X's mode index with U's second index."""
    shape = list(X.shape)
    shape[mode] = U.shape[0]
    return fold(U @ unfold(X, mode), mode, shape)


def make_engine(engine, seed=0):
    """ffsrqr/tensor.py:73-91 (``exact``, ``flipflop``, ``rsisvd`` or a callable)."""
    if callable(engine):
        return engine
    if engine == "exact":
        def _exact(M, r):
            U, s, Vt = np.linalg.svd(M, full_matrices=False)
            return OracleSvd(u=U[:, :r], s=s[:r], v=Vt[:r].T)
        return _exact
    if engine == "flipflop":
        def _ff(M, r):
            m = M.shape[0]
            l = min(r + 5, min(M.shape) - 1)
            b = min(32, max(m - 5, 1))
            p = min(5, max(m - b, 0))
            return flip_flop(M, r, l=max(l, r), b=b, p=p, seed=seed)
        return _ff
    if engine == "rsisvd":
        return lambda M, r: rsisvd(M, r, seed=seed)
    raise ValueError(f"unknown low-rank engine {engine!r}")


@dataclass
class OracleTucker:
    core: np.ndarray
    factors: list
    order: list = None


def hosvd(X, ranks, engine="flipflop", seed=0):
    """ffsrqr/tensor.py:104-120: factors from the original tensor's unfoldings,
    core formed at the end."""
    X = np.asarray(X, dtype=float)
    solve = make_engine(engine, seed)
    factors = [solve(unfold(X, n), r).u for n, r in enumerate(ranks)]
    G = X
    for n, U in enumerate(factors):
        G = nmode_product(G, U.T, n)
    return OracleTucker(core=G, factors=factors)


def st_hosvd(X, ranks, engine="flipflop", seed=0, order=None):
    """ffsrqr/tensor.py:123-145: modes truncated one at a time (default order:
    increasing mode size)."""
    X = np.asarray(X, dtype=float)
    solve = make_engine(engine, seed)
    order = sorted(range(X.ndim), key=lambda n: X.shape[n]) if order is None else list(order)
    factors = [None] * X.ndim
    G = X
    for n in order:
        U = solve(unfold(G, n), ranks[n]).u
        factors[n] = U
        G = nmode_product(G, U.T, n)
    return OracleTucker(core=G, factors=factors, order=order)


# --------------------------------------------------------- nuclear norm

def soft_shrink(X, tau):
    """ffsrqr/nuclear.py:21-23."""
    return np.sign(X) * np.maximum(np.abs(X) - tau, 0.0)


def _partial_svd(engine, seed, min_dim):
    """ffsrqr/nuclear.py:52-78 (_PartialSvd)."""
    cap = min_dim if engine == "exact" else max(min_dim - 1, 1)

    def call(M, sv):
        sv = min(sv, cap)
        if engine == "exact" or sv >= min_dim:
            U, s, Vt = np.linalg.svd(M, full_matrices=False)
            return U[:, :sv], s[:sv], Vt[:sv].T
        if engine == "flipflop":
            l = min(sv + 60, min_dim - 1)
            ap = flip_flop(M, sv, l=l, seed=seed)
        elif engine == "rsisvd":
            ap = rsisvd(M, sv, seed=seed)
        else:
            raise ValueError(f"unknown svd engine {engine!r}")
        return ap.u, ap.s, ap.v

    return call


def _grow_sv(rank, sv, min_dim):
    """ffsrqr/nuclear.py:81-88."""
    if rank < sv:
        return min(rank + 1, min_dim)
    nxt = sv + 5 if sv <= 50 else int(round(1.1 * sv))
    return min(nxt, min_dim)


def _shrink_spectrum(psvd, M, sv, mu):
    """ffsrqr/nuclear.py:91-97."""
    U, s, V = psvd(M, sv)
    keep = int(np.count_nonzero(s > 1.0 / mu))
    if keep == 0:
        return np.zeros_like(M), 0
    return (U[:, :keep] * (s[:keep] - 1.0 / mu)) @ V[:, :keep].T, keep


@dataclass
class OracleIalm:
    low_rank: np.ndarray
    sparse: np.ndarray
    rank: int
    iterations: int
    converged: bool
    residuals: list
    ranks: list
    mus: list


def _params(p):
    d = dict(lam=None, mu0=None, mu_bar=None, rho=1.5, tol=1e-7, max_iter=100, sv0=10,
             svd_engine="exact", seed=0)
    d.update(p or {})
    return d


def ialm_rpca(M, params=None):
    """ffsrqr/nuclear.py:105-145: robust PCA, M = low rank + sparse."""
    M = np.asarray(M, dtype=float)
    p = _params(params)
    m, n = M.shape
    lam = p["lam"] if p["lam"] is not None else 1.0 / math.sqrt(max(m, n))
    normF = np.linalg.norm(M)
    norm2 = np.linalg.svd(M, compute_uv=False)[0]
    mu = p["mu0"] if p["mu0"] is not None else 1.25 / norm2
    mu_bar = p["mu_bar"] if p["mu_bar"] is not None else mu * 1e7
    Y = M / max(norm2, float(np.max(np.abs(M))))
    E = np.zeros_like(M)
    psvd = _partial_svd(p["svd_engine"], p["seed"], min(m, n))
    sv = min(p["sv0"], min(m, n))
    X = np.zeros_like(M)
    out = OracleIalm(X, E, 0, 0, False, [], [], [])
    for it in range(1, p["max_iter"] + 1):
        X, rank = _shrink_spectrum(psvd, M - E + Y / mu, sv, mu)
        sv = _grow_sv(rank, sv, min(m, n))
        E = soft_shrink(M - X + Y / mu, lam / mu)
        Z = M - X - E
        Y = Y + mu * Z
        out.mus.append(mu)
        mu = min(p["rho"] * mu, mu_bar)
        res = float(np.linalg.norm(Z) / normF)
        out.residuals.append(res)
        out.ranks.append(rank)
        out.low_rank, out.sparse, out.rank, out.iterations = X, E, rank, it
        if res < p["tol"]:
            out.converged = True
            break
    return out


def ialm_mc(M, mask, params=None):
    """ffsrqr/nuclear.py:148-191: matrix completion from the observed entries."""
    M = np.asarray(M, dtype=float)
    mask = np.asarray(mask, dtype=bool)
    M = np.where(mask, M, 0.0)
    p = _params(params)
    m, n = M.shape
    norm2 = np.linalg.svd(M, compute_uv=False)[0]
    mu = p["mu0"] if p["mu0"] is not None else 1.25 / norm2
    mu_bar = p["mu_bar"] if p["mu_bar"] is not None else mu * 1e7
    normF = np.linalg.norm(M)
    Y = np.zeros_like(M)
    E = np.zeros_like(M)
    psvd = _partial_svd(p["svd_engine"], p["seed"], min(m, n))
    sv = min(p["sv0"], min(m, n))
    X = np.zeros_like(M)
    out = OracleIalm(X, E, 0, 0, False, [], [], [])
    for it in range(1, p["max_iter"] + 1):
        X, rank = _shrink_spectrum(psvd, M - E + Y / mu, sv, mu)
        sv = _grow_sv(rank, sv, min(m, n))
        E = np.where(mask, 0.0, M - X + Y / mu)
        Z = M - X - E
        Y = Y + mu * Z
        out.mus.append(mu)
        mu = min(p["rho"] * mu, mu_bar)
        res = float(np.linalg.norm(Z) / normF)
        out.residuals.append(res)
        out.ranks.append(rank)
        out.low_rank, out.sparse, out.rank, out.iterations = X, E, rank, it
        if res < p["tol"]:
            out.converged = True
            break
    return out
