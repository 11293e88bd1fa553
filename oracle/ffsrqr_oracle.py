"""Numpy restatement of the reference Flip-Flop SRQR path — TEST INFRASTRUCTURE.

This module is the *checker* for the B200 engine: it restates, step for step,
the CPU algorithm of the reference package ``ffsrqr`` (read-only at
``/root/reference/pkg/src/ffsrqr``, abbreviated ``ffsrqr/`` below).  It is
imported only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
legs.  Nothing under ``paper_1803_01982_b200/`` imports it.

Pinned against the reference itself: ``tests/golden/make_golden.py`` runs the
reference in the build container and stores inputs/outputs as ``.npz``
fixtures; ``tests/test_oracle_golden.py`` checks this module against them
(pivots exactly, factors to ~1e-12).

Differences from the reference that are deliberate and documented:

* ``flip_flop`` returns the *true* SRQR ``R`` (the reference overwrites
  ``meta["srqr"].fact.R`` with the QRNP workspace of ``R^T`` through a NumPy
  view, ``ffsrqr/svd.py:67-68``) and exposes ``diag_L`` explicitly.
* No thread-local flop counter; ``flip_flop_flops`` gives the paper formula.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

GUARD = 1e-8  # ffsrqr/_kernels_numpy.py:20, ffsrqr/qr.py:18
STREAM_SKETCH = 0  # ffsrqr/rng.py:11
STREAM_G2 = 1000  # ffsrqr/rng.py:12


class OracleError(Exception):
    """Raised with a ``kind`` matching the reference exception class name."""

    def __init__(self, kind, msg, payload=None):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.payload = payload


# --------------------------------------------------------------------------
# RNG and parameters
# --------------------------------------------------------------------------

def gaussian(rows, cols, seed, stream):
    """N(0,1) matrix from Philox keyed by (seed, stream) — ffsrqr/rng.py:17-23."""
    key = np.array([np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), np.uint64(stream)])
    return np.random.Generator(np.random.Philox(key=key)).standard_normal((rows, cols))


def resolve(m, n, k, l=None, b=32, p=5, epsilon=0.5, g=2.0, d=None, seed=0, clamp=True):
    """Parameter defaulting/validation.

    Clamp of b, p for small m: ffsrqr/svd.py:53-55 (flip_flop only).
    Validation: ffsrqr/sketch.py:41-59.  Returns a dict.
    """
    if clamp and b + p > m:
        b = max(1, m - p)
        p = m - b
    l = k if l is None else l
    d = min(l, 10) if d is None else d
    if not 1 <= k <= l <= min(m, n):
        raise OracleError("DimensionError", f"need 1 <= k <= l <= min(m,n); got k={k}, l={l}")
    if b < 1 or p < 0:
        raise OracleError("DimensionError", "need b >= 1 and p >= 0")
    if not 0.0 < epsilon < 1.0:
        raise OracleError("DimensionError", "epsilon must lie in (0,1)")
    if g <= 1.0:
        raise OracleError("DimensionError", "g must exceed 1")
    if not 1 <= d <= l:
        raise OracleError("DimensionError", "need 1 <= d <= l")
    if b + p > m:
        raise OracleError("DimensionError", f"sketch rows b+p={b + p} exceed m={m}")
    return dict(k=k, l=l, b=b, p=p, epsilon=epsilon, g=g, d=d, seed=seed)


# --------------------------------------------------------------------------
# Dense kernels
# --------------------------------------------------------------------------

def householder(x):
    """(v, beta, alpha) with v[0]=1 — ffsrqr/qr.py:21-43.

    tail == 0 gives the identity reflector (beta=0, alpha=x0); otherwise
    alpha = -sign(x0)*||x|| (alpha=+||x|| when x0 == 0).
    """
    x = np.asarray(x, dtype=float)
    x0 = float(x[0])
    tsq = float(x[1:] @ x[1:])
    v = np.zeros_like(x)
    v[0] = 1.0
    if tsq == 0.0:
        return v, 0.0, x0
    nrm = math.sqrt(x0 * x0 + tsq)
    alpha = nrm if x0 == 0.0 else -math.copysign(nrm, x0)
    v[1:] = x[1:] / (x0 - alpha)
    return v, (alpha - x0) / alpha, alpha


def qrcp_pivots(W, k):
    """k pivoted Householder steps on W (modified in place); returns the
    swap-history column arrangement.

    Semantics of ffsrqr/_kernels_numpy.py:23-81 (numba twin
    ffsrqr/_kernels_numba.py:15-94): first-max argmax (ties → lowest index),
    column swap, reflector with the identity branch, rank-1 update, squared
    norm downdate and the guard recompute r < 1e-8*r0 or r < 0.
    """
    m, n = W.shape
    order = np.arange(n, dtype=np.int64)
    r = np.einsum("ij,ij->j", W, W)
    r0 = r.copy()
    for j in range(k):
        q = j + int(np.argmax(r[j:]))
        if q != j:
            for arr in (order, r, r0):
                arr[[j, q]] = arr[[q, j]]
            W[:, [j, q]] = W[:, [q, j]]
        x0 = W[j, j]
        tail = W[j + 1:, j]
        tsq = float(tail @ tail)
        if tsq != 0.0:
            nrm = math.sqrt(x0 * x0 + tsq)
            alpha = nrm if x0 == 0.0 else -math.copysign(nrm, x0)
            W[j + 1:, j] = tail / (x0 - alpha)
            tau = (alpha - x0) / alpha
            if j + 1 < n:
                v = np.concatenate(([1.0], W[j + 1:, j]))
                w = v @ W[j:, j + 1:]
                W[j:, j + 1:] -= tau * np.outer(v, w)
            W[j, j] = alpha
        if j + 1 < n:
            rr = r[j + 1:]
            rr -= W[j, j + 1:] ** 2
            bad = np.flatnonzero((rr < GUARD * r0[j + 1:]) | (rr < 0.0))
            for b_ in bad:
                c = j + 1 + int(b_)
                col = W[j + 1:, c]
                r[c] = max(float(col @ col), 0.0)
    return order


def qrnp_inplace(W, k):
    """k unpivoted Householder steps, LAPACK storage — ffsrqr/_kernels_numpy.py:84-109.

    Returns taus; W holds R (upper) and reflector tails (strictly lower).
    """
    m, n = W.shape
    if k == n and k <= m and W.flags.f_contiguous:
        # all columns: LAPACK dgeqrf is the same factorization in the same
        # storage (dlarfg: beta = -sign(x0) ||x||, tau = (beta - x0)/beta, tail
        # scaled by 1/(x0 - beta), tau = 0 for a zero tail), blocked (BLAS-3)
        from scipy.linalg import lapack

        qr, taus, _, info = lapack.dgeqrf(W, overwrite_a=True)
        if info == 0:
            if qr is not W:
                W[...] = qr
            return np.asarray(taus[:k], dtype=float).copy()
    taus = np.zeros(k)
    for j in range(k):
        x0 = W[j, j]
        tail = W[j + 1:, j]
        tsq = float(tail @ tail)
        if tsq == 0.0:
            continue
        nrm = math.sqrt(x0 * x0 + tsq)
        alpha = nrm if x0 == 0.0 else -math.copysign(nrm, x0)
        W[j + 1:, j] = tail / (x0 - alpha)
        taus[j] = (alpha - x0) / alpha
        if j + 1 < n:
            v = np.concatenate(([1.0], W[j + 1:, j]))
            w = v @ W[j:, j + 1:]
            W[j:, j + 1:] -= taus[j] * np.outer(v, w)
        W[j, j] = alpha
    return taus


def wy_from_lapack(W, taus, k):
    """Compact WY (Y, T) from LAPACK storage — ffsrqr/qr.py:104-115."""
    m = W.shape[0]
    Y = np.tril(W[:, :k], -1)
    Y[np.arange(k), np.arange(k)] = 1.0
    T = np.zeros((k, k))
    for j in range(k):
        T[:j, j] = -taus[j] * (T[:j, :j] @ (Y[:, :j].T @ Y[:, j]))
        T[j, j] = taus[j]
    return Y, T


def tri_solve(R11, R12):
    """R11^{-1} R12 with the exact-zero-diagonal lstsq fallback — ffsrqr/sketch.py:75-83."""
    if np.min(np.abs(np.diag(R11))) == 0.0:
        if np.linalg.norm(R12) == 0.0:
            return np.zeros_like(R12)
        return np.linalg.lstsq(R11, R12, rcond=None)[0]
    return scipy.linalg.solve_triangular(R11, R12)


# --------------------------------------------------------------------------
# TRQRCP (Alg. 2)
# --------------------------------------------------------------------------

@dataclass
class OracleTrqrcp:
    Aw: np.ndarray
    Y: np.ndarray
    T: np.ndarray
    WT: np.ndarray
    R: np.ndarray
    B: np.ndarray
    omega: np.ndarray
    perm: np.ndarray
    prm: dict
    block_orders: list = field(default_factory=list)


def trqrcp(A, prm):
    """Truncated randomized QRCP to l steps — ffsrqr/sketch.py:101-147.

    Sketch B = Omega @ A with Omega = gaussian(b+p, m, seed, 0) (sketch.py:108-109),
    block pivots from QRCP on a copy of B[:, j0:] (sketch.py:62-67), physical
    reorder of Aw/B/WT/R (sketch.py:70-72,120-121), per-column left-looking
    Householder with W^T = T^T Y^T Aw rows (sketch.py:123-139), then the sketch
    update B[:, e:] -= B[:, j0:e] R11^{-1} R12 (sketch.py:141-144).
    """
    A = np.asarray(A, dtype=float)
    m, n = A.shape
    l, b, p = prm["l"], prm["b"], prm["p"]
    Aw = np.array(A, order="F")
    omega = gaussian(b + p, m, prm["seed"], STREAM_SKETCH)
    B = np.array(omega @ Aw, order="F")
    perm = np.arange(n, dtype=np.int64)
    Y = np.zeros((m, l))
    T = np.zeros((l, l))
    WT = np.zeros((l, n))
    R = np.zeros((l, n))
    orders = []
    j0 = 0
    while j0 < l:
        bb = min(b, l - j0)
        sub = np.asfortranarray(B[:, j0:].copy())
        order = j0 + qrcp_pivots(sub, bb)
        orders.append(order.copy())
        for M in (Aw, B, WT, R):
            M[:, j0:] = M[:, order]
        perm[j0:] = perm[order]
        for c in range(j0, j0 + bb):
            col = Aw[:, c] - Y[:, :c] @ WT[:c, c]
            v, beta, alpha = householder(col[c:])
            Y[c:, c] = v
            yv = Y[c:, :c].T @ v
            T[:c, c] = -beta * (T[:c, :c] @ yv)
            T[c, c] = beta
            WT[c, :] = beta * (v @ Aw[c:, :] - yv @ WT[:c, :])
            R[c, c:] = Aw[c, c:] - Y[c, :c + 1] @ WT[:c + 1, c:]
            R[c, c] = alpha
        e = j0 + bb
        if e < n:
            X = tri_solve(R[j0:e, j0:e], R[j0:e, e:])
            B[:, e:] -= B[:, j0:e] @ X
        j0 = e
    return OracleTrqrcp(Aw=Aw, Y=Y, T=T, WT=WT, R=R, B=B, omega=omega, perm=perm,
                        prm=prm, block_orders=orders)


# --------------------------------------------------------------------------
# SRQR (Alg. 3)
# --------------------------------------------------------------------------

@dataclass
class OracleSrqr:
    R: np.ndarray          # l x n, arrangement order (true R, upper trapezoidal)
    perm: np.ndarray
    Q: np.ndarray          # m x (l+1)
    rtilde: np.ndarray     # (l+1) x (l+1)
    alpha: float
    g1: float
    g2: float
    swaps: int
    tau_bound: float
    tau_hat_bound: float
    r22: float
    i_offs: list
    trq: OracleTrqrcp = None


def g2_estimate(Rt, alpha, d, seed, stream):
    """ffsrqr/srqr.py:49-64: Z = Rt^{-1} Omega^T, g2 = |alpha|/sqrt(d) * max row norm."""
    if np.min(np.abs(np.diag(Rt))) == 0.0:
        raise OracleError("SingularTrailingBlockError", "zero diagonal in leading triangular block")
    om = gaussian(d, Rt.shape[0], seed, stream)
    Z = scipy.linalg.solve_triangular(Rt, om.T)
    nr = np.sqrt(np.einsum("ij,ij->i", Z, Z))
    i = int(np.argmax(nr))
    return abs(alpha) / math.sqrt(d) * nr[i], i


class _State:
    """Swap-loop state — ffsrqr/srqr.py:79-171 (columns 0..l-1 factored, l = extension)."""

    def __init__(self, st, l):
        m, n = st.Aw.shape
        self.m, self.n, self.l = m, n, l
        self.Aw, self.perm = st.Aw, st.perm
        self.R = np.zeros((l + 1, n))
        self.R[:l] = st.R
        self.Q = np.eye(m, l + 1)
        self.Q[:, :l] -= st.Y @ (st.T @ st.Y[:l, :].T)          # srqr.py:91-93
        self.colsq = np.einsum("ij,ij->j", st.Aw, st.Aw)         # srqr.py:96
        s = st.B.shape[0]
        self.r = np.zeros(n)
        self.r[l:] = np.einsum("ij,ij->j", st.B[:, l:], st.B[:, l:]) / s   # srqr.py:100-101
        self.r_init = self.r.copy()
        self.anorm = float(np.linalg.norm(st.Aw))

    def exact_sq(self, i, rows):
        return max(self.colsq[i] - float(self.R[:rows, i] @ self.R[:rows, i]), 0.0)

    def _swap(self, a, b):
        if a != b:
            for M in (self.Aw, self.R):
                M[:, [a, b]] = M[:, [b, a]]
            for v in (self.perm, self.colsq, self.r, self.r_init):
                v[[a, b]] = v[[b, a]]

    def extend(self):
        """srqr.py:117-150."""
        l, n = self.l, self.n
        self._swap(l, l + int(np.argmax(self.r[l:])))
        Q1 = self.Q[:, :l]
        u = self.Aw[:, l] - Q1 @ self.R[:l, l]
        u -= Q1 @ (Q1.T @ u)
        alpha = float(np.linalg.norm(u))
        self.R[l, :] = 0.0
        if alpha <= 1e-14 * max(self.anorm, 1e-300):
            self.Q[:, l] = 0.0
            return 0.0
        q = u / alpha
        self.Q[:, l] = q
        self.R[l, l] = alpha
        self.r[l] = alpha * alpha
        if l + 1 < n:
            row = q @ self.Aw[:, l + 1:]
            self.R[l, l + 1:] = row
            self.r[l + 1:] -= row * row
            tail = self.r[l + 1:]
            for b_ in np.flatnonzero((tail < GUARD * self.r_init[l + 1:]) | (tail < 0.0)):
                i = l + 1 + int(b_)
                self.r[i] = self.exact_sq(i, l + 1)
        return alpha

    def rotate_out(self, i_off):
        """srqr.py:152-164 + givens_retriangularize/apply_rotations_right (qr.py:182-219)."""
        l = self.l
        if i_off < l:
            idx = list(range(i_off + 1, l + 1)) + [i_off]
            for M in (self.Aw, self.R):
                M[:, i_off:l + 1] = M[:, idx]
            for v in (self.perm, self.colsq, self.r, self.r_init):
                v[i_off:l + 1] = v[idx]
        R = self.R
        k, n = R.shape
        for i in range(i_off, min(k - 1, n)):
            bval = R[i + 1, i]
            if bval == 0.0:
                continue
            a = R[i, i]
            h = math.hypot(a, bval)
            c, s = a / h, bval / h
            up = c * R[i, i:] + s * R[i + 1, i:]
            lo = -s * R[i, i:] + c * R[i + 1, i:]
            R[i, i:] = up
            R[i + 1, i:] = lo
            R[i + 1, i] = 0.0
            q0 = self.Q[:, i].copy()
            q1 = self.Q[:, i + 1].copy()
            self.Q[:, i] = c * q0 + s * q1
            self.Q[:, i + 1] = -s * q0 + c * q1

    def revert(self):
        """srqr.py:166-171."""
        l, n = self.l, self.n
        self.r[l] = self.R[l, l] ** 2
        if l + 1 < n:
            self.r[l + 1:] += self.R[l, l + 1:] ** 2


def _pack(sw, alpha, g2, swaps, i_offs, trq):
    """srqr.py:213-235."""
    l, n = sw.l, sw.n
    trail = np.array([sw.exact_sq(i, l) for i in range(l, n)])
    r22 = math.sqrt(trail.max()) if trail.size else 0.0
    g1 = r22 / alpha if alpha > 0.0 else 0.0
    return OracleSrqr(
        R=sw.R[:l].copy(), perm=sw.perm.copy(), Q=sw.Q.copy(),
        rtilde=np.triu(sw.R[:l + 1, :l + 1]).copy(), alpha=abs(alpha), g1=g1, g2=g2,
        swaps=swaps, tau_bound=g1 * g2 * math.sqrt((l + 1) * (n - l)),
        tau_hat_bound=g1 * g2 * math.sqrt(l * (n - l)), r22=r22, i_offs=list(i_offs), trq=trq)


def srqr(A, prm):
    """Spectrum-revealing QR driver — ffsrqr/srqr.py:174-210.

    Raises OracleError('CertificationError', payload=OracleSrqr) at the swap cap 50*l.
    """
    A = np.asarray(A, dtype=float)
    m, n = A.shape
    l = prm["l"]
    if l + 1 > min(m, n):
        raise OracleError("DimensionError", f"srqr needs l+1 <= min(m,n); got l={l}")
    st = trqrcp(A, prm)
    sw = _State(st, l)
    alpha = sw.extend()
    swaps, g2, i_offs = 0, 0.0, []
    while alpha > 0.0:
        g2, i_off = g2_estimate(sw.R[:l + 1, :l + 1], alpha, prm["d"], prm["seed"], STREAM_G2 + swaps)
        if g2 <= prm["g"]:
            break
        if swaps >= 50 * l:
            raise OracleError("CertificationError", f"swap cap {50 * l} reached",
                              payload=_pack(sw, alpha, g2, swaps, i_offs, st))
        swaps += 1
        i_offs.append(i_off)
        sw.rotate_out(i_off)
        sw.revert()
        alpha = sw.extend()
    if alpha == 0.0:
        g2 = 0.0
    return _pack(sw, alpha, g2, swaps, i_offs, st)


# --------------------------------------------------------------------------
# Flip-Flop SRQR (Alg. 6)
# --------------------------------------------------------------------------

@dataclass
class OracleApprox:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    diag_L: np.ndarray     # signed diagonal of the partial-LQ factor (Householder convention)
    sv_all: np.ndarray     # all l singular values of tmp
    sr: OracleSrqr
    prm: dict


def flip_flop(A, k, l=None, b=32, p=5, epsilon=0.5, g=2.0, d=None, seed=0):
    """ffsrqr/svd.py:43-98: SRQR, QRNP of R^T (partial LQ), tmp = A P Qhat_1 via
    compact WY, LAPACK SVD of tmp, back-mapping of V through Qhat and perm."""
    A = np.asarray(A, dtype=float)
    m, n = A.shape
    prm = resolve(m, n, k, l, b, p, epsilon, g, d, seed)
    l = prm["l"]
    sr = srqr(A, prm)
    Rt = np.array(sr.R.T, order="F")     # a copy: the reference aliases here (svd.py:67)
    taus = qrnp_inplace(Rt, l)
    diag_L = np.diag(Rt[:l, :l]).copy()
    Y, T = wy_from_lapack(Rt, taus, l)
    Ap = A[:, sr.perm]
    tmp = Ap[:, :l] - (Ap @ Y) @ (T @ Y[:l, :].T)
    Ut, sv, Vtt = np.linalg.svd(tmp, full_matrices=False)
    W = np.zeros((n, k))
    W[:l, :] = Vtt.T[:, :k]
    W = W - Y @ (T @ (Y.T @ W))
    v = np.zeros((n, k))
    v[sr.perm, :] = W
    return OracleApprox(u=Ut[:, :k].copy(), s=sv[:k].copy(), v=v, diag_L=diag_L,
                        sv_all=sv.copy(), sr=sr, prm=prm)


def flip_flop_flops(m, n, l, b, p):
    """Paper flop budget 4mnl + 2(b+p)mn — ffsrqr/svd.py:258-260."""
    return 4 * m * n * l + 2 * (b + p) * m * n


def check_theorem_bounds(A, perm, R, Q, rtilde, u, s, v, l, slack=1e-8):
    """Restatement of ``ffsrqr/svd.py:174-255`` on explicit factors (the true
    SRQR ``R`` l x n, ``Q`` m x l, ``rtilde`` (l+1) x (l+1)).  Returns a dict
    with the report's scalars and flags."""
    A = np.asarray(A, dtype=float)
    k = s.shape[0]
    sig = np.linalg.svd(A, compute_uv=False)
    sig_l1 = float(sig[l]) if l < sig.size else 0.0
    sig_k1 = float(sig[k]) if k < sig.size else 0.0
    alpha = abs(float(rtilde[l, l]))
    if sig_l1 <= 1e-12 * max(float(sig[0]), 1e-300) or alpha == 0.0:
        return {"degenerate": True, "sv_upper_ok": bool(np.all(s <= sig[:k] * (1 + slack))),
                "all_ok": bool(np.all(s <= sig[:k] * (1 + slack)))}

    def inv_rows(T):                                   # svd.py:146-149
        inv = scipy.linalg.solve_triangular(T, np.eye(T.shape[0]))
        return float(np.sqrt(np.max(np.einsum("ij,ij->i", inv, inv))))

    M = A[:, perm] - Q[:, :l] @ R[:l]
    r22_2 = float(scipy.linalg.svdvals(M)[0])
    r22_12 = math.sqrt(float(np.max(np.einsum("ij,ij->j", M, M))))
    inv_rt, inv_r11 = inv_rows(rtilde), inv_rows(R[:l, :l])
    g1, g2 = r22_12 / alpha, alpha * inv_rt
    tau = g1 * g2 * (r22_2 / r22_12) / inv_rt / sig_l1
    tau_hat = g1 * g2 * (r22_2 / r22_12) / inv_r11 / float(s[k - 1])
    up, dn = 1 + slack, 1 - slack
    upper = bool(np.all(s <= sig[:k] * up))
    aux_lower = bool(np.all(s >= sig[:k] / np.power(1 + 2 * r22_2 ** 4 / s ** 4, 0.25) * dn))
    cap = np.minimum(2 * tau_hat ** 4, tau ** 4 * (2 + 4 * tau_hat ** 4) * (sig_l1 / sig[:k]) ** 4)
    lower = bool(np.all(s >= sig[:k] / np.power(1 + cap, 0.25) * dn))
    resid2 = float(scipy.linalg.svdvals(A - (u * s) @ v.T)[0])
    aux_budget = sig_k1 * (1 + 2 * (r22_2 / sig_k1) ** 4) ** 0.25 if sig_k1 > 0 else resid2
    budget2 = sig_k1 * (1 + 2 * tau ** 4 * (sig_l1 / sig_k1) ** 4) ** 0.25 if sig_k1 > 0 else resid2
    flags = dict(aux_lower_ok=aux_lower, sv_lower_ok=lower, sv_upper_ok=upper,
                 aux_residual_ok=bool(resid2 <= aux_budget * up),
                 residual_ok=bool(resid2 <= budget2 * up))
    return dict(degenerate=False, tau=tau, tau_hat=tau_hat, g1=g1, g2=g2, r22_2=r22_2,
                r22_12=r22_12, resid2=resid2, all_ok=all(flags.values()), **flags)
