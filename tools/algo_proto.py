"""Numpy prototype of the B200 engine's *formulation* (design validation only).

Not part of the product and not the oracle: it mirrors, in float64 numpy,
the exact sequence of operations the CUDA path performs, so the numerics of
the re-formulation can be checked against the reference goldens on CPU:

* storage in ORIGINAL column order + an arrangement array ``arr`` (no
  physical reorders);
* dense-Q blocked TRQRCP: panel = A[:,piv] - Q_prev R_prev[:,piv], one
  re-orthogonalisation pass (BCGS2), shifted CholeskyQR3, then
  Householder-convention signs recovered from an LU of the leading block of
  Q - I (Ballard et al.'s reconstruction pivots);
* R rows as one GEMM Q_blk^T A; sketch update B -= (B_piv R11^-1) R12;
* partial LQ of R via shifted CholeskyQR3 of R^T + the same sign rule;
* tmp = A (Pi Qhat1); QR(tmp) by CholeskyQR; Jacobi-free small SVD here
  (numpy), one-sided Jacobi on the device.
"""

import math
import os
import sys

import numpy as np
import scipy.linalg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (checker + qrcp semantics)

U64 = np.finfo(float).eps / 2


def chol_qr3(X):
    """Shifted CholeskyQR3 (Fukaya et al. 2020). Returns Q, R (upper, positive diag)."""
    M, N = X.shape
    G = X.T @ X
    shift = 11.0 * (M * N + N * (N + 1)) * U64 * np.trace(G)
    R1 = np.linalg.cholesky(G + shift * np.eye(N)).T
    Q = scipy.linalg.solve_triangular(R1, X.T, trans="T").T
    R = R1
    for _ in range(2):
        G = Q.T @ Q
        R2 = np.linalg.cholesky(G).T
        Q = scipy.linalg.solve_triangular(R2, Q.T, trans="T").T
        R = R2 @ R
    return Q, R


class SignLU:
    """Incremental LU of (Q D - I) on the leading block; picks D column by column."""

    def __init__(self, N):
        self.L = np.eye(N)
        self.U = np.zeros((N, N))
        self.nc = 0

    def add_columns(self, Qtop):
        """Qtop: (N x w) rows 0..N-1 of the new Q columns (unscaled). Returns D (w,)."""
        c0 = self.nc
        w = Qtop.shape[1]
        L, U = self.L, self.U
        D = np.ones(w)
        N = L.shape[0]
        for t in range(w):
            c = c0 + t
            y = Qtop[:, t]
            u = scipy.linalg.solve_triangular(L[:c, :c], y[:c], lower=True, unit_diagonal=True) if c else np.zeros(0)
            z = y[c] - L[c, :c] @ u
            if abs(z) == 1.0:          # identity-reflector branch (tail exactly 0)
                d = 1.0 if z > 0 else -1.0
            else:
                d = -1.0 if z > 0 else 1.0
            D[t] = d
            U[:c, c] = d * u
            ucc = d * z - 1.0
            U[c, c] = ucc
            if c + 1 < N:
                if ucc != 0.0:
                    L[c + 1:, c] = (d * y[c + 1:] - L[c + 1:, :c] @ U[:c, c]) / ucc
                else:
                    L[c + 1:, c] = 0.0
        self.nc += w
        return D


def proto_flip_flop(A, k, l, b, p, g=2.0, d=None, seed=0):
    A = np.asarray(A, dtype=float)
    m, n = A.shape
    prm = oracle.resolve(m, n, k, l, b, p, g=g, d=d, seed=seed)
    l, b, p, d = prm["l"], prm["b"], prm["p"], prm["d"]
    s = b + p
    Om = oracle.gaussian(s, m, seed, 0)
    B = Om @ A
    colsq = np.einsum("ij,ij->j", A, A)
    arr = np.arange(n)
    Q = np.zeros((m, l + 1))
    R = np.zeros((l + 1, n))
    slu = SignLU(l)
    j0 = 0
    while j0 < l:
        bb = min(b, l - j0)
        e = j0 + bb
        order = j0 + oracle.qrcp_pivots(np.array(B[:, arr[j0:]], order="F"), bb)
        arr[j0:] = arr[order]
        piv = arr[j0:e]
        P = A[:, piv] - Q[:, :j0] @ R[:j0, piv]
        if j0:
            P -= Q[:, :j0] @ (Q[:, :j0].T @ P)
        Qb, Rb = chol_qr3(P)
        D = slu.add_columns(Qb[:l, :])
        Qb *= D
        Rb = D[:, None] * Rb
        Q[:, j0:e] = Qb
        R[j0:e, :] = Qb.T @ A
        R[j0:e, piv] = np.triu(Rb)
        if j0:
            R[j0:e, arr[:j0]] = 0.0
        if e < n:
            Z = scipy.linalg.solve_triangular(Rb, B[:, piv].T, trans="T").T   # B_piv R11^-1
            B[:, arr[e:]] -= Z @ R[j0:e, arr[e:]]
        j0 = e
    # ---- SRQR (swap loop in arrangement order, same as oracle semantics)
    r = np.zeros(n)
    r[l:] = np.einsum("ij,ij->j", B[:, arr[l:]], B[:, arr[l:]]) / s
    anorm = math.sqrt(colsq.sum())
    pos_r = r  # by position
    q_ = int(np.argmax(pos_r[l:])) + l
    arr[[l, q_]] = arr[[q_, l]]
    pos_r[[l, q_]] = pos_r[[q_, l]]
    Q1 = Q[:, :l]
    u = A[:, arr[l]] - Q1 @ R[:l, arr[l]]
    u -= Q1 @ (Q1.T @ u)
    alpha = float(np.linalg.norm(u))
    if alpha <= 1e-14 * max(anorm, 1e-300):
        alpha = 0.0
    else:
        Q[:, l] = u / alpha
    Rarr = np.triu(R[:l + 1, arr])
    Rarr[l, l] = alpha
    g2 = 0.0
    if alpha > 0:
        g2, i_off = oracle.ffsrqr_oracle.g2_estimate(Rarr[:, :l + 1], alpha, d, seed, 1000)
        assert g2 <= g, "prototype covers the no-swap path only"
    trail = np.maximum(colsq[arr[l:]] - np.einsum("ij,ij->j", Rarr[:l, l:], Rarr[:l, l:]), 0)
    r22 = math.sqrt(trail.max())
    g1 = r22 / alpha if alpha > 0 else 0.0
    # ---- flip-flop
    X = Rarr[:l, :].T.copy()
    Qh, Lt = chol_qr3(X)
    Dl = SignLU(l).add_columns(Qh[:l, :])
    Qh *= Dl
    diag_L = Dl * np.diag(Lt)
    Yh = np.zeros((n, l))
    Yh[arr] = Qh
    tmp = A @ Yh
    Qt, Rt = chol_qr3(tmp)
    Us, sv, Vst = np.linalg.svd(Rt)
    u_ = Qt @ Us[:, :k]
    v_ = Yh @ Vst.T[:, :k]
    return dict(perm=arr.copy(), R=Rarr[:l], Q=Q, rtilde=Rarr[:, :l + 1], alpha=alpha, g1=g1,
                g2=g2, r22=r22, s=sv[:k], diag_L=diag_L, u=u_, v=v_)


if __name__ == "__main__":
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import load, names

    for nm in names():
        c = load(nm)
        if c["cert"][3] > 0 or "s" not in c:
            print(f"{nm:16s} (swap path / no flip-flop: skipped in prototype)")
            continue
        out = proto_flip_flop(c["A"], c["k"], c["l"], c["b"], c["p"], g=c["g"], d=c["d"], seed=c["seed"])
        perm_ok = np.array_equal(out["perm"], c["perm"])
        rel = lambda a, b_: float(np.max(np.abs(a - b_) / np.maximum(np.abs(b_), 1e-300)))
        es = rel(out["s"], c["s"])
        edl = rel(out["diag_L"], c["diag_L"])
        eR = float(np.max(np.abs(out["R"] - c["R"])) / np.max(np.abs(c["R"])))
        ert = float(np.max(np.abs(out["rtilde"] - c["rtilde"])) / np.max(np.abs(c["rtilde"])))
        cert = np.array([out["alpha"], out["g1"], out["g2"]])
        ec = rel(cert, c["cert"][:3]) if c["cert"][0] > 0 else float(np.max(np.abs(cert - c["cert"][:3])))
        print(f"{nm:16s} perm={perm_ok} s={es:.1e} diagL={edl:.1e} R={eR:.1e} rtilde={ert:.1e} cert={ec:.1e}")


# =====================================================================
# Variant H (the one the CUDA path implements): compact-WY TRQRCP like the
# reference, every Householder panel factored by shifted CholeskyQR3 +
# local Householder reconstruction (LU of Q_top*D - I, D chosen so the
# pivots are <= -1, i.e. the reference's alpha = -sign(x0)||x|| branch).
# =====================================================================

def recon_panel(X):
    """X (M' x w), M' >= w -> (Y unit-lower-trapezoidal, T upper, R upper) with
    Householder-convention signs (same as ffsrqr/_kernels_numpy.py:84-109)."""
    Mp, w = X.shape
    Qp, Rp = chol_qr3(X)
    Qtop = Qp[:w, :]
    L = np.eye(w)
    U = np.zeros((w, w))
    D = np.ones(w)
    for c in range(w):
        y = Qtop[:, c]
        u = scipy.linalg.solve_triangular(L[:c, :c], y[:c], lower=True, unit_diagonal=True) if c else np.zeros(0)
        z = y[c] - L[c, :c] @ u
        d = (1.0 if z > 0 else -1.0) if abs(z) == 1.0 else (-1.0 if z > 0 else 1.0)
        D[c] = d
        U[:c, c] = d * u
        U[c, c] = d * z - 1.0
        if c + 1 < w:
            L[c + 1:, c] = ((d * y[c + 1:] - L[c + 1:, :c] @ U[:c, c]) / U[c, c]) if U[c, c] != 0.0 else 0.0
    QD = Qp * D
    Y = np.zeros((Mp, w))
    Y[:w] = L
    rhs = QD[w:]
    for c in range(w):   # Y2 U = QD[w:]  (column-sequential, zero-pivot -> zero column)
        Y[w:, c] = ((rhs[:, c] - Y[w:, :c] @ U[:c, c]) / U[c, c]) if U[c, c] != 0.0 else 0.0
    T = -scipy.linalg.solve_triangular(L, U.T, lower=True, unit_diagonal=True).T   # -U L^{-T}
    return Y, T, D[:, None] * Rp


def householder_blocked(X, w):
    """Blocked Householder QR of X (M x N) with recon panels of width w.
    Returns Y (M x N), T (N x N), R (N x N)."""
    M, N = X.shape
    X = X.copy()
    Y = np.zeros((M, N))
    T = np.zeros((N, N))
    R = np.zeros((N, N))
    for c0 in range(0, N, w):
        c1 = min(N, c0 + w)
        Yp, Tp, Rp = recon_panel(X[c0:, c0:c1])
        Y[c0:, c0:c1] = Yp
        R[c0:c1, c0:c1] = np.triu(Rp)
        if c1 < N:
            R[c0:c1, c1:] = X[c0:c1, c1:] - Yp[:c1 - c0] @ (Tp.T @ (Yp.T @ X[c0:, c1:]))
            X[c0:, c1:] -= Yp @ (Tp.T @ (Yp.T @ X[c0:, c1:]))
        T[:c0, c0:c1] = -T[:c0, :c0] @ (Y[:, :c0].T @ Y[:, c0:c1]) @ Tp
        T[c0:c1, c0:c1] = Tp
    return Y, T, R


def proto_h(A, k, l, b, p, g=2.0, d=None, seed=0, w_lq=64):
    A = np.asarray(A, dtype=float)
    m, n = A.shape
    prm = oracle.resolve(m, n, k, l, b, p, g=g, d=d, seed=seed)
    l, b, p, d = prm["l"], prm["b"], prm["p"], prm["d"]
    s = b + p
    Om = oracle.gaussian(s, m, seed, 0)
    B = Om @ A
    colsq = np.einsum("ij,ij->j", A, A)
    arr = np.arange(n)
    Y = np.zeros((m, l))
    T = np.zeros((l, l))
    WT = np.zeros((l, n))
    R = np.zeros((l + 1, n))
    j0 = 0
    while j0 < l:
        bb = min(b, l - j0)
        e = j0 + bb
        order = j0 + oracle.qrcp_pivots(np.array(B[:, arr[j0:]], order="F"), bb)
        arr[j0:] = arr[order]
        piv = arr[j0:e]
        P = A[:, piv] - Y[:, :j0] @ WT[:j0, piv]
        Yb, Tb, Rb = recon_panel(P[j0:, :])
        Y[j0:, j0:e] = Yb
        T[:j0, j0:e] = -T[:j0, :j0] @ (Y[:, :j0].T @ Y[:, j0:e]) @ Tb
        T[j0:e, j0:e] = Tb
        WT[j0:e, :] = Tb.T @ (Y[:, j0:e].T @ A - (Y[:, j0:e].T @ Y[:, :j0]) @ WT[:j0, :])
        R[j0:e, :] = A[j0:e, :] - Y[j0:e, :e] @ WT[:e, :]
        R[j0:e, piv] = np.triu(Rb)
        if j0:
            R[j0:e, arr[:j0]] = 0.0
        if e < n:
            Z = scipy.linalg.solve_triangular(Rb, B[:, piv].T, trans="T").T
            B[:, arr[e:]] -= Z @ R[j0:e, arr[e:]]
        j0 = e
    Q = np.zeros((m, l + 1))
    Q[:, :l] = np.eye(m, l) - Y @ (T @ Y[:l, :].T)
    r = np.zeros(n)
    r[l:] = np.einsum("ij,ij->j", B[:, arr[l:]], B[:, arr[l:]]) / s
    anorm = math.sqrt(colsq.sum())
    q_ = int(np.argmax(r[l:])) + l
    arr[[l, q_]] = arr[[q_, l]]
    Q1 = Q[:, :l]
    u = A[:, arr[l]] - Q1 @ R[:l, arr[l]]
    u -= Q1 @ (Q1.T @ u)
    alpha = float(np.linalg.norm(u))
    if alpha <= 1e-14 * max(anorm, 1e-300):
        alpha = 0.0
    else:
        Q[:, l] = u / alpha
    Rarr = np.triu(R[:l + 1, arr])
    Rarr[l, l] = alpha
    g2 = 0.0
    if alpha > 0:
        g2, i_off = oracle.ffsrqr_oracle.g2_estimate(Rarr[:, :l + 1], alpha, d, seed, 1000)
        assert g2 <= g, "prototype covers the no-swap path only"
    trail = np.maximum(colsq[arr[l:]] - np.einsum("ij,ij->j", Rarr[:l, l:], Rarr[:l, l:]), 0)
    r22 = math.sqrt(trail.max())
    g1 = r22 / alpha if alpha > 0 else 0.0
    Yl, Tl, Ll = householder_blocked(Rarr[:l, :].T.copy(), w_lq)
    diag_L = np.diag(Ll).copy()
    Qh = np.eye(n, l) - Yl @ (Tl @ Yl[:l, :].T)
    Yh = np.zeros((n, l))
    Yh[arr] = Qh
    tmp = A @ Yh
    Qt, Rt = chol_qr3(tmp)
    Us, sv, Vst = np.linalg.svd(Rt)
    return dict(perm=arr.copy(), R=Rarr[:l], Q=Q, rtilde=Rarr[:, :l + 1], alpha=alpha, g1=g1,
                g2=g2, r22=r22, s=sv[:k], diag_L=diag_L, u=Qt @ Us[:, :k], v=Yh @ Vst.T[:, :k])


def _report(fn):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import load, names

    for nm in names():
        c = load(nm)
        if c["cert"][3] > 0 or "s" not in c:
            continue
        out = fn(c["A"], c["k"], c["l"], c["b"], c["p"], g=c["g"], d=c["d"], seed=c["seed"])
        perm_ok = np.array_equal(out["perm"], c["perm"])
        rel = lambda a, b_: float(np.max(np.abs(a - b_) / np.maximum(np.abs(b_), 1e-300)))
        es = rel(out["s"], c["s"])
        edl = rel(out["diag_L"], c["diag_L"])
        eR = float(np.max(np.abs(out["R"] - c["R"])) / np.max(np.abs(c["R"])))
        ert = float(np.max(np.abs(out["rtilde"] - c["rtilde"])) / np.max(np.abs(c["rtilde"])))
        cert = np.array([out["alpha"], out["g1"], out["g2"]])
        ec = rel(cert, c["cert"][:3]) if c["cert"][0] > 0 else float(np.max(np.abs(cert - c["cert"][:3])))
        print(f"H {nm:16s} perm={perm_ok} s={es:.1e} diagL={edl:.1e} R={eR:.1e} rtilde={ert:.1e} cert={ec:.1e}")
