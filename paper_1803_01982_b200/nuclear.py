"""Nuclear-norm minimization (IALM) on the device — mirrors ffsrqr/nuclear.py
(IalmParams, IalmState, ialm_rpca, ialm_mc, soft_shrink, nmae) over the B200
engine.

Per iteration: the partial SVD (flip-flop / RSISVD engine, device-resident
input, no host copies), the shrunk low-rank product X = (U (s - 1/mu)) V^T
(``ffb_shrink_cols`` + one DMMA GEMM), and ONE fused HBM pass
(``ffb_ialm_update``) for the sparse/slack update, the residual Z, the
multiplier Y, the next SVD input and ||Z||_F.  The only host reads per
iteration are the singular values (to count what survives the threshold, as
the reference does) and ||Z||_F.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi, dense
from .engine import _torch, flip_flop_srqr, rsisvd
from .errors import DimensionError, NumericalError


def soft_shrink(X, tau):
    """Entrywise soft-thresholding (nuclear.py:21-23); numpy in, numpy out."""
    torch = _torch()
    if isinstance(X, torch.Tensor):
        return torch.sign(X) * torch.clamp(torch.abs(X) - tau, min=0.0)
    return np.sign(X) * np.maximum(np.abs(X) - tau, 0.0)


@dataclass
class IalmParams:
    """nuclear.py:26-37."""
    lam: float = None
    mu0: float = None
    mu_bar: float = None
    rho: float = 1.5
    tol: float = 1e-7
    max_iter: int = 100
    sv0: int = 10
    svd_engine: str = "exact"
    seed: int = 0


@dataclass
class IalmState:
    """nuclear.py:40-50."""
    low_rank: object
    sparse: object
    rank: int
    iterations: int
    converged: bool
    residuals: list = field(default_factory=list)
    ranks: list = field(default_factory=list)
    mus: list = field(default_factory=list)
    iterates: list = field(default_factory=list)


class _PartialSvd:
    """nuclear.py:52-78 on the device engines."""

    def __init__(self, engine, seed, min_dim):
        self.engine = engine
        self.seed = seed
        self.min_dim = min_dim
        self.cap = min_dim if engine == "exact" else max(min_dim - 1, 1)

    def __call__(self, M, sv):
        sv = min(sv, self.cap)
        if self.engine == "exact" or sv >= self.min_dim:
            ap = rsisvd(M, sv, p=self.min_dim - sv, q=0, seed=self.seed)
        elif self.engine == "flipflop":
            l = min(sv + 60, self.min_dim - 1)
            ap = flip_flop_srqr(M, sv, l=l, seed=self.seed)
        elif self.engine == "rsisvd":
            ap = rsisvd(M, sv, seed=self.seed)
        else:
            raise ValueError(f"unknown svd engine {self.engine!r}")
        return ap.u, ap.s, ap.v


def _grow_sv(rank, sv, min_dim):
    """nuclear.py:81-88."""
    if rank < sv:
        return min(rank + 1, min_dim)
    nxt = sv + 5 if sv <= 50 else int(round(1.1 * sv))
    return min(nxt, min_dim)


def _shrink_spectrum(psvd, W, sv, mu):
    """nuclear.py:91-97: X = U[:, :keep] diag(s - 1/mu) V[:, :keep]^T."""
    torch = _torch()
    U, s, V = psvd(W, sv)
    s_host = s.detach().cpu().numpy()
    keep = int(np.count_nonzero(s_host > 1.0 / mu))
    m, n = W.shape
    X = dense.colmajor(torch, m, n, W.device)
    if keep == 0:
        X.zero_()
        return X, 0
    Us = dense.colmajor(torch, m, keep, W.device)
    lib = _capi.load()
    with torch.cuda.device(W.device):
        stream = torch.cuda.current_stream(W.device).cuda_stream
        rc = lib.ffb_shrink_cols(C.c_void_p(stream), C.c_void_p(U.data_ptr()), U.stride(1), m, keep,
                                 C.c_void_p(s.data_ptr()), 1.0 / mu, C.c_void_p(Us.data_ptr()), m)
    if rc != _capi.FFB_OK:
        raise RuntimeError(f"ffb_shrink_cols failed ({rc})")
    dense.gemm(Us, V[:, :keep].t(), out=X)
    return X, keep


def _device_matrix(M):
    torch = _torch()
    as_np = not isinstance(M, torch.Tensor)
    if as_np:
        a = np.asarray(M, dtype=float)
        t = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    else:
        t = M.to(dtype=torch.float64, device=M.device if M.is_cuda else "cuda")
        if t.stride(0) != 1 or t.stride(1) != t.shape[0]:
            t = t.t().contiguous().t()
    return t, as_np


def _update(mode, M, X, Y, E, mask, mu, thresh, mu_next, W, part, zsq):
    torch = _torch()
    lib = _capi.load()
    with torch.cuda.device(M.device):
        stream = torch.cuda.current_stream(M.device).cuda_stream
        rc = lib.ffb_ialm_update(C.c_void_p(stream), mode, C.c_void_p(M.data_ptr()),
                                 C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()),
                                 C.c_void_p(E.data_ptr()), C.c_void_p(mask.data_ptr() if mask is not None else 0),
                                 M.numel(), float(mu), float(thresh), float(mu_next),
                                 C.c_void_p(W.data_ptr()), C.c_void_p(part.data_ptr()),
                                 C.c_void_p(zsq.data_ptr()))
    if rc != _capi.FFB_OK:
        raise RuntimeError(f"ffb_ialm_update failed ({rc})")


def _run(mode, Md, maskd, p, lam, mu, mu_bar, normF, Y, record_iterates, as_np):
    torch = _torch()
    m, n = Md.shape
    E = torch.zeros_like(Md)
    W = Md - E + Y / mu                       # first partial-SVD input
    W = W.t().contiguous().t()
    psvd = _PartialSvd(p.svd_engine, p.seed, min(m, n))
    sv = min(p.sv0, min(m, n))
    part = torch.empty(_capi.load().ffb_svt_partials(), dtype=torch.float64, device=Md.device)
    zsq = torch.empty(1, dtype=torch.float64, device=Md.device)
    st = IalmState(torch.zeros_like(Md), E, 0, 0, False)
    cv = (lambda t: t.detach().cpu().numpy()) if as_np else (lambda t: t)
    for it in range(1, p.max_iter + 1):
        X, rank = _shrink_spectrum(psvd, W, sv, mu)
        sv = _grow_sv(rank, sv, min(m, n))
        mu_next = min(p.rho * mu, mu_bar)
        _update(mode, Md, X, Y, E, maskd, mu, lam / mu if mode == 0 else 0.0, mu_next, W, part, zsq)
        st.mus.append(mu)
        mu = mu_next
        res = math.sqrt(float(zsq[0])) / normF
        st.residuals.append(res)
        st.ranks.append(rank)
        if record_iterates:
            st.iterates.append((cv(X.clone()), cv(E.clone())))
        st.low_rank, st.sparse, st.rank, st.iterations = X, E, rank, it
        if res < p.tol:
            st.converged = True
            break
    st.low_rank, st.sparse = cv(st.low_rank), cv(st.sparse.clone())
    return st


def ialm_rpca(M, params=None, record_iterates=False):
    """Robust PCA, M = low_rank + sparse (nuclear.py:105-145), on the device."""
    torch = _torch()
    if len(tuple(M.shape)) != 2:
        raise DimensionError("ialm_rpca expects a matrix")
    Md, as_np = _device_matrix(M)
    if not bool(torch.isfinite(Md).all()):
        raise NumericalError("ialm_rpca input contains non-finite entries")
    p = params or IalmParams()
    m, n = Md.shape
    lam = p.lam if p.lam is not None else 1.0 / np.sqrt(max(m, n))
    normF = math.sqrt(float(dense.sumsq(Md)[0]))
    if normF == 0.0:
        z = torch.zeros_like(Md)
        zz = z.cpu().numpy() if as_np else z
        return IalmState(zz, zz.copy() if as_np else z.clone(), 0, 0, True)
    norm2 = dense.spectral_norm(Md)
    mu = p.mu0 if p.mu0 is not None else 1.25 / norm2
    mu_bar = p.mu_bar if p.mu_bar is not None else mu * 1e7
    Y = Md / max(norm2, float(Md.abs().max()))
    Y = Y.t().contiguous().t()
    return _run(0, Md, None, p, lam, mu, mu_bar, normF, Y, record_iterates, as_np)


def ialm_mc(M, mask, params=None, record_iterates=False):
    """Matrix completion from the observed entries (nuclear.py:148-191), on the device."""
    torch = _torch()
    if tuple(M.shape) != tuple(mask.shape) or len(tuple(M.shape)) != 2:
        raise DimensionError("ialm_mc needs a matrix and a same-shaped mask")
    Md, as_np = _device_matrix(M)
    mk = mask if isinstance(mask, torch.Tensor) else torch.from_numpy(np.asarray(mask, dtype=bool))
    maskd = mk.to(device=Md.device, dtype=torch.uint8).t().contiguous().t()
    Md = torch.where(maskd.bool(), Md, torch.zeros((), dtype=Md.dtype, device=Md.device))
    Md = Md.t().contiguous().t()
    if not bool(torch.isfinite(Md).all()):
        raise NumericalError("ialm_mc observed entries contain non-finite values")
    p = params or IalmParams()
    norm2 = dense.spectral_norm(Md)
    if norm2 == 0.0:
        z = torch.zeros_like(Md)
        zz = z.cpu().numpy() if as_np else z
        return IalmState(zz, zz.copy() if as_np else z.clone(), 0, 0, True)
    mu = p.mu0 if p.mu0 is not None else 1.25 / norm2
    mu_bar = p.mu_bar if p.mu_bar is not None else mu * 1e7
    normF = math.sqrt(float(dense.sumsq(Md)[0]))
    Y = torch.zeros_like(Md)
    return _run(1, Md, maskd, p, 0.0, mu, mu_bar, normF, Y, record_iterates, as_np)


def nmae(truth, predicted, mask, lo, hi):
    """nuclear.py:194-204 (host-side metric)."""
    mask = np.asarray(mask, dtype=bool)
    cnt = int(mask.sum())
    if cnt == 0:
        raise DimensionError("nmae needs at least one evaluation entry")
    if hi <= lo:
        raise DimensionError("nmae needs hi > lo")
    t = truth.detach().cpu().numpy() if hasattr(truth, "detach") else np.asarray(truth, dtype=float)
    pr = predicted.detach().cpu().numpy() if hasattr(predicted, "detach") else np.asarray(predicted, dtype=float)
    err = np.abs(t - pr)
    return float(err[mask].sum() / (cnt * (hi - lo)))
