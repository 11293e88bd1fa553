"""Tucker compression on the device — mirrors ffsrqr/tensor.py (names, arguments,
result type, errors) over the B200 engine.

Tensors live in HBM first-index-fastest (Fortran strides), exactly the
reference's storage convention (tensor.py:1-10), so the mode-0 and last-mode
unfoldings are zero-copy column- / row-major views; n-mode products run on the
engine's FP64 DMMA GEMM (``dense.gemm``), the per-mode factors on the
flip-flop / RSISVD engines.  A middle mode is moved to the front with one
layout copy first.  numpy inputs give numpy results, CUDA tensors stay on the
device.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import dense
from .engine import _torch, flip_flop_srqr, rsisvd
from .errors import DimensionError


def _fortran(t):
    """Same tensor with first-index-fastest strides (copy only when needed)."""
    rev = tuple(range(t.dim() - 1, -1, -1))
    return t.permute(rev).contiguous().permute(rev)


def _is_fortran(t):
    s = 1
    for d, st in zip(t.shape, t.stride()):
        if d > 1 and st != s:
            return False
        s *= d
    return True


def to_device(X, device=None):
    """float64 CUDA tensor with Fortran strides (numpy arrays are copied once)."""
    torch = _torch()
    if isinstance(X, torch.Tensor):
        t = X.to(device=device or (X.device if X.is_cuda else "cuda"), dtype=torch.float64)
    else:
        a = np.asarray(X, dtype=float)
        t = torch.from_numpy(np.ascontiguousarray(a.transpose(tuple(range(a.ndim - 1, -1, -1)))))
        t = t.to(device or "cuda").permute(tuple(range(a.ndim - 1, -1, -1)))
    return t if _is_fortran(t) else _fortran(t)


def _rest(shape, mode):
    r = 1
    for i, d in enumerate(shape):
        if i != mode:
            r *= d
    return r


def unfold(X, mode):
    """Mode-n unfolding (tensor.py:21-27): rows index mode n, columns the other
    modes in Fortran order.  Zero-copy for the first and last mode."""
    torch = _torch()
    if not isinstance(X, torch.Tensor):
        X = np.asarray(X)
        if not 0 <= mode < X.ndim:
            raise DimensionError(f"mode {mode} out of range for ndim {X.ndim}")
        return np.reshape(np.moveaxis(X, mode, 0), (X.shape[mode], -1), order="F")
    if not 0 <= mode < X.dim():
        raise DimensionError(f"mode {mode} out of range for ndim {X.dim()}")
    X = X if _is_fortran(X) else _fortran(X)
    rev = tuple(range(X.dim() - 1, -1, -1))
    In, R = X.shape[mode], _rest(X.shape, mode)
    if mode == 0:
        return X.permute(rev).reshape(R, In).t()
    if mode == X.dim() - 1:
        return X.permute(rev).reshape(In, R)
    return unfold(_fortran(torch.movedim(X, mode, 0)), 0)


def fold(M, mode, shape):
    """Inverse of unfold for a tensor of the given shape (tensor.py:30-38)."""
    torch = _torch()
    shape = tuple(int(s) for s in shape)
    if not 0 <= mode < len(shape):
        raise DimensionError(f"mode {mode} out of range for shape {shape}")
    if tuple(M.shape) != (shape[mode], int(np.prod(shape)) // shape[mode]):
        raise DimensionError(f"unfolded shape {tuple(M.shape)} does not match {shape}")
    if not isinstance(M, torch.Tensor):
        lead = (shape[mode],) + shape[:mode] + shape[mode + 1:]
        return np.moveaxis(np.reshape(M, lead, order="F"), 0, mode)
    lead = (shape[mode],) + shape[:mode] + shape[mode + 1:]
    Mc = M.t().contiguous().t() if M.stride(0) != 1 else M        # column-major
    rev = tuple(range(len(lead) - 1, -1, -1))
    T = Mc.t().reshape(tuple(reversed(lead))).permute(rev)        # Fortran (lead)
    return _fortran(torch.movedim(T, 0, mode))


def nmode_product(X, U, mode):
    """Tensor-times-matrix along one mode (tensor.py:41-52) on the DMMA GEMM."""
    torch = _torch()
    if not isinstance(X, torch.Tensor):
        out = nmode_product(to_device(X), torch.as_tensor(np.asarray(U, float), device="cuda"), mode)
        return out.cpu().numpy()
    if U.dim() != 2 or U.shape[1] != X.shape[mode]:
        raise DimensionError(f"matrix {tuple(U.shape)} cannot contract mode {mode} of tensor "
                             f"{tuple(X.shape)}")
    X = X if _is_fortran(X) else _fortran(X)
    U = U.to(device=X.device, dtype=torch.float64)
    nd = X.dim()
    J = U.shape[0]
    shape = list(X.shape)
    shape[mode] = J
    rev = tuple(range(nd - 1, -1, -1))
    R = _rest(X.shape, mode)
    if mode == 0:
        C = dense.gemm(U, unfold(X, 0))                            # (J x R) col-major
        return C.t().reshape(tuple(reversed(shape))).permute(rev)
    if mode == nd - 1:
        Xc = X.permute(rev).reshape(X.shape[mode], R).t()          # (R x I_n) col-major
        C = dense.gemm(Xc, U.t())                                  # (R x J) col-major
        return C.t().reshape(tuple(reversed(shape))).permute(rev)
    Y = nmode_product(_fortran(torch.movedim(X, mode, 0)), U, 0)
    return _fortran(torch.movedim(Y, 0, mode))


@dataclass
class TuckerDecomp:
    """tensor.py:55-70."""
    core: object
    factors: list
    flop_count: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def ranks(self):
        return tuple(U.shape[1] for U in self.factors)

    def reconstruct(self):
        G = self.core
        for n, U in enumerate(self.factors):
            G = nmode_product(G, U, n)
        return G


def _make_engine(engine, seed):
    """tensor.py:73-91 on the device engines."""
    if callable(engine):
        return engine
    if engine == "flipflop":
        def _ff(M, r):
            m = M.shape[0]
            l = min(r + 5, min(M.shape) - 1)
            b = min(32, max(m - 5, 1))
            p = min(5, max(m - b, 0))
            return flip_flop_srqr(M, r, l=max(l, r), b=b, p=p, seed=seed)
        return _ff
    if engine == "rsisvd":
        return lambda M, r: rsisvd(M, r, seed=seed)
    if engine == "exact":
        # full-width RSISVD with no power step is an exact SVD (Q spans range(M))
        def _exact(M, r):
            mn = min(M.shape)
            return rsisvd(M, r, p=mn - r, q=0, seed=seed)
        return _exact
    raise ValueError(f"unknown low-rank engine {engine!r}")


def _check_ranks(shape, ranks):
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != len(shape):
        raise DimensionError(f"need one rank per mode: got {ranks} for {tuple(shape)}")
    for r, s in zip(ranks, shape):
        if not 1 <= r <= s:
            raise DimensionError(f"rank {r} invalid for mode of size {s}")
    return ranks


def _out(x, as_np):
    return x.detach().cpu().numpy() if as_np else x


def hosvd(X, ranks, engine="exact", seed=0):
    """Higher-order SVD (tensor.py:104-120): factors from the original tensor's
    unfoldings, core formed at the end with DMMA n-mode products."""
    torch = _torch()
    as_np = not isinstance(X, torch.Tensor)
    Xd = to_device(X)
    ranks = _check_ranks(Xd.shape, ranks)
    solve = _make_engine(engine, seed)
    factors, fl = [], 0
    for n, r in enumerate(ranks):
        ap = solve(unfold(Xd, n), r)
        factors.append(torch.as_tensor(ap.u, device=Xd.device))
        fl += ap.flop_count
    G = Xd
    for n, U in enumerate(factors):
        G = nmode_product(G, U.t(), n)
    return TuckerDecomp(core=_out(G, as_np), factors=[_out(U, as_np) for U in factors], flop_count=fl,
                        meta={"engine": engine, "method": "hosvd"})


def st_hosvd(X, ranks, engine="exact", seed=0, order=None):
    """Sequentially truncated HOSVD (tensor.py:123-145)."""
    torch = _torch()
    as_np = not isinstance(X, torch.Tensor)
    Xd = to_device(X)
    ranks = _check_ranks(Xd.shape, ranks)
    solve = _make_engine(engine, seed)
    if order is None:
        order = sorted(range(Xd.dim()), key=lambda n: Xd.shape[n])
    else:
        order = list(order)
        if sorted(order) != list(range(Xd.dim())):
            raise DimensionError(f"order {order} is not a permutation of the modes")
    factors = [None] * Xd.dim()
    G, fl = Xd, 0
    for n in order:
        ap = solve(unfold(G, n), ranks[n])
        U = torch.as_tensor(ap.u, device=Xd.device)
        factors[n] = U
        fl += ap.flop_count
        G = nmode_product(G, U.t(), n)
    return TuckerDecomp(core=_out(G, as_np), factors=[_out(U, as_np) for U in factors], flop_count=fl,
                        meta={"engine": engine, "method": "st_hosvd", "order": order})


def tucker_error(X, decomp):
    """Relative Frobenius reconstruction error (tensor.py:146-152)."""
    torch = _torch()
    Xd = to_device(X)
    nrm = float(torch.sqrt(dense.sumsq(Xd.reshape(-1)))[0])
    if nrm == 0.0:
        return 0.0
    core = to_device(decomp.core)
    fac = [torch.as_tensor(U, device=Xd.device, dtype=torch.float64) for U in decomp.factors]
    R = TuckerDecomp(core, fac).reconstruct()
    return float(torch.sqrt(dense.sumsq((Xd - R).reshape(-1)))[0]) / nrm
