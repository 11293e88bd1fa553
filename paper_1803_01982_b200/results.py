"""Result/parameter types mirroring the reference's public dataclasses.

SketchParams  — ffsrqr/sketch.py:22-59 (same fields, defaults and validation)
WYFactor      — ffsrqr/qr.py:46-80
PartialFactorization — ffsrqr/qr.py:118-141
SrqrCertificate, SrqrResult — ffsrqr/srqr.py:30-46
ApproxSvd     — ffsrqr/svd.py:24-40
Arrays are numpy when the caller passed numpy, torch CUDA tensors otherwise.
"""
from dataclasses import dataclass, field, replace

import numpy as np

from .errors import DimensionError


def _np(x):
    if isinstance(x, np.ndarray):
        return x
    return x.detach().cpu().numpy()


@dataclass
class SketchParams:
    k: int
    l: int = None
    b: int = 32
    p: int = 5
    epsilon: float = 0.5
    g: float = 2.0
    d: int = None
    seed: int = 0

    def resolve(self, m, n):
        l = self.k if self.l is None else self.l
        d = min(l, 10) if self.d is None else self.d
        out = replace(self, l=l, d=d)
        if not 1 <= self.k <= l <= min(m, n):
            raise DimensionError(f"need 1 <= k <= l <= min(m,n); got k={self.k}, l={l}")
        if out.b < 1 or out.p < 0:
            raise DimensionError("need b >= 1 and p >= 0")
        if not 0.0 < out.epsilon < 1.0:
            raise DimensionError("epsilon must lie in (0,1)")
        if out.g <= 1.0:
            raise DimensionError("g must exceed 1")
        if not 1 <= d <= l:
            raise DimensionError("need 1 <= d <= l")
        if out.b + out.p > m:
            raise DimensionError(f"sketch rows b+p={out.b + out.p} exceed m={m}; no compression")
        return out


@dataclass
class WYFactor:
    """Q = I - Y T Y^T (Y unit lower trapezoidal m x j, T upper j x j)."""

    Y: object
    T: object

    @property
    def j(self):
        return self.Y.shape[1]

    @property
    def m(self):
        return self.Y.shape[0]

    def q(self, ncols=None):
        Y, T = _np(self.Y), _np(self.T)
        ncols = self.m if ncols is None else ncols
        E = np.eye(self.m, ncols)
        if self.j == 0:
            return E
        return E - Y @ (T @ (Y.T @ E))

    def apply_left(self, C, transpose=False):
        Y, T = _np(self.Y), _np(self.T)
        if C.shape[0] != self.m:
            raise DimensionError("row mismatch in WY apply")
        if self.j == 0:
            return C.copy()
        TT = T.T if transpose else T
        return C - Y @ (TT @ (Y.T @ C))


class _HostOnAccess:
    """Large factor arrays of a numpy-in call stay in HBM until first read, then
    are copied to the host once (numpy out, like the reference): a caller that
    only uses u, s, v (the HOSVD / SVT callers, tensor.py:114, nuclear.py:74)
    never pays the PCIe transfer of R, Q and R-tilde."""

    _lazy_fields = ()
    _host = False

    def __getattribute__(self, name):
        v = object.__getattribute__(self, name)
        if name in type(self)._lazy_fields and hasattr(v, "detach") and \
                object.__getattribute__(self, "_host"):
            v = v.detach().cpu().numpy()
            object.__setattr__(self, name, v)
        return v


@dataclass
class PartialFactorization(_HostOnAccess):
    """A[:, perm] ~ Q[:, :k] @ R with R k-by-n."""

    _lazy_fields = ("R", "q_dense")

    R: object
    perm: object
    k: int
    wy: WYFactor = None
    q_dense: object = None

    def q(self):
        if self.q_dense is not None:
            return self.q_dense
        return self.wy.q(self.k)

    def reconstruction_error(self, A):
        A = _np(A)
        lead = A[:, _np(self.perm)[: self.k]]
        return float(np.linalg.norm(lead - _np(self.q()) @ _np(self.R)[:, : self.k]))


@dataclass
class SrqrCertificate:
    alpha: float
    g1: float
    g2: float
    swaps: int
    tau_bound: float
    tau_hat_bound: float


@dataclass
class SrqrResult(_HostOnAccess):
    _lazy_fields = ("rtilde", "q_ext")

    fact: PartialFactorization
    cert: SrqrCertificate
    r22_norm_estimate: float
    rtilde: object
    q_ext: object


@dataclass
class ApproxSvd:
    u: object
    s: object
    v: object
    flop_count: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def k(self):
        return self.s.shape[0]

    def matrix(self):
        u, s, v = _np(self.u), _np(self.s), _np(self.v)
        return (u * s) @ v.T

    def error(self, A):
        return float(np.linalg.norm(_np(A) - self.matrix()))


def flip_flop_flop_formula(m, n, l, b, p):
    """Leading-order flop budget 4mnl + 2(b+p)mn (ffsrqr/svd.py:258-260)."""
    return 4 * m * n * l + 2 * (b + p) * m * n


def rsisvd_flop_formula(m, n, k, p, q):
    """Leading-order flop budget (4q+4)mn(k+p) of subspace iteration (ffsrqr/svd.py:263-265)."""
    return (4 * q + 4) * m * n * (k + p)
