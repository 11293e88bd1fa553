"""A-posteriori quality check of a flip-flop result (ffsrqr/svd.py:146-255).

``check_theorem_bounds(A, approx, slack=1e-8)`` recomputes tau and tau-hat
exactly from the factorization and checks the five inequalities the
reference checks: two singular-value lower bounds, the upper bound and two
rank-k residual bounds.  It runs on the device: A, the factors and the
residual blocks stay in HBM, and the exact singular values come from
``torch.linalg.svdvals`` (cuSOLVER) as the reference takes them from LAPACK
(svd.py:188, 205, 233).  It is a verification routine, not the hot path.

One documented difference: the reference's ``flip_flop_srqr`` overwrites
``meta["srqr"].fact.R`` in place with its partial-LQ workspace (svd.py:67-68,
``np.asfortranarray(R.T)`` is a view), so its check reads a clobbered R.
Here ``fact.R`` is the true SRQR R, so M = AP - QR is the real residual
block of Theorem 4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import EngineUnavailable


@dataclass
class BoundReport:
    """Same fields as the reference's BoundReport (svd.py:152-171)."""

    k: int
    l: int
    tau: float
    tau_hat: float
    sigma_exact: np.ndarray
    sigma_approx: np.ndarray
    aux_lower_ok: bool
    sv_lower_ok: bool
    sv_upper_ok: bool
    aux_residual_ok: bool
    residual_ok: bool
    degenerate: bool
    detail: dict = field(default_factory=dict)

    @property
    def all_ok(self):
        return (self.aux_lower_ok and self.sv_lower_ok and self.sv_upper_ok
                and self.aux_residual_ok and self.residual_ok)


def _dev(torch, x, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64)
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=device)


def _max_row_norm_of_inverse(torch, T):
    """Largest row 2-norm of T^-1 for upper-triangular T (svd.py:146-149)."""
    eye = torch.eye(T.shape[0], dtype=T.dtype, device=T.device)
    inv = torch.linalg.solve_triangular(T, eye, upper=True)
    return float(torch.sqrt(torch.max(torch.sum(inv * inv, dim=1))))


def check_theorem_bounds(A, approx, slack=1e-8, device=None):
    """Verify the spectrum-revealing guarantees of ``approx`` on A
    (ffsrqr/svd.py:174-255).  Returns a ``BoundReport``."""
    import torch

    if device is None:
        device = A.device if isinstance(A, torch.Tensor) and A.is_cuda else "cuda"
    if not torch.cuda.is_available():
        raise EngineUnavailable("check_theorem_bounds runs on the device; no CUDA device")
    Ad = _dev(torch, A, device)
    m, n = Ad.shape
    res = approx.meta["srqr"]
    sk_t = _dev(torch, approx.s, device)
    k = int(sk_t.shape[0])
    l = int(res.fact.k)

    sig_t = torch.linalg.svdvals(Ad)
    sig = sig_t.cpu().numpy()
    sk = sk_t.cpu().numpy()
    sig_l1 = float(sig[l]) if l < sig.size else 0.0
    sig_k1 = float(sig[k]) if k < sig.size else 0.0

    rtilde = _dev(torch, res.rtilde, device)
    alpha_ext = abs(float(rtilde[l, l]))
    if sig_l1 <= 1e-12 * max(float(sig[0]), 1e-300) or alpha_ext == 0.0:
        ok = np.all(sk <= sig[:k] * (1 + slack))
        return BoundReport(k=k, l=l, tau=0.0, tau_hat=0.0, sigma_exact=sig[:k].copy(),
                           sigma_approx=sk.copy(), aux_lower_ok=True, sv_lower_ok=True,
                           sv_upper_ok=bool(ok), aux_residual_ok=True, residual_ok=True,
                           degenerate=True)

    perm = torch.as_tensor(np.asarray(res.fact.perm) if not isinstance(res.fact.perm, torch.Tensor)
                           else res.fact.perm, device=device).long()
    R = _dev(torch, res.fact.R, device)[:l]
    Q = _dev(torch, res.fact.q(), device)[:, :l]
    M = Ad[:, perm] - Q @ R
    r22_2 = float(torch.linalg.svdvals(M)[0])
    r22_12 = math.sqrt(float(torch.max(torch.sum(M * M, dim=0))))
    alpha = alpha_ext

    inv_rt = _max_row_norm_of_inverse(torch, rtilde)
    inv_r11 = _max_row_norm_of_inverse(torch, R[:l, :l])
    g1 = r22_12 / alpha
    g2 = alpha * inv_rt
    sig_k_hat = float(sk[k - 1])

    tau = g1 * g2 * (r22_2 / r22_12) * (1.0 / inv_rt) / sig_l1
    tau_hat = g1 * g2 * (r22_2 / r22_12) * (1.0 / inv_r11) / sig_k_hat

    up, dn = 1 + slack, 1 - slack
    upper = bool(np.all(sk <= sig[:k] * up))
    aux_denom = np.power(1.0 + 2.0 * r22_2 ** 4 / sk ** 4, 0.25)
    aux_lower = bool(np.all(sk >= sig[:k] / aux_denom * dn))
    cap = np.minimum(2.0 * tau_hat ** 4,
                     tau ** 4 * (2.0 + 4.0 * tau_hat ** 4) * (sig_l1 / sig[:k]) ** 4)
    lower = bool(np.all(sk >= sig[:k] / np.power(1.0 + cap, 0.25) * dn))

    u = _dev(torch, approx.u, device)
    v = _dev(torch, approx.v, device)
    resid2 = float(torch.linalg.svdvals(Ad - (u * sk_t) @ v.T)[0])
    aux_budget = sig_k1 * (1.0 + 2.0 * (r22_2 / sig_k1) ** 4) ** 0.25 if sig_k1 > 0 else resid2
    budget2 = sig_k1 * (1.0 + 2.0 * tau ** 4 * (sig_l1 / sig_k1) ** 4) ** 0.25 \
        if sig_k1 > 0 else resid2

    return BoundReport(
        k=k, l=l, tau=tau, tau_hat=tau_hat, sigma_exact=sig[:k].copy(), sigma_approx=sk.copy(),
        aux_lower_ok=aux_lower, sv_lower_ok=lower, sv_upper_ok=upper,
        aux_residual_ok=bool(resid2 <= aux_budget * up), residual_ok=bool(resid2 <= budget2 * up),
        degenerate=False,
        detail={"g1": g1, "g2": g2, "r22_2": r22_2, "r22_12": r22_12, "sigma_l1": sig_l1,
                "resid2": resid2, "aux_budget": aux_budget, "budget2": budget2})
