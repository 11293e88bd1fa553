"""The reference's flop accounting, restated in closed form.

The reference tallies multiply-adds in a thread-local counter as its numpy /
numba kernels run (ffsrqr/flops.py:17-54); ``ApproxSvd.flop_count`` is that
tally.  The device engine runs different algorithms (CholeskyQR panels, a
Jacobi SVD, DMMA GEMMs), so the flops it executes are not the reference's
number.  For a drop-in ``flop_count`` this module replays the reference's
``flops.add`` / ``flops.mm`` call sites with the shapes of the run.  Every
term is a function of (m, n, k, l, b, p, d) and of the swap trace, except two
data-dependent corrections the counter also sees and this restatement leaves
out: the norm recomputations inside ``qrcp_core`` (2(s-j-1) flops each,
``_kernels_numba.py:87-92``) and reflectors whose tail is exactly zero
(``_kernels_numba.py:60-61,110-112``).  Both are O(s) or O(n) per event
against O(mnl) in total.

The device-executed flops stay available as ``meta["device_flops"]``.
"""
from __future__ import annotations


def _qrcp_core(m, n, k):
    """qrcp_core(A m x n, k) without recomputations (_kernels_numba.py:15-94)."""
    fl = 2 * m * n
    for j in range(k):
        fl += 2 * (m - j)
        if j + 1 < m:                      # non-empty reflector tail
            fl += 4 * (m - j) * (n - j - 1)
        fl += 2 * (n - j - 1)
    return fl


def _qrnp_core(m, n, k):
    """qrnp_core(A m x n, k) (_kernels_numba.py:97-131)."""
    fl = 0
    for j in range(k):
        fl += 2 * (m - j)
        if j + 1 < m:
            fl += 4 * (m - j) * (n - j - 1)
    return fl


def trqrcp_count(m, n, l, b, p):
    """_trqrcp_state (sketch.py:101-147)."""
    s = b + p
    fl = 2 * s * m * n                                        # sketch.py:109
    j0 = 0
    while j0 < l:
        bb = min(l - j0, b)
        fl += _qrcp_core(s, n - j0, bb)                       # sketch.py:62-67
        for c in range(j0, j0 + bb):
            fl += 2 * m * c                                   # sketch.py:125
            fl += 2 * (m - c) * c + 2 * c * c                 # :133
            fl += 2 * (m - c) * n + 2 * c * n                 # :136
            fl += 2 * (c + 1) * (n - c)                       # :139
        e = j0 + bb
        if e < n:
            fl += bb * bb * (n - e)                           # _tri_solve, :78
            fl += 2 * s * bb * (n - e)                        # :144
        j0 = e
    return fl


def srqr_count(m, n, l, b, p, d, swaps=0, i_offs=(), alpha_zero=False):
    """srqr (srqr.py:174-210): TRQRCP, the swap state, extensions, g2 tests,
    Givens re-triangularisations.  ``i_offs`` lists the offending column of each
    swap (missing entries count a full chase from column 0); ``alpha_zero`` is a
    final extension that found an exactly rank-l trailing block."""
    fl = trqrcp_count(m, n, l, b, p)
    fl += 2 * m * l * l                                       # srqr.py:94
    n_ext = 1 + swaps
    for i in range(n_ext):
        fl += 8 * m * l                                       # srqr.py:128
        last = i == n_ext - 1
        if not (last and alpha_zero) and l + 1 < n:
            fl += 2 * m * (n - l - 1)                         # srqr.py:140
    n_g2 = swaps + (0 if alpha_zero else 1)
    fl += n_g2 * d * (l + 1) * (l + 1)                        # srqr.py:61
    for sw in range(swaps):
        i_off = i_offs[sw] if sw < len(i_offs) else 0
        for i in range(i_off, min(l, n)):                     # qr.py:196-208
            fl += 6 * (n - i)
    return fl


def flip_flop_count(m, n, k, l, b, p, d, swaps=0, i_offs=(), alpha_zero=False):
    """flip_flop_srqr (svd.py:43-98) as the reference's counter tallies it."""
    fl = srqr_count(m, n, l, b, p, d, swaps, i_offs, alpha_zero)
    fl += _qrnp_core(n, l, l)                                 # svd.py:67-69
    fl += 2 * m * n * l                                       # svd.py:75
    fl += 2 * m * l * l                                       # svd.py:76
    fl += 2 * l * l * l                                       # svd.py:77
    fl += 6 * m * l * min(m, l) if m >= l else 6 * l * m * m  # count_svd, svd.py:80
    fl += 2 * l * n * k                                       # apply_left, qr.py:80
    fl += 4 * n * l * k                                       # svd.py:88
    return fl


def count_qr_thin(rows, cols, form_q=True):
    """flops.count_qr_thin (flops.py:41-46)."""
    c = 2 * rows * cols ** 2 - (2 * cols ** 3) // 3
    if form_q:
        c += rows * cols ** 2 + cols ** 3 // 3
    return c


def count_svd(rows, cols):
    """flops.count_svd (flops.py:49-52)."""
    small = min(rows, cols)
    return 6 * rows * cols * small if rows >= cols else 6 * cols * rows * small


def rsisvd_count(m, n, k, r, q):
    """rsisvd (svd.py:101-133)."""
    fl = 2 * m * n * r                                        # svd.py:113
    fl += count_qr_thin(m, r)
    for _ in range(q):
        fl += 2 * n * m * r + count_qr_thin(n, r)             # svd.py:117-119
        fl += 2 * m * n * r + count_qr_thin(m, r)             # svd.py:120-122
    fl += 2 * r * m * n                                       # svd.py:123
    fl += count_svd(r, n)                                     # svd.py:125
    fl += 2 * m * r * k                                       # svd.py:126
    return fl
