"""CPU oracle for the Flip-Flop SRQR hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU reference.  The product (``paper_1803_01982_b200``) never imports
it and has no CPU fallback.

Pinning: ``ffsrqr_oracle`` restates the reference algorithm
(``/root/reference/pkg/src/ffsrqr``); it is pinned against golden vectors
produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``), checked by
``tests/test_oracle_golden.py``.
"""

from .ffsrqr_oracle import (  # noqa: F401
    OracleApprox,
    OracleSrqr,
    OracleTrqrcp,
    check_theorem_bounds,
    flip_flop,
    flip_flop_flops,
    gaussian,
    householder,
    qrcp_pivots,
    qrnp_inplace,
    resolve,
    srqr,
    trqrcp,
)
from . import callers_oracle  # noqa: E402,F401  (RSISVD, HOSVD/ST-HOSVD, IALM restatements)
