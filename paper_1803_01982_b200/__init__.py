"""B200-native Flip-Flop SRQR engine (arXiv:1803.01982 hot path, sm_100a).

Drop-in for the reference ``ffsrqr`` hot path: ``flip_flop_srqr``, ``srqr``,
``trqrcp`` and their result types, plus caller seams for HOSVD and the SVT
(IALM) solvers.  Compute runs in hand-written CUDA (libffb200.so, C ABI in
include/ffb200.h); this package is host glue only and has no CPU fallback.
"""
import os as _os

# Batches run one problem per stream on up to 16 host threads (batch.NativeBatch);
# CUDA's default of 8 hardware work queues makes streams beyond the 8th share a
# queue and serialise behind each other's cooperative kernels (cfg5, 16 threads:
# 499 -> 938 factorizations/s with 32 queues).  Only effective when set before
# the CUDA context exists; a caller's own setting wins.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .errors import (CertificationError, DimensionError, EngineUnavailable, NonFiniteInputError,
                     NumericalError, SingularTrailingBlockError)
from .results import (ApproxSvd, PartialFactorization, SketchParams, SrqrCertificate, SrqrResult,
                      WYFactor, flip_flop_flop_formula, rsisvd_flop_formula)
from .engine import flip_flop_srqr, rsisvd, srqr, trqrcp
from .bounds import BoundReport, check_theorem_bounds

__version__ = "0.1.0"

__all__ = [
    "ApproxSvd", "BoundReport", "CertificationError", "DimensionError", "EngineUnavailable", "NonFiniteInputError",
    "NumericalError",
    "PartialFactorization", "SingularTrailingBlockError", "SketchParams", "SrqrCertificate",
    "SrqrResult", "WYFactor", "check_theorem_bounds", "flip_flop_flop_formula", "flip_flop_srqr", "rsisvd", "srqr",
    "trqrcp", "rsisvd_flop_formula",
]
