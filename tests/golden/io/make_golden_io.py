"""DMAT / DTEN fixtures written by the REFERENCE's own writers (ffsrqr/io.py:27-58),
build container only:  python tests/golden/io/make_golden_io.py"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from ffsrqr import io  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rs = np.random.default_rng(99)
A = rs.standard_normal((37, 23))
X = rs.standard_normal((5, 4, 3))
io.write_dmat(os.path.join(HERE, "a37x23.dmat"), A)
io.write_dten(os.path.join(HERE, "x5x4x3.dten"), X)
np.savez_compressed(os.path.join(HERE, "expected.npz"), A=A, X=X)
