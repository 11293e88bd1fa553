"""flop_count parity: the closed-form replay of the reference's counter
(paper_1803_01982_b200/flops.py) against the counts the reference itself
recorded in the golden fixtures, and the reference's own 15 % band test
(ffsrqr tests/test_svd.py:105-119)."""
import numpy as np
import pytest

from golden_io import load, names
from paper_1803_01982_b200 import flip_flop_flop_formula, flops, rsisvd_flop_formula


def _case_params(c):
    m, n, b, p = c["m"], c["n"], c["b"], c["p"]
    if b + p > m:                                   # svd.py:53-55
        b = max(1, m - p)
        p = m - b
    return m, n, c["k"], c["l"], b, p, c["d"]


@pytest.mark.parametrize("name", [n for n in names() if "flop_count" in load(n)])
def test_count_matches_reference_tally(name):
    c = load(name)
    cert = c["cert"]
    swaps, alpha_zero = int(cert[3]), cert[0] == 0.0
    got = flops.flip_flop_count(*_case_params(c), swaps, (), alpha_zero)
    want = int(c["flop_count"])
    if swaps == 0 and not alpha_zero and c["m"] > c["b"] + c["p"]:
        # no swap, full rank, no clamp: every reference call site is shape-only
        assert got == want
    else:
        # Givens chases start at the traced i_off (not stored in these
        # fixtures), norm recomputations and zero-tail reflectors are data
        assert abs(got - want) <= 0.03 * want


def test_flip_flop_counter_near_formula():
    # ffsrqr tests/test_svd.py:105-112 at the same 1000 x 1000, k=25, l=30, b=32, p=5
    got = flops.flip_flop_count(1000, 1000, 25, 30, 32, 5, 10)
    formula = flip_flop_flop_formula(1000, 1000, 30, 32, 5)
    assert abs(got - formula) <= 0.15 * formula


def test_rsisvd_counter_near_formula():
    # ffsrqr tests/test_svd.py:114-119
    got = flops.rsisvd_count(1000, 1000, 30, 35, 1)
    formula = rsisvd_flop_formula(1000, 1000, 30, 5, 1)
    assert abs(got - formula) <= 0.15 * formula


@pytest.mark.parametrize("cfg,ratio", [("cfg1", 1.21), ("cfg2", 1.16), ("cfg3", 1.28), ("cfg5", 1.26)])
def test_counter_ratio_at_baseline_configs(cfg, ratio):
    # counted / formula measured on the reference at each config
    from paper_1803_01982_b200 import workloads
    w = workloads.CONFIGS[cfg]
    got = flops.flip_flop_count(w.m, w.n, w.k, w.l, w.b, w.p, min(w.l, 10))
    assert abs(got / flip_flop_flop_formula(w.m, w.n, w.l, w.b, w.p) - ratio) < 0.01
