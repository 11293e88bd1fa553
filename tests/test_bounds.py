"""check_theorem_bounds (ffsrqr/svd.py:174-255): the oracle restatement against
golden reports the reference produced (tests/golden/bounds/make_golden_bounds.py),
and the device version (paper_1803_01982_b200.bounds) against the same goldens
on the engine's own factorization.  Cases follow the reference's
tests/test_svd.py:80-101 and tests/test_acceptance.py:101-110.

Tolerance: tau, tau-hat, ||R22||_2, max column norm and the residual norm
within 1e-8 relative (they are built from factors that agree to ~1e-12 and
from singular values of a residual block whose entries are ~sigma_{l+1});
every boolean flag identical.
"""
import glob
import os

import numpy as np
import pytest

import oracle

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bounds")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))
FLAGS = ("aux_lower_ok", "sv_lower_ok", "sv_upper_ok", "aux_residual_ok", "residual_ok")
RTOL = 1e-8


def _load(name):
    z = np.load(os.path.join(HERE, name + ".npz"))
    return {k: z[k] for k in z.files}


def _close(a, b):
    return abs(a - b) <= RTOL * max(abs(b), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_oracle_bounds_match_reference(name):
    c = _load(name)
    A, k, l, seed = c["A"], int(c["k"]), int(c["l"]), int(c["seed"])
    ap = oracle.flip_flop(A, k, l=l, seed=seed)
    sr = ap.sr
    rep = oracle.check_theorem_bounds(A, sr.perm, sr.R, sr.Q, sr.rtilde, ap.u, ap.s, ap.v, l)
    assert rep["degenerate"] == bool(c["degenerate"])
    assert rep["all_ok"] == bool(c["all_ok"]) is True
    if rep["degenerate"]:
        return
    assert [rep[f] for f in FLAGS] == list(c["flags"])
    for key in ("tau", "tau_hat", "r22_2", "r22_12", "resid2", "g1", "g2"):
        assert _close(rep[key], float(c[key])), (key, rep[key], float(c[key]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_bounds_match_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200.bounds import check_theorem_bounds

    c = _load(name)
    A, k, l, seed = c["A"], int(c["k"]), int(c["l"]), int(c["seed"])
    for inp in (A, torch.as_tensor(A, device="cuda")):
        ap = ffb.flip_flop_srqr(inp, k, l=l, seed=seed)
        rep = check_theorem_bounds(inp, ap)
        assert rep.degenerate == bool(c["degenerate"])
        assert rep.all_ok and bool(c["all_ok"])
        if rep.degenerate:
            continue
        assert [getattr(rep, f) for f in FLAGS] == list(c["flags"])
        np.testing.assert_allclose(rep.sigma_exact, c["sigma_exact"], rtol=1e-12)
        for key in ("tau", "tau_hat"):
            assert _close(getattr(rep, key), float(c[key])), (key, getattr(rep, key))
        for key in ("r22_2", "r22_12", "resid2", "g1", "g2"):
            assert _close(rep.detail[key], float(c[key])), (key, rep.detail[key], float(c[key]))


def _gen_type1(m, n, s, seed):
    """Test-side restatement of ffsrqr/generators.py:17-28 (U D V^T + 1e-4 E,
    D geometric 1 -> 1e-3 over s planted values, Philox stream 3e6)."""
    from paper_1803_01982_b200 import rng

    rs = rng.philox(seed, rng.STREAM_GEN)
    U, _ = np.linalg.qr(rs.standard_normal((m, s)))
    V, _ = np.linalg.qr(rs.standard_normal((n, s)))
    return (U * np.geomspace(1.0, 1e-3, s)) @ V.T + 1e-4 * rs.standard_normal((m, n))


def test_gen_type1_matches_golden():
    c = _load("bounds_type1_300_s3")
    np.testing.assert_array_equal(_gen_type1(300, 300, 100, 3), c["A"])


@pytest.mark.gpu
def test_device_bound_suite_acceptance():
    """The reference's acceptance item 3 (tests/test_acceptance.py:101-110) and
    TestBounds.test_hold_on_decaying_spectrum (tests/test_svd.py:81-87): every
    bound holds, zero violations, and tau obeys the dimensional budget
    (tests/test_svd.py:89-95)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1803_01982_b200 as ffb

    violations = []
    for seed in range(20):
        A = torch.as_tensor(_gen_type1(300, 300, 100, seed), device="cuda")
        rep = ffb.check_theorem_bounds(A, ffb.flip_flop_srqr(A, 20, l=25, seed=seed), slack=1e-8)
        if not rep.all_ok:
            violations.append(seed)
    for seed in range(3):
        A = torch.as_tensor(_gen_type1(120, 120, 50, seed), device="cuda")
        rep = ffb.check_theorem_bounds(A, ffb.flip_flop_srqr(A, 10, l=15, seed=seed))
        if not (rep.all_ok and rep.tau >= 0 and rep.tau_hat >= 0):
            violations.append(("120", seed))
    assert violations == []
    A = _gen_type1(100, 100, 40, 7)
    ap = ffb.flip_flop_srqr(A, 10, l=15, seed=1)
    rep = ffb.check_theorem_bounds(A, ap)
    cert = ap.meta["srqr"].cert
    assert rep.tau <= cert.g1 * cert.g2 * np.sqrt((rep.l + 1) * (100 - rep.l)) + 1e-8
