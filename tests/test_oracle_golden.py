"""Pin the CPU oracle (oracle/ffsrqr_oracle.py) against the reference's own outputs.

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  Pivots must match exactly; factors to the
reference's own backend-to-backend spread (SURVEY.md §0.6 measured ~5e-15).
"""
import numpy as np
import pytest

import oracle
from golden_io import load, names

CASES = names()


def _rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    c = load(name)
    A = c["A"]
    prm = oracle.resolve(c["m"], c["n"], c["k"], c["l"], c["b"], c["p"], g=c["g"], d=c["d"],
                         seed=c["seed"], clamp=False)
    trq = oracle.trqrcp(A, prm)
    r = c["num_rank"]
    j0 = 0
    for i, o in enumerate(c["orders"]):
        keep = max(0, min(len(o), r - j0))
        assert np.array_equal(trq.block_orders[i][:keep], o[:keep]), f"block {i} pivots differ"
        j0 += min(c["b"], c["l"] - j0)
    try:
        sr = oracle.srqr(A, prm)
        status = "ok"
    except oracle.ffsrqr_oracle.OracleError as e:
        assert e.kind == "CertificationError"
        sr, status = e.payload, "CertificationError"
    assert status == c["srqr_status"]
    if r < c["l"]:
        # numerically rank-deficient: the factor is pinned up to the numerical rank
        assert np.array_equal(sr.perm[:r], c["perm"][:r])
        assert _rel(sr.R[:r, :r], c["R"][:r, :r]) < 1e-11
        assert sr.alpha == 0.0 and c["cert"][0] == 0.0
        return_after_cert = True
    else:
        assert np.array_equal(sr.perm, c["perm"])
        assert _rel(sr.R, c["R"]) < 1e-11
        assert _rel(sr.rtilde, c["rtilde"]) < 1e-11
        if c["q_ext"].shape[1]:
            assert np.max(np.abs(sr.Q - c["q_ext"])) < 1e-10
        return_after_cert = False
    cert = np.array([sr.alpha, sr.g1, sr.g2, sr.swaps, sr.tau_bound, sr.tau_hat_bound, sr.r22])
    assert cert[3] == c["cert"][3]
    if return_after_cert:
        np.testing.assert_allclose(cert[:6], c["cert"][:6], rtol=1e-9, atol=1e-13)
    else:
        np.testing.assert_allclose(cert, c["cert"], rtol=1e-9, atol=1e-13)
    if "s" in c:
        ff = oracle.flip_flop(A, c["k"], c["l"], c["b"], c["p"], g=c["g"], d=c["d"], seed=c["seed"])
        np.testing.assert_allclose(ff.s, c["s"], rtol=1e-12, atol=1e-14 * c["s"][0])
        np.testing.assert_allclose(ff.diag_L, c["diag_L"], rtol=1e-10, atol=1e-13 * abs(c["diag_L"][0]))
        if "u" in c:
            # columns agree up to sign
            du = np.abs(np.sum(ff.u * c["u"], axis=0))
            dv = np.abs(np.sum(ff.v * c["v"], axis=0))
            gap_ok = np.ones_like(du, dtype=bool)
            gap_ok[:-1] = np.abs(np.diff(c["s"])) > 1e-8 * c["s"][0]
            assert np.all(du[gap_ok] > 1 - 1e-9) and np.all(dv[gap_ok] > 1 - 1e-9)
        else:
            from paper_1803_01982_b200 import workloads

            w = workloads.philox(12345, 777)
            xu = w.standard_normal(c["m"])
            xv = w.standard_normal(c["n"])
            np.testing.assert_allclose(np.abs(ff.u.T @ xu), c["u_proj_abs"], rtol=1e-8, atol=1e-10)
            np.testing.assert_allclose(np.abs(ff.v.T @ xv), c["v_proj_abs"], rtol=1e-8, atol=1e-10)


def test_oracle_householder_known_answers():
    # ffsrqr tests/test_dense_core.py:22-37 known answers
    v, beta, alpha = oracle.householder(np.array([3.0, -1.0, 2.0, 0.5]))
    y = np.array([3.0, -1.0, 2.0, 0.5]) - beta * v * (v @ np.array([3.0, -1.0, 2.0, 0.5]))
    assert abs(y[0] - alpha) < 1e-14 and np.max(np.abs(y[1:])) < 1e-14
    assert alpha < 0  # opposite sign of x0
    assert oracle.householder(np.zeros(3))[1:] == (0.0, 0.0)
    assert oracle.householder(np.array([2.0, 0.0, 0.0]))[1:] == (0.0, 2.0)


def test_oracle_spec_example_pivot_swap():
    # [[0,2],[0,1]] pivots column 1 first with |R11| = sqrt(5)
    W = np.array([[0.0, 2.0], [0.0, 1.0]])
    order = oracle.qrcp_pivots(W, 2)
    assert list(order) == [1, 0]
    assert abs(abs(W[0, 0]) - np.sqrt(5.0)) < 1e-15


def test_oracle_rng_streams():
    a = oracle.gaussian(12, 30, 7, 0)
    assert np.array_equal(a, oracle.gaussian(12, 30, 7, 0))
    assert not np.allclose(a, oracle.gaussian(12, 30, 7, 1000))
