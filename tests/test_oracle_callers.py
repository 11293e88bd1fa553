"""The callers' CPU oracle (oracle/callers_oracle.py) against fixtures produced
by the reference itself (tests/golden/callers/make_golden_callers.py):
RSISVD (svd.py:101-133), HOSVD / ST-HOSVD (tensor.py:104-145) and IALM RPCA /
matrix completion (nuclear.py:105-191)."""
import numpy as np
import pytest

from callers_io import cols_match_up_to_sign, load, names, tucker_reconstruct
from oracle import callers_oracle as co


@pytest.mark.parametrize("name", names("rsisvd_"))
def test_rsisvd_oracle_matches_reference(name):
    c = load(name)
    ap = co.rsisvd(c["A"], c["k"], p=c["p"], q=c["q"], seed=c["seed"])
    np.testing.assert_allclose(ap.s, c["s"], rtol=1e-12)
    assert cols_match_up_to_sign(ap.u, c["u"], 1e-10)
    assert cols_match_up_to_sign(ap.v, c["v"], 1e-10)


@pytest.mark.parametrize("name", names("hosvd_") + names("sthosvd_"))
def test_tucker_oracle_matches_reference(name):
    c = load(name)
    eng = name.split("_")[1]
    fn = co.hosvd if name.startswith("hosvd") else co.st_hosvd
    d = fn(c["X"], tuple(int(r) for r in c["ranks"]), engine=eng, seed=c["seed"])
    ref_f = [c["f0"], c["f1"], c["f2"]]
    for U, R in zip(d.factors, ref_f):
        assert cols_match_up_to_sign(U, R, 1e-10)
    Xr = tucker_reconstruct(d.core, d.factors)
    Xref = tucker_reconstruct(c["core"], ref_f)
    assert np.abs(Xr - Xref).max() <= 1e-10 * np.abs(Xref).max()
    np.testing.assert_allclose(np.abs(d.core), np.abs(c["core"]), atol=1e-10 * np.abs(c["core"]).max())


@pytest.mark.parametrize("name", names("ialm_"))
def test_ialm_oracle_matches_reference(name):
    c = load(name)
    prm = dict(svd_engine=c["engine"], max_iter=c["max_iter"], seed=c["seed"])
    if "_mc_" in name:
        st = co.ialm_mc(c["M"], c["mask"], prm)
    else:
        st = co.ialm_rpca(c["M"], prm)
    assert st.iterations == c["iterations"] and st.rank == c["rank"]
    assert list(st.ranks) == list(c["ranks"])
    np.testing.assert_allclose(st.residuals, c["residuals"], rtol=1e-6)
    scale = np.abs(c["low_rank"]).max()
    assert np.abs(st.low_rank - c["low_rank"]).max() <= 1e-8 * scale
    assert np.abs(st.sparse - c["sparse"]).max() <= 1e-8 * scale
