"""GPU parity of the callers around the hot path: RSISVD
(svd.py:101-133), Tucker HOSVD / ST-HOSVD with device n-mode products
(tensor.py:21-152) and the IALM solvers with the fused SVT update
(nuclear.py:91-191) — against fixtures produced by the reference itself
(tests/golden/callers/) and the CPU oracle on the same inputs.

Tolerances: singular values 1e-10 relative; singular vectors / Tucker factors
equal up to column sign to 1 - |cos| <= 1e-10; IALM iterates 1e-8 of the
iterate's scale (the iteration re-amplifies rounding of the partial SVD)."""
import numpy as np
import pytest

from callers_io import cols_match_up_to_sign, load, names, tucker_reconstruct
from oracle import callers_oracle as co

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ffb():
    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import _capi

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _capi.load()
    return ffb


@pytest.mark.parametrize("name", names("rsisvd_"))
def test_rsisvd_matches_reference(ffb, name):
    c = load(name)
    ap = ffb.rsisvd(c["A"], c["k"], p=c["p"], q=c["q"], seed=c["seed"])
    np.testing.assert_allclose(ap.s, c["s"], rtol=1e-10)
    assert cols_match_up_to_sign(ap.u, c["u"], 1e-10)
    assert cols_match_up_to_sign(ap.v, c["v"], 1e-10)
    assert ap.meta["method"] == "rsisvd" and ap.flop_count > 0


def test_rsisvd_device_input_matches_oracle(ffb):
    from paper_1803_01982_b200 import workloads

    A = workloads.numpy_matrix("cfg5", seed=4, m=1024, n=512)
    ref = co.rsisvd(A, 64, p=16, q=2, seed=5)
    Ad = torch.from_numpy(A).cuda()
    ap = ffb.rsisvd(Ad, 64, p=16, q=2, seed=5)
    assert ap.u.is_cuda and ap.v.is_cuda
    np.testing.assert_allclose(ap.s.cpu().numpy(), ref.s, rtol=1e-10)
    assert cols_match_up_to_sign(ap.u.cpu().numpy(), ref.u, 1e-10)
    assert cols_match_up_to_sign(ap.v.cpu().numpy(), ref.v, 1e-10)


def test_rsisvd_errors(ffb):
    A = np.random.default_rng(0).standard_normal((30, 20))
    with pytest.raises(ffb.DimensionError):
        ffb.rsisvd(A, 0)
    with pytest.raises(ffb.DimensionError):
        ffb.rsisvd(A, 5, q=-1)


def test_unfold_fold_nmode_product_match_numpy(ffb):
    from paper_1803_01982_b200 import tensor as T

    g = np.random.default_rng(3)
    X = np.asfortranarray(g.standard_normal((7, 5, 6, 4)))
    Xd = T.to_device(X)
    for mode in range(4):
        M = co.unfold(X, mode)
        Md = T.unfold(Xd, mode)
        np.testing.assert_array_equal(Md.cpu().numpy(), M)
        np.testing.assert_array_equal(T.fold(Md, mode, X.shape).cpu().numpy(), X)
        U = g.standard_normal((3, X.shape[mode]))
        ref = co.nmode_product(X, U, mode)
        got = T.nmode_product(Xd, torch.from_numpy(U).cuda(), mode).cpu().numpy()
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("name", names("hosvd_") + names("sthosvd_"))
def test_tucker_matches_reference(ffb, name):
    from paper_1803_01982_b200 import tensor as T

    c = load(name)
    eng = name.split("_")[1]
    fn = T.hosvd if name.startswith("hosvd") else T.st_hosvd
    d = fn(c["X"], tuple(int(r) for r in c["ranks"]), engine=eng, seed=c["seed"])
    ref_f = [c["f0"], c["f1"], c["f2"]]
    for U, R in zip(d.factors, ref_f):
        assert cols_match_up_to_sign(U, R, 1e-10)
    Xr = tucker_reconstruct(d.core, d.factors)
    Xref = tucker_reconstruct(c["core"], ref_f)
    assert np.abs(Xr - Xref).max() <= 1e-10 * np.abs(Xref).max()
    np.testing.assert_allclose(np.abs(d.core), np.abs(c["core"]), atol=1e-10 * np.abs(c["core"]).max())
    if name.startswith("sthosvd"):
        assert list(d.meta["order"]) == list(c["order"])
    err = T.tucker_error(c["X"], d)
    err_ref = np.linalg.norm(c["X"] - Xref) / np.linalg.norm(c["X"])    # tensor.py:146-152
    assert abs(err - err_ref) <= 1e-10 * max(err_ref, 1e-300) + 1e-14


def test_hosvd_exact_engine_matches_numpy(ffb):
    from paper_1803_01982_b200 import tensor as T

    c = load("hosvd_flipflop")
    d = T.hosvd(c["X"], (5, 4, 3), engine="exact")
    ref = co.hosvd(c["X"], (5, 4, 3), engine="exact")
    for U, R in zip(d.factors, ref.factors):
        assert cols_match_up_to_sign(U, R, 1e-10)


@pytest.mark.parametrize("name", names("ialm_"))
def test_ialm_matches_reference(ffb, name):
    from paper_1803_01982_b200 import nuclear as N

    c = load(name)
    prm = N.IalmParams(svd_engine=c["engine"], max_iter=c["max_iter"], seed=c["seed"])
    if "_mc_" in name:
        st = N.ialm_mc(c["M"], c["mask"], prm)
    else:
        st = N.ialm_rpca(c["M"], prm)
    assert st.iterations == c["iterations"] and st.rank == c["rank"]
    assert list(st.ranks) == list(c["ranks"])
    # late residuals are tiny and re-amplify rounding of every earlier partial SVD:
    # relative 1e-6 plus 1e-8 of the first residual
    res_ref = np.asarray(c["residuals"])
    assert np.all(np.abs(np.asarray(st.residuals) - res_ref) <= 1e-6 * res_ref + 1e-8 * res_ref[0])
    np.testing.assert_allclose(st.mus, c["mus"], rtol=1e-10)
    scale = np.abs(c["low_rank"]).max()
    assert np.abs(st.low_rank - c["low_rank"]).max() <= 1e-8 * scale
    assert np.abs(st.sparse - c["sparse"]).max() <= 1e-8 * scale


@pytest.mark.parametrize("mode", [0, 1])
def test_fused_ialm_update_matches_torch_fp64(ffb, mode):
    """ffb_ialm_update vs the reference's elementwise formulas in torch fp64."""
    import ctypes as C

    from paper_1803_01982_b200 import _capi

    g = torch.Generator(device="cuda").manual_seed(11)
    m, n = 777, 301
    M, X, Y0 = (torch.randn(m * n, generator=g, dtype=torch.float64, device="cuda") for _ in range(3))
    mask = (torch.rand(m * n, generator=g, device="cuda") < 0.4).to(torch.uint8)
    mu, thresh, mu_next = 0.37, 0.21, 0.555
    Y = Y0.clone()
    E = torch.empty_like(M)
    W = torch.empty_like(M)
    lib = _capi.load()
    part = torch.empty(lib.ffb_svt_partials(), dtype=torch.float64, device="cuda")
    zsq = torch.empty(1, dtype=torch.float64, device="cuda")
    rc = lib.ffb_ialm_update(C.c_void_p(torch.cuda.current_stream().cuda_stream), mode,
                             C.c_void_p(M.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()),
                             C.c_void_p(E.data_ptr()), C.c_void_p(mask.data_ptr()), m * n, mu, thresh,
                             mu_next, C.c_void_p(W.data_ptr()), C.c_void_p(part.data_ptr()),
                             C.c_void_p(zsq.data_ptr()))
    assert rc == 0
    a = M - X + Y0 / mu
    E_ref = torch.sign(a) * torch.clamp(a.abs() - thresh, min=0.0) if mode == 0 else \
        torch.where(mask.bool(), torch.zeros_like(a), a)
    Z = M - X - E_ref
    Y_ref = Y0 + mu * Z
    W_ref = M - E_ref + Y_ref / mu_next
    # a few roundings of O(|M| + |X| + |Y|/mu) terms
    scale = float(M.abs().max() + X.abs().max() + Y0.abs().max() / mu) * (1 + mu / mu_next)
    for got, ref in ((E, E_ref), (Y, Y_ref), (W, W_ref)):
        assert float((got - ref).abs().max()) <= 8 * 2.0 ** -52 * scale
    assert abs(float(zsq[0]) - float((Z * Z).sum())) <= 1e-12 * float((Z * Z).sum())
