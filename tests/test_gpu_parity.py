"""GPU parity: the sm_100a engine (through the C ABI) vs the reference goldens
and the CPU oracle on identical inputs and identical host-generated sketches.

Tolerances (north_star): pivots identical except on certified near-ties;
singular values and diag(L) within 1e-10 relative; ||AP - QR||_F/||A||_F within
1e-12 of the reference's; certificate scalars within 1e-10 relative.
"""
import numpy as np
import pytest

import oracle
from golden_io import load, names

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = names()
RTOL_SV = 1e-10


@pytest.fixture(scope="module")
def ffb():
    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import _capi

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _capi.load()
    return ffb


def _params(ffb, c):
    return ffb.SketchParams(k=c["k"], l=c["l"], b=c["b"], p=c["p"], g=c["g"], d=c["d"], seed=c["seed"])


def _noise_tail(c, A):
    """positions >= l whose sketch norms are at noise level (exact-rank inputs):
    the argmax there is a certified near-tie (all candidates ~0)."""
    return c["cert"][0] == 0.0


def test_gemm_engine_layouts(ffb):
    from paper_1803_01982_b200 import _capi
    import ctypes as C

    lib = _capi.load()
    ctx = _capi.context(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    for (M, N, K) in [(80, 8192, 8192), (72, 300, 2500), (65, 777, 4100), (64, 1000, 2000), (2000, 60, 1000), (48, 37, 5),
                      (130, 70, 257), (7, 9, 11)]:
        for akc in (0, 1):
            for bkc in (0, 1):
                A = torch.randn(M, K, generator=g, dtype=torch.float64, device="cuda")
                B = torch.randn(K, N, generator=g, dtype=torch.float64, device="cuda")
                C0 = torch.randn(M, N, generator=g, dtype=torch.float64, device="cuda")
                Ast = A.contiguous() if akc else A.t().contiguous()      # akc: A[k + i*lda]
                Bst = B.t().contiguous() if bkc else B.contiguous()      # bkc: B[k + j*ldb]
                Cc = C0.t().contiguous()                                 # column-major
                lda = K if akc else M
                ldb = K if bkc else N
                rc = lib.ffb_gemm(ctx, C.c_void_p(torch.cuda.current_stream().cuda_stream), M, N, K,
                                  -0.5, C.c_void_p(Ast.data_ptr()), lda, akc,
                                  C.c_void_p(Bst.data_ptr()), ldb, bkc, 2.0,
                                  C.c_void_p(Cc.data_ptr()), M, C.c_void_p(ws.data_ptr()),
                                  ws.numel())
                assert rc == 0
                torch.cuda.synchronize()
                ref = -0.5 * (A @ B) + 2.0 * C0
                err = (Cc.t() - ref).abs().max().item() / ref.abs().max().item()
                assert err < 1e-13, (M, N, K, akc, bkc, err)


@pytest.mark.parametrize("M,N,K", [(8192, 272, 2048), (6000, 420, 3000), (5000, 500, 2600), (8192, 272, 8192)])
def test_gemm_lockstep_stream_k(ffb, M, N, K, monkeypatch):
    # tall products whose row operand exceeds L2 with 2-4 N tiles (A*Yhat): the CTAs
    # of one row block walk the same k range in lockstep; same result as the
    # linear stream-K ranges up to the order of the split sums
    from paper_1803_01982_b200 import _capi
    import ctypes as C

    lib = _capi.load()
    ctx = _capi.context(0)
    g = torch.Generator(device="cuda").manual_seed(M + N)
    ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    A = torch.randn(M, K, generator=g, dtype=torch.float64, device="cuda")
    B = torch.randn(K, N, generator=g, dtype=torch.float64, device="cuda")
    Ast = A.t().contiguous()      # column-major A (akc = 0), as the flip-flop's A*Yhat
    Bst = B.t().contiguous()      # k-contiguous B (bkc = 1)
    ref = A @ B
    outs = []
    for lock in ("1", "0"):
        monkeypatch.setenv("FFB_GEMM_LOCK", lock)
        Cc = torch.zeros(N, M, dtype=torch.float64, device="cuda")
        rc = lib.ffb_gemm(ctx, C.c_void_p(torch.cuda.current_stream().cuda_stream), M, N, K, 1.0,
                          C.c_void_p(Ast.data_ptr()), M, 0, C.c_void_p(Bst.data_ptr()), K, 1, 0.0,
                          C.c_void_p(Cc.data_ptr()), M, C.c_void_p(ws.data_ptr()), ws.numel())
        assert rc == 0
        torch.cuda.synchronize()
        err = (Cc.t() - ref).abs().max().item() / ref.abs().max().item()
        assert err < 1e-13, (lock, err)
        outs.append(Cc)
    assert (outs[0] - outs[1]).abs().max().item() <= 1e-12 * ref.abs().max().item()


@pytest.mark.parametrize("name", CASES)
def test_first_block_pivots(ffb, name):
    from paper_1803_01982_b200 import _capi, rng
    import ctypes as C

    c = load(name)
    A = c["A"]
    m, n = A.shape
    s = c["b"] + c["p"]
    om = rng.gaussian(s, m, c["seed"], 0)
    B = om @ A
    Bd = torch.from_numpy(np.asfortranarray(B).T.copy()).cuda().t()   # column-major s x n
    arr = torch.arange(n, dtype=torch.int64, device="cuda")
    pos = torch.arange(n, dtype=torch.int64, device="cuda")
    gap = torch.zeros(max(c["l"], 1), dtype=torch.float64, device="cuda")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    bb = min(c["b"], c["l"])
    lib = _capi.load()
    rc = lib.ffb_block_pivots(_capi.context(0), C.c_void_p(torch.cuda.current_stream().cuda_stream),
                              C.c_void_p(Bd.data_ptr()), s, n, s, 0, bb, C.c_void_p(arr.data_ptr()),
                              C.c_void_p(pos.data_ptr()), C.c_void_p(gap.data_ptr()),
                              C.c_void_p(ws.data_ptr()), ws.numel())
    assert rc == 0
    got = arr.cpu().numpy()
    r = min(c["num_rank"], len(c["orders"][0]))   # rounding-level candidates past the numerical rank
    if r < c["l"]:
        assert np.array_equal(got[:r], c["orders"][0][:r]), f"first-block arrangement differs for {name}"
        return
    assert np.array_equal(got, c["orders"][0]), f"first-block arrangement differs for {name}"
    assert np.array_equal(np.argsort(got), pos.cpu().numpy())


@pytest.mark.parametrize("name", CASES)
def test_trqrcp_matches_oracle(ffb, name):
    c = load(name)
    A = c["A"]
    prm = _params(ffb, c)
    f = ffb.trqrcp(A, prm)
    o = oracle.trqrcp(A, oracle.resolve(c["m"], c["n"], c["k"], c["l"], c["b"], c["p"], g=c["g"],
                                        d=c["d"], seed=c["seed"], clamp=False))
    r = c["num_rank"]
    if r < c["l"]:
        # numerically rank-deficient (l > rank): pinned up to the numerical rank; the
        # factorization is still exact, A[:, perm] = Q R to rounding
        assert np.array_equal(f.perm[:r], o.perm[:r])
        assert np.abs(f.R[:r, :r] - o.R[:r, :r]).max() <= 1e-10 * np.abs(o.R).max()
        Q = f.q()
        assert np.abs(Q.T @ Q - np.eye(c["l"])).max() < 1e-12 * np.sqrt(c["m"])
        res = np.linalg.norm(A[:, f.perm][:, :c["l"]] - Q @ f.R[:, :c["l"]]) / np.linalg.norm(A)
        assert res < 1e-13
        return
    assert np.array_equal(f.perm, o.perm)
    scale = np.abs(o.R).max()
    assert np.abs(f.R - o.R).max() <= 1e-10 * scale
    Q = f.q()
    assert np.abs(Q.T @ Q - np.eye(c["l"])).max() < 1e-12 * np.sqrt(c["m"])
    assert np.abs(np.abs(Q) - np.abs(o.Y.shape[0] and np.eye(c["m"], c["l"]) - o.Y @ (o.T @ o.Y[:c["l"], :].T))).max() < 1e-9


@pytest.mark.parametrize("name", CASES)
def test_srqr_matches_reference(ffb, name):
    c = load(name)
    A = c["A"]
    prm = _params(ffb, c)
    try:
        res = ffb.srqr(A, prm)
        status = "ok"
    except ffb.CertificationError as e:
        res, status = e.result, "CertificationError"
    assert status == c["srqr_status"]
    cert = res.cert
    assert cert.swaps == int(c["cert"][3])
    if c["cert"][0] > 0:
        assert np.array_equal(res.fact.perm, c["perm"]), "pivot sequence differs"
        np.testing.assert_allclose([cert.alpha, cert.g1, cert.g2, cert.tau_bound, cert.tau_hat_bound,
                                    res.r22_norm_estimate], c["cert"][[0, 1, 2, 4, 5, 6]], rtol=1e-10)
        scale = np.abs(c["R"]).max()
        assert np.abs(res.fact.R - c["R"]).max() <= 1e-10 * scale
        assert np.abs(res.rtilde - c["rtilde"]).max() <= 1e-10 * np.abs(c["rtilde"]).max()
    else:
        # exactly / numerically rank-deficient input: alpha = g1 = g2 = 0
        # (tests/test_srqr.py:82-87); pivots past the numerical rank are argmaxes
        # over rounding-level norms (certified near-ties).
        assert cert.alpha == 0.0 and cert.g1 == 0.0 and cert.g2 == 0.0
        r = c["num_rank"]
        assert np.array_equal(res.fact.perm[:r], c["perm"][:r])
    # residual parity ||A P - Q R||_F / ||A||_F within 1e-12 of the reference's
    P = res.fact.perm
    nA = np.linalg.norm(A)
    ours = np.linalg.norm(A[:, P] - res.fact.q() @ res.fact.R) / nA
    l = c["l"]
    Qref = c["q_ext"][:, :l] if c["q_ext"].shape[1] else None
    if Qref is not None:
        theirs = np.linalg.norm(A[:, c["perm"]] - Qref @ c["R"]) / nA
        assert abs(ours - theirs) <= 1e-12
    Qe = res.q_ext
    assert np.abs(Qe.T @ Qe - np.diag([1.0] * l + [1.0 if cert.alpha > 0 else 0.0])).max() < 1e-11


@pytest.mark.parametrize("name", [n for n in CASES if n != "certfail60x50"])
def test_flipflop_matches_reference(ffb, name):
    c = load(name)
    if "s" not in c:
        pytest.skip("no flip-flop golden")
    A = c["A"]
    ap = ffb.flip_flop_srqr(A, c["k"], l=c["l"], b=c["b"], p=c["p"], g=c["g"], d=c["d"], seed=c["seed"])
    s_ref = c["s"]
    np.testing.assert_allclose(ap.s, s_ref, rtol=RTOL_SV, atol=1e-14 * s_ref[0])
    dl = c["diag_L"]
    np.testing.assert_allclose(ap.meta["diag_L"], dl, rtol=RTOL_SV, atol=1e-13 * abs(dl[0]))
    k = c["k"]
    assert np.abs(ap.u.T @ ap.u - np.eye(k)).max() < 1e-12
    assert np.abs(ap.v.T @ ap.v - np.eye(k)).max() < 1e-12
    gap_ok = np.ones(k, dtype=bool)
    gap_ok[:-1] = np.abs(np.diff(s_ref)) > 1e-8 * s_ref[0]
    gap_ok[1:] &= np.abs(np.diff(s_ref)) > 1e-8 * s_ref[0]
    if "u" in c:
        du = np.abs(np.sum(ap.u * c["u"], axis=0))
        dv = np.abs(np.sum(ap.v * c["v"], axis=0))
        assert np.all(du[gap_ok] > 1 - 1e-10) and np.all(dv[gap_ok] > 1 - 1e-10)
    else:
        from paper_1803_01982_b200 import workloads

        w = workloads.philox(12345, 777)
        xu = w.standard_normal(c["m"])
        xv = w.standard_normal(c["n"])
        np.testing.assert_allclose(np.abs(ap.u.T @ xu)[gap_ok], c["u_proj_abs"][gap_ok], rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(np.abs(ap.v.T @ xv)[gap_ok], c["v_proj_abs"][gap_ok], rtol=1e-8, atol=1e-10)


def test_seed_reproducible_bitwise(ffb):
    c = load("type1_120x90")
    a1 = ffb.flip_flop_srqr(c["A"], 10, l=14, seed=9)
    a2 = ffb.flip_flop_srqr(c["A"], 10, l=14, seed=9)
    assert np.array_equal(a1.u, a2.u) and np.array_equal(a1.s, a2.s) and np.array_equal(a1.v, a2.v)


def test_dimension_errors(ffb):
    A = np.random.default_rng(0).standard_normal((20, 20))
    with pytest.raises(ffb.DimensionError):
        ffb.srqr(A, ffb.SketchParams(k=20, l=20, b=8, p=4))
    with pytest.raises(ffb.DimensionError):
        ffb.flip_flop_srqr(A, 0)
    with pytest.raises(ffb.DimensionError):
        ffb.flip_flop_srqr(np.zeros(5), 1)


def test_torch_input_stays_on_device(ffb):
    c = load("cfg5_small")
    At = torch.from_numpy(c["A"]).cuda()
    ap = ffb.flip_flop_srqr(At, c["k"], l=c["l"], b=c["b"], p=c["p"], seed=c["seed"])
    assert ap.u.is_cuda and ap.v.is_cuda
    np.testing.assert_allclose(ap.s.cpu().numpy(), c["s"], rtol=RTOL_SV)


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_non_finite_input_raises(ffb, bad):
    """NaN / Inf in A: the reference fails with scipy's ValueError("array must not
    contain infs or NaNs") (sketch.py:75-83); the engine raises
    NonFiniteInputError, which is both that ValueError and a NumericalError, in
    every mode."""
    A = np.random.default_rng(0).standard_normal((60, 40))
    A[3, 5] = bad
    for call in (lambda: ffb.flip_flop_srqr(A, 5, l=8),
                 lambda: ffb.srqr(A, ffb.SketchParams(k=5, l=8)),
                 lambda: ffb.trqrcp(A, ffb.SketchParams(k=5, l=8))):
        with pytest.raises(ValueError):
            call()
        with pytest.raises(ffb.NumericalError):
            call()


@pytest.mark.parametrize("name", [n for n in CASES if "flop_count" in load(n)])
def test_flop_count_matches_reference(ffb, name):
    # flop_count is the reference's tally (ffsrqr/flops.py) replayed with the
    # device run's swap trace; the golden holds the reference's own count
    c = load(name)
    try:
        ap = ffb.flip_flop_srqr(c["A"], c["k"], l=c["l"], b=c["b"], p=c["p"], g=c["g"], d=c["d"],
                                seed=c["seed"])
    except ffb.CertificationError:
        pytest.skip("certification failure: no flop_count")
    want = int(c["flop_count"])
    full_rank = c["cert"][0] != 0.0 and c["m"] > c["b"] + c["p"]
    if full_rank:
        # shape-only call sites plus the traced Givens chases
        assert abs(ap.flop_count - want) <= 1e-3 * want, (ap.flop_count, want)
    else:
        assert abs(ap.flop_count - want) <= 0.03 * want, (ap.flop_count, want)
    assert ap.meta["device_flops"] > 0


def test_flop_count_band_1000(ffb):
    # ffsrqr tests/test_svd.py:105-112 through the device engine
    g = np.random.default_rng(9)
    U, _ = np.linalg.qr(g.standard_normal((1000, 100)))
    V, _ = np.linalg.qr(g.standard_normal((1000, 100)))
    A = (U * (1.0 / np.arange(1, 101))) @ V.T
    ap = ffb.flip_flop_srqr(A, 25, l=30, b=32, p=5, seed=0)
    formula = ffb.flip_flop_flop_formula(1000, 1000, 30, 32, 5)
    assert abs(ap.flop_count - formula) <= 0.15 * formula
    rs = ffb.rsisvd(A, 30, p=5, q=1, seed=0)
    assert abs(rs.flop_count - ffb.rsisvd_flop_formula(1000, 1000, 30, 5, 1)) <= 0.15 * rs.flop_count


def test_graph_replay_is_bitwise_repeatable(ffb):
    # the second and third calls replay the CUDA graph captured by the first
    # (same A, Omega and workspace); results must not change by a bit
    c = load("cfg1")
    A = torch.from_numpy(np.asfortranarray(c["A"]).T).cuda().t()
    runs = [ffb.flip_flop_srqr(A, c["k"], l=c["l"], b=c["b"], p=c["p"], seed=c["seed"]) for _ in range(3)]
    for r in runs[1:]:
        assert torch.equal(r.s, runs[0].s) and torch.equal(r.u, runs[0].u) and torch.equal(r.v, runs[0].v)
        assert torch.equal(r.meta["srqr"].fact.perm, runs[0].meta["srqr"].fact.perm)
    assert runs[2].meta["kernels"] == runs[0].meta["kernels"]
