"""GPU: batched problems on several CUDA streams give bitwise the same results as
one-at-a-time (the engine is deterministic and per-thread host staging keeps
concurrent calls independent); the HOSVD caller recovers an exact Tucker tensor."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffb():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1803_01982_b200 as m
    return m


def _mat(i, m=600, n=300):
    g = np.random.default_rng(100 + i)
    U, _ = np.linalg.qr(g.standard_normal((m, n)))
    V, _ = np.linalg.qr(g.standard_normal((n, n)))
    s = np.arange(1, n + 1, dtype=float) ** -1.5
    return torch.from_numpy((U * s) @ V.T).cuda()


def test_streams_match_sequential(ffb):
    from paper_1803_01982_b200 import batch

    probs = {i: _mat(i) for i in range(6)}
    solve = lambda i: ffb.flip_flop_srqr(probs[i], 30, l=40, b=16, p=8, seed=i)
    seq = [solve(i) for i in range(6)]
    par = batch.run_streams(list(range(6)), solve, n_streams=3)
    for a, b in zip(seq, par):
        assert torch.equal(a.s, b.s)
        assert torch.equal(a.u, b.u)
        assert torch.equal(a.v, b.v)


def test_batch_driver_single_rank(ffb):
    from paper_1803_01982_b200 import batch

    probs = {i: _mat(i) for i in range(4)}
    res, got = batch.flip_flop_batch(None, 4, 30, 40, 16, 8, solve=lambda i: ffb.flip_flop_srqr(
        probs[i], 30, l=40, b=16, p=8, seed=i), gather=("s",))
    assert got["s"].shape == (4, 30)
    for i in range(4):
        assert torch.equal(got["s"][i], res[i].s)


def test_hosvd_exact_tucker(ffb):
    from paper_1803_01982_b200 import callers

    g = np.random.default_rng(7)
    G = g.standard_normal((6, 5, 4))
    Us = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in zip((40, 35, 30), (6, 5, 4))]
    X = np.einsum("abc,ia,jb,kc->ijk", G, *Us)
    core, factors, _ = callers.hosvd(X, (6, 5, 4), l_extra=2, b=4, p=3)
    for U, F in zip(Us, factors):
        F = F.cpu().numpy()
        # same column space: the projection of U onto span(F) is U itself
        assert np.linalg.norm(U - F @ (F.T @ U)) < 1e-10
    Xr = core.cpu().numpy()
    for mode, F in enumerate(factors):
        Xr = np.moveaxis(np.tensordot(F.cpu().numpy(), np.moveaxis(Xr, mode, 0), axes=1), 0, mode)
    assert np.linalg.norm(Xr - X) / np.linalg.norm(X) < 1e-12


def test_c_abi_run_batched(ffb):
    """ffb_run_batched (C ABI, one host thread per in-flight problem) matches
    one-at-a-time ffb_run bitwise."""
    import ctypes as C

    from paper_1803_01982_b200 import _capi, engine

    lib = _capi.load()
    ctx = _capi.context(0)
    n_prob, k, l, b, p = 4, 30, 40, 16, 8
    As = [_mat(i) for i in range(n_prob)]
    want = [ffb.flip_flop_srqr(As[i], k, l=l, b=b, p=p, seed=i) for i in range(n_prob)]
    items = (_capi.BatchItem * n_prob)()
    keep = []
    streams = [torch.cuda.Stream() for _ in range(n_prob)]
    for i, A in enumerate(As):
        m, n = A.shape
        Ad = A.t().contiguous().t()
        prm = _capi.Params(k, l, b, p, min(l, 10), 0.5, 2.0, i)
        nb = C.c_size_t()
        assert lib.ffb_workspace_query(m, n, C.byref(prm), _capi.FFB_MODE_FLIPFLOP, C.byref(nb)) == 0
        ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
        om = engine._omega(torch, torch.device("cuda", 0), b + p, m, i)
        s = torch.empty(k, dtype=torch.float64, device="cuda")
        u = torch.empty((k, m), dtype=torch.float64, device="cuda").t()
        v = torch.empty((k, n), dtype=torch.float64, device="cuda").t()
        perm = torch.empty(n, dtype=torch.int64, device="cuda")
        res = _capi.Result()
        res.s, res.u, res.ldu, res.v, res.ldv, res.perm = s.data_ptr(), u.data_ptr(), m, v.data_ptr(), n, perm.data_ptr()
        it = items[i]
        it.stream, it.mode, it.A, it.m, it.n, it.lda = streams[i].cuda_stream, _capi.FFB_MODE_FLIPFLOP, Ad.data_ptr(), m, n, m
        it.a_layout = _capi.FFB_LAYOUT_COL
        it.prm, it.omega, it.workspace, it.workspace_bytes = prm, om.data_ptr(), ws.data_ptr(), ws.numel()
        it.out = C.pointer(res)
        keep.append((Ad, ws, om, s, u, v, perm, res))
    torch.cuda.synchronize()
    rc = lib.ffb_run_batched(ctx, items, n_prob, 3, engine._gauss_cb, None)
    torch.cuda.synchronize()
    assert rc == 0, _capi.last_error(ctx)
    for i in range(n_prob):
        assert items[i].status == 0
        s = keep[i][3]
        assert torch.equal(s, want[i].s)
        assert torch.equal(keep[i][6], want[i].meta["srqr"].fact.perm if isinstance(want[i].meta["srqr"].fact.perm, torch.Tensor) else torch.as_tensor(want[i].meta["srqr"].fact.perm, device="cuda"))


def test_native_batch_matches_single_calls(ffb):
    """batch.NativeBatch (ffb_run_batched on C++ threads with an SM budget per
    problem, Omega regenerated on host threads, chunks of 3) gives every problem
    bitwise the single-call result: the budget changes grids, not arithmetic."""
    from paper_1803_01982_b200 import batch

    n_prob, k, l, b, p = 7, 30, 40, 16, 8
    As = [_mat(i) for i in range(n_prob)]
    want = [ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, seed=10 + i) for i, A in enumerate(As)]
    nb = batch.NativeBatch(As, k, l, b, p, seeds=[10 + i for i in range(n_prob)], threads=3)
    for rep in range(2):
        out = nb.run(fresh_omega=True, chunk=3)
        torch.cuda.synchronize()
        for i in range(n_prob):
            assert torch.equal(out[i]["s"], want[i].s)
            assert torch.equal(out[i]["u"], want[i].u) and torch.equal(out[i]["v"], want[i].v)
            assert torch.equal(out[i]["perm"], want[i].meta["srqr"].fact.perm)
            assert out[i]["g2"] == want[i].meta["srqr"].cert.g2
