"""numpy inputs above the staging threshold go through the pinned ring upload
(engine._upload_bytes): results must be bitwise those of the same matrix passed
as a CUDA tensor, for F- and C-ordered arrays with a ragged last chunk."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("order", ["F", "C"])
def test_staged_upload_matches_device_input(order):
    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import engine

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rs = np.random.default_rng(11)
    m, n = 3001, 2999                         # 72 MB: > 2 staging chunks, ragged tail
    assert m * n * 8 >= 2 * engine._STAGE_CHUNK
    A = rs.standard_normal((m, n))
    A = np.asfortranarray(A) if order == "F" else np.ascontiguousarray(A)
    ap_np = ffb.flip_flop_srqr(A, 20, l=40, b=16, p=4, seed=3)
    # the same storage order on the device: F -> column-major view, C -> row-major
    # (FFB_LAYOUT_ROW, read in place)
    Ad = torch.from_numpy(np.asfortranarray(A).T).cuda().t() if order == "F" else torch.from_numpy(A).cuda()
    ap_dev = ffb.flip_flop_srqr(Ad, 20, l=40, b=16, p=4, seed=3)
    assert np.array_equal(np.asarray(ap_np.s), ap_dev.s.cpu().numpy())
    assert np.array_equal(np.asarray(ap_np.u), ap_dev.u.cpu().numpy())
    assert np.array_equal(ap_np.meta["srqr"].fact.perm, ap_dev.meta["srqr"].fact.perm.cpu().numpy())


@pytest.mark.parametrize("layout", ["row", "col"])
def test_staged_download_matches_cpu_copy(layout):
    from paper_1803_01982_b200 import engine

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = torch.Generator(device="cuda").manual_seed(5)
    base = torch.randn(3003, 2999, generator=g, dtype=torch.float64, device="cuda")
    x = base if layout == "row" else base.t()      # contiguous / column-major view
    got = engine._download(torch, x)
    ref = x.cpu().numpy()
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


def test_host_pipeline_matches_direct_calls():
    """batch.run_host_pipeline (uploads on a copy stream, compute on a stream pool)
    returns, in input order, exactly what one-at-a-time calls return."""
    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import batch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rs = np.random.default_rng(21)
    hosts = []
    for i in range(7):
        A = rs.standard_normal((400 + 10 * i, 300))
        h = torch.empty((300, 400 + 10 * i), dtype=torch.float64, pin_memory=True)
        h.copy_(torch.from_numpy(A.T))
        hosts.append(h.t())                       # column-major pinned view
    got = batch.run_host_pipeline(
        hosts, lambda i, Ad: ffb.flip_flop_srqr(Ad, 10, l=24, b=8, p=4, seed=i).s.cpu().numpy(),
        n_streams=3, prefetch=1)
    for i, h in enumerate(hosts):
        ref = ffb.flip_flop_srqr(h.cuda(), 10, l=24, b=8, p=4, seed=i).s.cpu().numpy()
        assert np.array_equal(got[i], ref)


@pytest.mark.parametrize("shape", [(700, 500), (500, 700)])
def test_row_major_layout_matches_column_major(shape):
    """FFB_LAYOUT_ROW (a C-ordered matrix read in place: row-major sketch / WT /
    A*Qhat GEMM operands, row-major column norms, gathers and row copies) gives
    the column-major factorization: same pivots, sigma and certificate to
    rounding, for flip_flop_srqr, srqr and rsisvd."""
    import paper_1803_01982_b200 as ffb

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n = shape
    rs = np.random.default_rng(m)
    U, _ = np.linalg.qr(rs.standard_normal((m, 200)))
    V, _ = np.linalg.qr(rs.standard_normal((n, 200)))
    A = (U * np.geomspace(1, 1e-5, 200)) @ V.T + 1e-9 * rs.standard_normal((m, n))
    Ac = torch.from_numpy(np.ascontiguousarray(A)).cuda()            # row-major
    Af = torch.from_numpy(np.asfortranarray(A).T).cuda().t()         # column-major
    assert Ac.stride(1) == 1 and Af.stride(0) == 1
    a_r = ffb.flip_flop_srqr(Ac, 40, l=60, b=32, p=8, g=1.2, seed=5)
    a_c = ffb.flip_flop_srqr(Af, 40, l=60, b=32, p=8, g=1.2, seed=5)
    assert torch.equal(a_r.meta["srqr"].fact.perm, a_c.meta["srqr"].fact.perm)
    assert a_r.meta["srqr"].cert.swaps == a_c.meta["srqr"].cert.swaps
    torch.testing.assert_close(a_r.s, a_c.s, rtol=1e-12, atol=0)
    assert abs(a_r.meta["srqr"].cert.g2 - a_c.meta["srqr"].cert.g2) <= 1e-12 * a_c.meta["srqr"].cert.g2
    r_r = ffb.rsisvd(Ac, 30, p=10, q=1, seed=2)
    r_c = ffb.rsisvd(Af, 30, p=10, q=1, seed=2)
    torch.testing.assert_close(r_r.s, r_c.s, rtol=1e-12, atol=0)
