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
    Ad = torch.from_numpy(np.asfortranarray(A).T).cuda().t()
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
