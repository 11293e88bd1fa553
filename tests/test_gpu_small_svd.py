"""ffb_small_svd — the device replacement for the dgesdd of the flip-flop tail
(ffsrqr/svd.py:79) — against LAPACK over the column-ring kernel's whole domain
(l <= 448 with FFB_RING_MAXL lifted: every lane-group width and rows-per-lane
instance, odd l, one CTA up to a 16-CTA cluster), both iterate orientations, and
degenerate inputs."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _check(R, rtol=1e-11):
    from paper_1803_01982_b200 import dense

    l = R.shape[0]
    U, sig, V, sweeps = dense.small_svd(torch.from_numpy(np.asfortranarray(R)).cuda())
    s = sig.cpu().numpy()
    want = np.linalg.svd(R, compute_uv=False)
    scale = max(want[0], np.finfo(float).tiny)
    big = want > 1e-13 * scale
    np.testing.assert_allclose(s[big], want[big], rtol=rtol)
    assert np.all(np.abs(s[~big] - want[~big]) <= 1e-13 * scale)
    assert np.all(np.diff(s) <= 0)
    Uh, Vh = U.cpu().numpy(), V.cpu().numpy()
    assert np.abs((Uh * s) @ Vh.T - R).max() <= 1e-13 * l * scale
    r = int(big.sum())
    assert np.abs(Uh[:, :r].T @ Uh[:, :r] - np.eye(r)).max() < 1e-12 * l
    assert np.abs(Vh[:, :r].T @ Vh[:, :r] - np.eye(r)).max() < 1e-12 * l
    assert 0 < sweeps < 30
    return sweeps


def _rt(l, lo, seed):
    g = np.random.default_rng(seed)
    U0, _ = np.linalg.qr(g.standard_normal((l, l)))
    V0, _ = np.linalg.qr(g.standard_normal((l, l)))
    return np.linalg.qr((U0 * np.geomspace(1.0, lo, l)) @ V0.T, mode="r")


@pytest.mark.parametrize("l", [2, 3, 17, 31, 32, 33, 50, 60, 64, 65, 96, 127, 144, 161, 200, 223, 256, 272,
                               289, 300, 333, 352, 385, 420, 447, 448])
def test_ring_sizes_against_lapack(l, monkeypatch):
    monkeypatch.setenv("FFB_RING_MAXL", "448")   # the default hands l > 160 to the block kernel
    _check(_rt(l, 1e-3, l))


@pytest.mark.parametrize("env", [{"FFB_RING_NOTRANS": "1"}, {"FFB_RING_C": "16"}, {"FFB_RING_C": "1"},
                                 {"FFB_RING_C": "2", "FFB_RING_G": "4"}, {"FFB_RING_PPC": "3"},
                                 {"FFB_RING_G": "8"}, {"FFB_RING_G": "16"}, {"FFB_RING_G": "32"}])
def test_ring_geometry_knobs(env, monkeypatch):
    # iterate on M instead of M^T; forced lane-group widths and cluster sizes
    # (halo pushes on every boundary, CTAs without slots, several pairs per
    # warp) — the library reads the knobs per call; geometries that do not fit
    # fall back to the block kernel
    monkeypatch.setenv("FFB_RING_MAXL", "448")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for l in (7, 60, 61, 144, 272):
        _check(_rt(l, 1e-3, 7 * l))


def test_ring_dense_and_graded():
    g = np.random.default_rng(5)
    _check(g.standard_normal((150, 150)))
    _check(_rt(100, 1e-12, 3), rtol=1e-10)
    _check(1e-140 * _rt(90, 1e-3, 4))
    _check(1e140 * _rt(90, 1e-3, 6))


def test_ring_rank_deficient_and_zero():
    g = np.random.default_rng(9)
    l, r = 120, 7
    R = g.standard_normal((l, r)) @ g.standard_normal((r, l))
    _check(R)
    _check(np.diag(np.r_[np.ones(5), np.zeros(35)]))
    from paper_1803_01982_b200 import dense

    U, sig, V, sweeps = dense.small_svd(torch.zeros(40, 40, dtype=torch.float64, device="cuda").t())
    assert float(sig.abs().max()) == 0.0


def test_ring_is_bitwise_repeatable():
    from paper_1803_01982_b200 import dense

    R = torch.from_numpy(np.asfortranarray(_rt(272, 0.5, 1))).cuda()
    U0, s0, V0, _ = dense.small_svd(R)
    for _ in range(3):
        U, s, V, _ = dense.small_svd(R)
        assert torch.equal(U, U0) and torch.equal(s, s0) and torch.equal(V, V0)


def test_block_kernel_still_matches(monkeypatch):
    # the block kernels stay the path for l > 448 and behind FFB_JACOBI_BLOCK
    monkeypatch.setenv("FFB_JACOBI_BLOCK", "1")
    _check(_rt(144, 1e-3, 2))
