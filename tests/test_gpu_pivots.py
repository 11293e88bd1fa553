"""Sketch QRCP pivots (K2) through the C ABI (ffb_block_pivots) against the
oracle's restatement of ffsrqr/_kernels_numba.py:15-94 on the same sketch:
register-resident, shared-memory and large-sketch variants, grids smaller than
the device (FFB_PIV_G), later blocks, exact ties and rank-deficient sketches."""
import ctypes as C

import numpy as np
import pytest

import oracle.ffsrqr_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _pivots(B, j0, bb, arr0=None):
    from paper_1803_01982_b200 import _capi

    s, n = B.shape
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()   # column-major s x n
    arr = torch.arange(n, dtype=torch.int64, device="cuda") if arr0 is None else torch.from_numpy(arr0).cuda()
    pos = torch.empty_like(arr)
    pos[arr] = torch.arange(n, dtype=torch.int64, device="cuda")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    lib = _capi.load()
    rc = lib.ffb_block_pivots(_capi.context(0), C.c_void_p(torch.cuda.current_stream().cuda_stream),
                              C.c_void_p(Bd.data_ptr()), s, n, s, j0, bb, C.c_void_p(arr.data_ptr()),
                              C.c_void_p(pos.data_ptr()), None, C.c_void_p(ws.data_ptr()), ws.numel())
    assert rc == 0
    a, p = arr.cpu().numpy(), pos.cpu().numpy()
    assert np.array_equal(np.argsort(a), p)
    return a


def _sketch(s, n, seed, decay=None):
    g = np.random.default_rng(seed)
    B = g.standard_normal((s, n))
    if decay is not None:
        B *= np.geomspace(1.0, decay, n)[g.permutation(n)]
    return B


SHAPES = [(80, 8192, 64), (80, 5000, 64), (42, 1000, 32), (48, 2048, 32), (128, 4100, 96), (20, 130, 16),
          (37, 513, 32), (96, 64 * 17, 64), (8, 64 * 16, 8), (200, 3000, 160)]


@pytest.mark.parametrize("s,n,bb", SHAPES)
def test_block_pivots_match_oracle(s, n, bb):
    B = _sketch(s, n, 11 * s + n, decay=1e-3)
    got = _pivots(B, 0, bb)
    want = orc.qrcp_pivots(B.copy(), bb)
    assert np.array_equal(got[:bb], want[:bb])


@pytest.mark.parametrize("g", ["7", "18", "40"])
def test_small_grids_give_the_same_arrangement(g, monkeypatch):
    # an SM budget (batches) shrinks the grid: more columns per CTA, other kernel variants
    B = _sketch(48, 2048, 5, decay=1e-2)
    full = _pivots(B, 0, 32)
    monkeypatch.setenv("FFB_PIV_G", g)
    assert np.array_equal(_pivots(B, 0, 32), full)


def test_later_block_and_ties():
    # a later block (positions < j0 fixed, arranged input) and exact ties
    # (duplicate columns: the lowest position wins)
    s, n, j0, bb = 48, 2048, 64, 32
    g = np.random.default_rng(3)
    B = _sketch(s, n, 4)
    B[:, 100] = B[:, 7]
    B[:, 1900] = B[:, 7]
    arr0 = g.permutation(n).astype(np.int64)
    got = _pivots(B, j0, bb, arr0.copy())
    assert np.array_equal(got[:j0], arr0[:j0])
    W = B[:, arr0[j0:]].copy()             # the block restarts at sketch row 0 on the trailing columns
    want = arr0[j0:][orc.qrcp_pivots(W, bb)]
    assert np.array_equal(got[j0:j0 + bb], want[:bb])


def test_rank_deficient_sketch_is_a_permutation():
    # fewer independent columns than steps: candidates' norms hit rounding level
    g = np.random.default_rng(8)
    B = g.standard_normal((40, 5)) @ g.standard_normal((5, 1024))
    B[:, 512:] = 0.0
    got = _pivots(B, 0, 32)
    want = orc.qrcp_pivots(B.copy(), 32)
    assert np.array_equal(got[:5], want[:5])
    assert np.array_equal(np.sort(got), np.arange(1024))
