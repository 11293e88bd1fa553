"""Caller seams: unfold column order matches ffsrqr/tensor.py:21-27 (numpy and
torch), the hosvd engine honours config 4's parameters, and install_into
rebinds the reference's tensor/nuclear names."""
import types

import numpy as np
import pytest

from paper_1803_01982_b200 import callers


def _ref_unfold(X, mode):
    return np.reshape(np.moveaxis(X, mode, 0), (X.shape[mode], -1), order="F")


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_unfold_order(mode):
    X = np.random.default_rng(0).standard_normal((3, 4, 5))
    assert np.array_equal(callers.unfold(X, mode), _ref_unfold(X, mode))
    torch = pytest.importorskip("torch")
    Mt = callers.unfold(torch.from_numpy(X), mode)
    assert Mt.stride(0) == 1  # column-major for the engine
    assert np.array_equal(Mt.numpy(), _ref_unfold(X, mode))


def test_install_into_rebinds_and_restores():
    fake = types.SimpleNamespace(tensor=types.SimpleNamespace(flip_flop_srqr="t"),
                                 nuclear=types.SimpleNamespace(flip_flop_srqr="n"))
    prev = callers.install_into(fake)
    assert prev == ("t", "n")
    from paper_1803_01982_b200 import flip_flop_srqr

    assert fake.tensor.flip_flop_srqr is flip_flop_srqr and fake.nuclear.flip_flop_srqr is flip_flop_srqr


def test_hosvd_engine_parameters(monkeypatch):
    seen = {}

    def fake(M, r, l=None, b=32, p=5, seed=0):
        seen.update(r=r, l=l, b=b, p=p, seed=seed)
        return "ok"

    monkeypatch.setattr(callers, "flip_flop_srqr", fake)
    eng = callers.hosvd_engine()
    assert eng(np.zeros((400, 160000)), 40) == "ok"
    assert seen == dict(r=40, l=50, b=32, p=10, seed=0)
