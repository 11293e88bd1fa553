"""GPU parity at BASELINE.json's FULL sizes: the engine (C ABI) vs the CPU oracle
on the same input bytes and the same host-generated sketches.

The oracle (pinned to the reference goldens by test_oracle_golden.py) finishes
cfg2/cfg3 in ~5-12 s on the box's host cores, so these configurations are
compared directly, not only through size-independent properties:

* pivots identical, or divergent only after a certified near-tie
  (recorded top-2 relative gap below 1e-12);
* swap count and the i_off sequence identical (cfg3 at g = 1.5 takes the
  reference's swap path);
* singular values and diag(L) within 1e-10 relative;
* certificate scalars (alpha, g1, g2, tau bounds) within 1e-10 relative;
* ||A P - Q R||_F / ||A||_F within 1e-12 of the oracle's;
* u / v columns equal up to sign where the spectrum is not clustered
  (|u_i . u'_i| >= 1 - 1e-10), u / v orthonormal to 1e-12.

Plus the size-independent properties the domain offers on the device-resident
path (no host copies): orthonormality, the SRQR certificate identities, and
bitwise determinism of a repeated call.
"""
import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RTOL = 1e-10


@pytest.fixture(scope="module")
def ffb():
    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import _capi

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _capi.load()
    return ffb


def _matrix(name):
    """(numpy A, device A) with identical bytes."""
    from paper_1803_01982_b200 import workloads

    if name == "cfg2":
        Ad = workloads.torch_matrix("cfg2", seed=0)
        return Ad.cpu().numpy(), Ad
    if name == "cfg4":
        Xs = workloads.torch_tensor_unfoldings(seed=0)
        Ad = Xs[0]
        del Xs
        return Ad.cpu().numpy(), Ad
    A = np.asfortranarray(workloads.numpy_matrix(name, seed=0))
    return A, torch.from_numpy(A.T.copy()).cuda().t()


def _first_divergence(a, b):
    d = np.nonzero(np.asarray(a) != np.asarray(b))[0]
    return int(d[0]) if d.size else -1


def _compare(ffb, A, Ad, k, l, b, p, g):
    ap = ffb.flip_flop_srqr(Ad, k, l=l, b=b, p=p, g=g, seed=0, trace_gaps=True)
    ref = oracle.flip_flop(A, k, l=l, b=b, p=p, g=g, seed=0)
    sr = ap.meta["srqr"]
    perm = sr.fact.perm.cpu().numpy()
    j = _first_divergence(perm, ref.sr.perm)
    if j >= 0:
        gap = ap.meta["pivot_gap"].cpu().numpy()
        assert j < l and gap[j] < 1e-12, f"pivot {j} differs without a certified near-tie"
        pytest.skip(f"certified near-tie at pivot {j} (gap {gap[j]:.1e}); sequences legitimately differ")
    assert sr.cert.swaps == ref.sr.swaps
    assert ap.meta["i_offs"] == [int(i) for i in ref.sr.i_offs[:64]]
    s = ap.s.cpu().numpy()
    np.testing.assert_allclose(s, ref.s, rtol=RTOL, atol=1e-14 * ref.s[0])
    dl = ap.meta["diag_L"].cpu().numpy()
    np.testing.assert_allclose(dl, ref.diag_L, rtol=RTOL, atol=1e-13 * abs(ref.diag_L[0]))
    np.testing.assert_allclose([sr.cert.alpha, sr.cert.g1, sr.cert.g2, sr.cert.tau_bound,
                                sr.cert.tau_hat_bound],
                               [ref.sr.alpha, ref.sr.g1, ref.sr.g2, ref.sr.tau_bound,
                                ref.sr.tau_hat_bound], rtol=RTOL)
    # residual parity on the device: ||A P - Q R||_F / ||A||_F
    Q = sr.q_ext[:, :l]
    R = sr.fact.R
    P = torch.as_tensor(perm, device=Ad.device)
    nA = float(torch.linalg.norm(Ad))
    ours = float(torch.linalg.norm(Ad[:, P] - Q @ R)) / nA
    theirs = np.linalg.norm(A[:, ref.sr.perm] - ref.sr.Q[:, :l] @ ref.sr.R) / np.linalg.norm(A)
    assert abs(ours - theirs) <= 1e-12, (ours, theirs)
    # singular vectors: orthonormal, and equal to the oracle's up to sign off clusters
    u = ap.u.cpu().numpy()
    v = ap.v.cpu().numpy()
    assert np.abs(u.T @ u - np.eye(k)).max() < 1e-12
    assert np.abs(v.T @ v - np.eye(k)).max() < 1e-12
    rel_gap = np.full(k, np.inf)
    sv = ref.sv_all
    for i in range(k):
        lo = abs(sv[i] - sv[i - 1]) if i > 0 else np.inf
        hi = abs(sv[i] - sv[i + 1])
        rel_gap[i] = min(lo, hi) / sv[0]
    ok = rel_gap > 1e-6
    # subspace angle error of a singular vector ~ eps * ||A|| / gap
    du = np.abs(np.sum(u * ref.u, axis=0))
    dv = np.abs(np.sum(v * ref.v, axis=0))
    assert np.all(du[ok] > 1 - 1e-10) and np.all(dv[ok] > 1 - 1e-10), (du[ok].min(), dv[ok].min())
    return ap, ref


@pytest.mark.parametrize("g", [2.0, 1.5])
def test_cfg3_full_size(ffb, g):
    A, Ad = _matrix("cfg3")
    ap, ref = _compare(ffb, A, Ad, 400, 420, 64, 20, g)
    if g == 1.5:
        assert ref.sr.swaps > 0, "g = 1.5 must exercise the swap path"


def test_cfg2_full_size(ffb):
    A, Ad = _matrix("cfg2")
    _compare(ffb, A, Ad, 256, 272, 64, 16, 2.0)


def test_cfg5_one_matrix_full_size(ffb):
    A, Ad = _matrix("cfg5")
    _compare(ffb, A, Ad, 128, 144, 32, 16, 2.0)


def test_cfg4_one_unfolding_full_size(ffb):
    A, Ad = _matrix("cfg4")
    _compare(ffb, A, Ad, 40, 50, 32, 10, 2.0)


def test_cfg2_device_properties_and_determinism(ffb):
    """Size-independent checks on the device-resident path (no oracle):
    orthonormal u, v, Q; R upper trapezoidal in arranged order; the certificate
    identities g1 = r22/alpha and tau = g1 g2 sqrt((l+1)(n-l)); bitwise repeat."""
    from paper_1803_01982_b200 import workloads

    Ad = workloads.torch_matrix("cfg2", seed=1)
    m, n = Ad.shape
    k, l = 256, 272
    a1 = ffb.flip_flop_srqr(Ad, k, l=l, b=64, p=16, seed=3)
    a2 = ffb.flip_flop_srqr(Ad, k, l=l, b=64, p=16, seed=3)
    assert torch.equal(a1.u, a2.u) and torch.equal(a1.s, a2.s) and torch.equal(a1.v, a2.v)
    eye = torch.eye(k, dtype=torch.float64, device=Ad.device)
    assert float((a1.u.T @ a1.u - eye).abs().max()) < 1e-12
    assert float((a1.v.T @ a1.v - eye).abs().max()) < 1e-12
    sr = a1.meta["srqr"]
    Q = sr.q_ext
    assert float((Q.T @ Q - torch.eye(l + 1, dtype=torch.float64, device=Ad.device)).abs().max()) < 1e-11
    R = sr.fact.R
    assert float(torch.tril(R[:, :l], -1).abs().max()) == 0.0
    c = sr.cert
    assert math.isclose(c.g1, sr.r22_norm_estimate / c.alpha, rel_tol=1e-12)
    assert math.isclose(c.tau_bound, c.g1 * c.g2 * math.sqrt((l + 1) * (n - l)), rel_tol=1e-12)
    # interlacing: the singular values of A P Qhat_1 (orthonormal Qhat_1) never
    # exceed A's own, which the generator fixes exactly
    true = torch.as_tensor(workloads.spectrum("cfg2", k), device=Ad.device)
    assert bool((a1.s <= true * (1 + 1e-10)).all())
    assert bool((a1.s[:-1] >= a1.s[1:]).all())
    # u^T A v = diag(s) up to the rank-l truncation error
    S = a1.u.T @ (Ad @ a1.v)
    assert float((torch.diagonal(S) - a1.s).abs().max()) < 1e-10
