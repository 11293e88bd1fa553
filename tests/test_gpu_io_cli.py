"""GPU: DMAT/DTEN straight into HBM (pinned readinto + async H2D) and the CLI's
compute verbs on the engine (ffsrqr/cli.py:372-441), checked against the
numpy readers and the direct API calls."""
import csv
import io as pyio
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


@pytest.fixture(scope="module")
def ffb():
    import paper_1803_01982_b200 as ffb

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return ffb


def test_read_into_device(ffb):
    from paper_1803_01982_b200 import io

    A = io.read_dmat(os.path.join(GOLD, "a37x23.dmat"), device="cuda")
    X = io.read_dten(os.path.join(GOLD, "x5x4x3.dten"), device="cuda")
    exp = np.load(os.path.join(GOLD, "expected.npz"))
    assert A.is_cuda and A.stride(0) == 1            # column-major, zero reordering
    assert X.is_cuda and X.stride(0) == 1            # first index fastest
    np.testing.assert_array_equal(A.cpu().numpy(), exp["A"])
    np.testing.assert_array_equal(X.cpu().numpy(), exp["X"])


def _records(out):
    rows = list(csv.reader(pyio.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[1:]]


def test_cli_svd_matches_api(ffb, tmp_path, capsys):
    from paper_1803_01982_b200 import cli, io, workloads

    A = workloads.numpy_matrix("cfg1", m=400, n=300)
    io.write_dmat(tmp_path / "a.dmat", A)
    rc = cli.main(["svd", "--in", str(tmp_path / "a.dmat"), "--k", "20", "--l", "30", "--p", "10",
                   "--artifacts", str(tmp_path / "ap")])
    assert rc == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    ap = ffb.flip_flop_srqr(A, 20, l=30, p=10)
    assert rec["kind"] == "svd" and int(rec["k"]) == 20
    np.testing.assert_allclose(float(rec["sigma_1"]), ap.s[0], rtol=1e-12)
    err = np.linalg.norm(A - (ap.u * ap.s) @ ap.v.T) / np.linalg.norm(A)
    assert abs(float(rec["rel_error"]) - err) <= 1e-10
    back = io.load_approx_svd(str(tmp_path / "ap"))
    np.testing.assert_allclose(back.s, ap.s, rtol=1e-12)


def test_cli_tensor_and_rpca(ffb, tmp_path, capsys):
    from paper_1803_01982_b200 import cli, io

    g = np.random.default_rng(5)
    core = g.standard_normal((4, 3, 2))
    Us = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in ((20, 4), (15, 3), (12, 2))]
    X = np.einsum("abc,ia,jb,kc->ijk", core, *Us)
    io.write_dten(tmp_path / "x.dten", X)
    assert cli.main(["tensor", "--in", str(tmp_path / "x.dten"), "--ranks", "4,3,2",
                     "--engine", "rsisvd"]) == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    assert float(rec["rel_error"]) < 1e-12
    L = g.standard_normal((60, 3)) @ g.standard_normal((3, 40))
    io.write_dmat(tmp_path / "m.dmat", L)
    assert cli.main(["rpca", "--in", str(tmp_path / "m.dmat"), "--engine", "flipflop",
                     "--max-iter", "10"]) == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    assert rec["kind"] == "rpca" and int(rec["iterations"]) >= 1
