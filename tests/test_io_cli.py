"""DMAT / DTEN readers and writers (ffsrqr/io.py:27-155) against files written
by the reference's own writers (tests/golden/io/make_golden_io.py), and the CLI
front end's argument / exit-code contract (ffsrqr/cli.py:455-477).  CPU only."""
import os

import numpy as np
import pytest

from paper_1803_01982_b200 import cli, io

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def test_read_reference_dmat_dten():
    exp = np.load(os.path.join(GOLD, "expected.npz"))
    A = io.read_dmat(os.path.join(GOLD, "a37x23.dmat"))
    X = io.read_dten(os.path.join(GOLD, "x5x4x3.dten"))
    np.testing.assert_array_equal(A, exp["A"])
    np.testing.assert_array_equal(X, exp["X"])


def test_writers_are_byte_identical_to_reference(tmp_path):
    exp = np.load(os.path.join(GOLD, "expected.npz"))
    io.write_dmat(tmp_path / "a.dmat", exp["A"])
    io.write_dten(tmp_path / "x.dten", exp["X"])
    assert (tmp_path / "a.dmat").read_bytes() == open(os.path.join(GOLD, "a37x23.dmat"), "rb").read()
    assert (tmp_path / "x.dten").read_bytes() == open(os.path.join(GOLD, "x5x4x3.dten"), "rb").read()


def test_bad_and_truncated_files(tmp_path):
    from paper_1803_01982_b200.errors import NumericalError

    (tmp_path / "bad.dmat").write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(NumericalError):
        io.read_dmat(tmp_path / "bad.dmat")
    good = open(os.path.join(GOLD, "a37x23.dmat"), "rb").read()
    (tmp_path / "short.dmat").write_bytes(good[:-8])
    with pytest.raises(NumericalError):
        io.read_dmat(tmp_path / "short.dmat")
    with pytest.raises(NumericalError):
        io.write_dmat(tmp_path / "nan.dmat", np.array([[np.nan]]))


def test_observations_to_dense():
    M, mask = io.observations_to_dense(np.array([0, 2]), np.array([1, 0]), np.array([3.0, 4.0]))
    assert M.shape == (3, 2) and mask.sum() == 2 and M[0, 1] == 3.0 and M[2, 0] == 4.0


def test_cli_contract_without_device(capsys):
    assert cli.main(["svd", "--in", os.path.join(GOLD, "a37x23.dmat")]) == cli.EXIT_CONFIG   # no --k
    assert cli.main(["bogus-verb"]) == cli.EXIT_CONFIG
    assert cli.CSV_COLUMNS[:8] == ["kind", "method", "k", "rel_error", "flop_count", "iterations",
                                   "sv_count", "status"]
