"""``python -m paper_1803_01982_b200 <verb>`` — the reference CLI's compute verbs
on the B200 engine (ffsrqr/cli.py:250-477): ``svd``, ``tensor``, ``rpca``,
``complete``.  Same flags, same CSV/TSV record columns, same exit codes
(0 ok, 2 config error, 3 numerical failure).  Inputs go straight from
DMAT/DTEN/CSV into HBM (``io.py``); ``rel_error`` is computed on the device.
The experiment-sweep verb ``bench`` is out of scope (bench.py measures the
BASELINE workloads).
"""
from __future__ import annotations

import argparse
import csv
import math
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import io
from .errors import CertificationError, DimensionError, NumericalError, SingularTrailingBlockError

EXIT_OK = 0
EXIT_CONFIG = 2
EXIT_NUMERICAL = 3

_SIGMA_COLS = 20
CSV_COLUMNS = (["kind", "method", "k", "rel_error", "flop_count", "iterations", "sv_count",
                "status"] + [f"sigma_{j}" for j in range(1, _SIGMA_COLS + 1)] + ["runtime_s"])


@dataclass
class ResultRecord:
    """ffsrqr/cli.py:39-58."""
    kind: str
    method: str
    k: int
    rel_error: float = float("nan")
    flop_count: int = 0
    iterations: int = 0
    sv_count: int = 0
    status: str = "ok"
    sigmas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    runtime_s: float = 0.0

    def row(self):
        sig = ["" for _ in range(_SIGMA_COLS)]
        for j, v in enumerate(self.sigmas[:_SIGMA_COLS]):
            sig[j] = repr(float(v))
        return ([self.kind, self.method, self.k, repr(float(self.rel_error)), self.flop_count,
                 self.iterations, self.sv_count, self.status] + sig + [f"{self.runtime_s:.6f}"])


def write_records(records, path, fmt="csv"):
    delim = "," if fmt == "csv" else "\t"
    out = open(path, "w", newline="") if path else sys.stdout
    try:
        w = csv.writer(out, delimiter=delim)
        w.writerow(CSV_COLUMNS)
        for rec in records:
            w.writerow(rec.row())
    finally:
        if path:
            out.close()


def _ints(text):
    return tuple(int(t) for t in str(text).split(",") if t.strip())


def _load_matrix(args, dev):
    if args.input is None:
        raise ValueError("--in is required")
    if args.input.endswith(".csv"):
        return io.read_csv_matrix(args.input, dev)
    return io.read_dmat(args.input, dev)


def _rel_error(A, ap):
    """||A - U diag(s) V^T||_F / ||A||_F on the device (DMMA GEMM)."""
    from . import dense

    X = dense.gemm(ap.u * ap.s, ap.v.t())
    num = math.sqrt(float(dense.sumsq((A - X).t().contiguous())[0]))
    den = math.sqrt(float(dense.sumsq(A.t().contiguous())[0]))
    return num / max(den, 1e-300)


def _run_svd(args, dev):
    from .engine import flip_flop_srqr, rsisvd

    if args.k is None:
        raise ValueError("--k is required")
    A = _load_matrix(args, dev)
    t0 = time.perf_counter()
    if args.method == "flipflop":
        ap = flip_flop_srqr(A, args.k, l=args.l, b=args.b, p=args.p, epsilon=args.epsilon,
                            g=args.g, seed=args.seed)
    elif args.method == "rsisvd":
        ap = rsisvd(A, args.k, p=args.p, q=args.q, seed=args.seed)
    else:
        mn = min(A.shape)
        ap = rsisvd(A, args.k, p=mn - args.k, q=0, seed=args.seed)
    rt = time.perf_counter() - t0
    if args.artifacts:
        io.save_approx_svd(args.artifacts, ap)
    rec = ResultRecord(kind="svd", method=args.method, k=args.k, rel_error=_rel_error(A, ap),
                       flop_count=ap.flop_count, sv_count=ap.k, sigmas=ap.s.cpu().numpy(),
                       runtime_s=rt)
    write_records([rec], args.out, args.format)


def _run_tensor(args, dev):
    from . import tensor

    X = io.read_dten(args.input, dev)
    ranks = _ints(args.ranks)
    t0 = time.perf_counter()
    dec = tensor.st_hosvd(X, ranks, engine=args.engine, seed=args.seed)
    rt = time.perf_counter() - t0
    if args.artifacts:
        io.write_dten(args.artifacts + ".core.dten", dec.core)
        for i, U in enumerate(dec.factors):
            io.write_dmat(args.artifacts + f".factor{i}.dmat", U)
    rec = ResultRecord(kind="tensor", method=args.engine, k=max(ranks),
                       rel_error=tensor.tucker_error(X, dec), flop_count=dec.flop_count,
                       runtime_s=rt)
    write_records([rec], args.out, args.format)


def _ialm_params(args):
    from .nuclear import IalmParams

    return IalmParams(lam=args.lam, mu0=args.mu0, rho=args.rho, tol=args.tol,
                      max_iter=args.max_iter, sv0=args.sv0, svd_engine=args.engine, seed=args.seed)


def _run_rpca(args, dev):
    from . import nuclear

    M = _load_matrix(args, dev)
    t0 = time.perf_counter()
    st = nuclear.ialm_rpca(M, _ialm_params(args))
    rt = time.perf_counter() - t0
    if args.artifacts:
        io.write_dmat(args.artifacts + ".x.dmat", st.low_rank)
        io.write_dmat(args.artifacts + ".e.dmat", st.sparse)
    res = st.residuals[-1] if st.residuals else float("nan")
    rec = ResultRecord(kind="rpca", method=args.engine, k=st.rank, rel_error=res,
                       iterations=st.iterations, sv_count=st.rank,
                       status="ok" if st.converged else "maxiter", runtime_s=rt)
    write_records([rec], args.out, args.format)


def _run_complete(args, dev):
    from . import nuclear

    if args.ratings:
        rows, cols, vals = io.read_ratings(args.ratings)
    else:
        rows, cols, vals = io.read_observations(args.input)
    shape = _ints(args.shape) if args.shape else None
    M, mask = io.observations_to_dense(rows, cols, vals, shape, device=dev)
    t0 = time.perf_counter()
    st = nuclear.ialm_mc(M, mask, _ialm_params(args))
    rt = time.perf_counter() - t0
    if args.artifacts:
        io.write_dmat(args.artifacts + ".x.dmat", st.low_rank)
    res = st.residuals[-1] if st.residuals else float("nan")
    rec = ResultRecord(kind="complete", method=args.engine, k=st.rank, rel_error=res,
                       iterations=st.iterations, sv_count=st.rank,
                       status="ok" if st.converged else "maxiter", runtime_s=rt)
    write_records([rec], args.out, args.format)


def build_parser():
    """Flags of ffsrqr/cli.py:255-317 for the compute verbs."""
    p = argparse.ArgumentParser(prog="python -m paper_1803_01982_b200")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", help="CSV output path (default stdout)")
    p.add_argument("--format", choices=("csv", "tsv"), default="csv")
    p.add_argument("--device", default="cuda:0")
    sub = p.add_subparsers(dest="verb", required=True)

    def common(sp):
        sp.add_argument("--in", dest="input", help="input file")
        sp.add_argument("--artifacts", help="output artifact path prefix")

    ps = sub.add_parser("svd", help="rank-k approximate SVD")
    common(ps)
    ps.add_argument("--k", type=int)
    ps.add_argument("--l", type=int)
    ps.add_argument("--b", type=int, default=32)
    ps.add_argument("--p", type=int, default=5)
    ps.add_argument("--g", type=float, default=2.0)
    ps.add_argument("--epsilon", type=float, default=0.5)
    ps.add_argument("--q", type=int, default=1)
    ps.add_argument("--method", choices=("flipflop", "rsisvd", "exact"), default="flipflop")
    pt = sub.add_parser("tensor", help="Tucker compression (ST-HOSVD)")
    common(pt)
    pt.add_argument("--ranks", required=True)
    pt.add_argument("--engine", choices=("exact", "flipflop", "rsisvd"), default="exact")
    for name in ("rpca", "complete"):
        pr = sub.add_parser(name)
        common(pr)
        if name == "complete":
            pr.add_argument("--ratings")
            pr.add_argument("--shape")
        pr.add_argument("--engine", choices=("exact", "flipflop", "rsisvd"), default="exact")
        pr.add_argument("--lam", type=float)
        pr.add_argument("--mu0", type=float)
        pr.add_argument("--rho", type=float, default=1.5)
        pr.add_argument("--tol", type=float, default=1e-7)
        pr.add_argument("--max-iter", type=int, default=100)
        pr.add_argument("--sv0", type=int, default=10)
    return p


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return EXIT_CONFIG if exc.code not in (0, None) else 0
    runner = {"svd": _run_svd, "tensor": _run_tensor, "rpca": _run_rpca,
              "complete": _run_complete}[args.verb]
    try:
        runner(args, args.device)
    except (NumericalError, CertificationError, SingularTrailingBlockError) as exc:
        print(f"ffb200: numerical failure: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL
    except (ValueError, OSError, KeyError) as exc:
        print(f"ffb200: config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    return EXIT_OK
