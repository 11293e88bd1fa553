"""Load golden fixtures (tests/golden/*.npz) and rebuild their inputs."""
import glob
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    case = {k: z[k] for k in z.files}
    for k in ("m", "n", "k", "l", "b", "p", "d", "seed", "n_blocks"):
        case[k] = int(case[k])
    case["g"] = float(case["g"])
    case["recipe"] = json.loads(str(case["recipe"]))
    case["srqr_status"] = str(case["srqr_status"])
    case["sha256"] = str(case["sha256"])
    if "A" not in case:
        from paper_1803_01982_b200 import workloads

        r = case["recipe"]
        A = workloads.numpy_matrix(r["cfg"], seed=r["seed"], m=r.get("m"), n=r.get("n"))
        case["A"] = A
    got = hashlib.sha256(np.ascontiguousarray(case["A"], dtype=np.float64).tobytes()).hexdigest()
    case["orders"] = [case[f"block_order_{i}"] for i in range(case["n_blocks"])]
    # numerical rank of the reference factor: with alpha = 0 (exactly / numerically
    # rank-deficient input, l >= rank) every pivot candidate past it is a
    # rounding-level norm, so pivot parity is defined up to num_rank only
    d = np.abs(np.diag(case["R"][:, : case["l"]]))
    case["num_rank"] = int(np.sum(d > 1e-12 * d[0])) if case["cert"][0] == 0.0 and d.size and d[0] > 0 else case["l"]
    case["source"] = "reference"
    if got != case["sha256"]:
        # LAPACK/BLAS rounding differs across host CPUs, so a recipe-built input is not
        # bit-identical off the build container: re-derive the reference outputs with
        # the oracle (itself pinned to the reference goldens by test_oracle_golden.py).
        _rederive_with_oracle(case)
    return case


def _rederive_with_oracle(c):
    import oracle

    prm = oracle.resolve(c["m"], c["n"], c["k"], c["l"], c["b"], c["p"], g=c["g"], d=c["d"],
                         seed=c["seed"], clamp=False)
    trq = oracle.trqrcp(c["A"], prm)
    c["orders"] = trq.block_orders
    try:
        sr = oracle.srqr(c["A"], prm)
        c["srqr_status"] = "ok"
    except oracle.ffsrqr_oracle.OracleError as e:
        sr, c["srqr_status"] = e.payload, "CertificationError"
    c["perm"], c["R"], c["rtilde"], c["q_ext"] = sr.perm, sr.R, sr.rtilde, sr.Q
    c["cert"] = np.array([sr.alpha, sr.g1, sr.g2, sr.swaps, sr.tau_bound, sr.tau_hat_bound, sr.r22])
    if "s" in c:
        ff = oracle.flip_flop(c["A"], c["k"], c["l"], c["b"], c["p"], g=c["g"], d=c["d"], seed=c["seed"])
        c["s"], c["diag_L"] = ff.s, ff.diag_L
        from paper_1803_01982_b200 import workloads

        w = workloads.philox(12345, 777)
        xu = w.standard_normal(c["m"])
        xv = w.standard_normal(c["n"])
        c["u_proj_abs"] = np.abs(ff.u.T @ xu)
        c["v_proj_abs"] = np.abs(ff.v.T @ xv)
    c["source"] = "oracle"
