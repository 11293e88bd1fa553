"""Load the caller golden fixtures (tests/golden/callers/*.npz, made by the reference)."""
import glob
import os

import numpy as np

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "callers")


def names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(DIR, prefix + "*.npz")))


def load(name):
    z = np.load(os.path.join(DIR, name + ".npz"), allow_pickle=False)
    out = {k: z[k] for k in z.files}
    for k in ("k", "p", "q", "seed", "max_iter", "rank", "iterations"):
        if k in out:
            out[k] = int(out[k])
    if "engine" in out:
        out["engine"] = str(out["engine"])
    return out


def cols_match_up_to_sign(a, b, tol):
    """max over columns of 1 - |a_i . b_i| / (|a_i| |b_i|)."""
    num = np.abs(np.sum(a * b, axis=0))
    den = np.linalg.norm(a, axis=0) * np.linalg.norm(b, axis=0)
    return float(np.max(1.0 - num / den)) <= tol


def tucker_reconstruct(core, factors):
    G = core
    for n, U in enumerate(factors):
        G = np.moveaxis(np.tensordot(U, np.moveaxis(G, n, 0), axes=1), 0, n)
    return G
