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
    assert got == case["sha256"], f"input bytes for {name} differ from the golden run"
    case["orders"] = [case[f"block_order_{i}"] for i in range(case["n_blocks"])]
    return case
