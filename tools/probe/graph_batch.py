"""Concurrent factorizations on several streams with the graph cache on:
every call must succeed and match the one-stream results bitwise."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1803_01982_b200 as ffb  # noqa: E402
from paper_1803_01982_b200 import batch, engine  # noqa: E402

g = np.random.default_rng(0)
probs = [torch.from_numpy(np.asfortranarray(g.standard_normal((1024, 512)))).cuda() for _ in range(16)]
ref = [ffb.flip_flop_srqr(A, 64, l=72, b=32, p=16, seed=i).s.cpu() for i, A in enumerate(probs)]
bad = 0
for rep in range(4):
    engine.clear_omega_cache()
    engine.prefetch_omega_async([(48, 1024, i) for i in range(16)], threads=4)
    try:
        got = batch.run_streams(list(range(16)), lambda i: ffb.flip_flop_srqr(probs[i], 64, l=72, b=32, p=16, seed=i).s.cpu(),
                                n_streams=8)
        bad += sum(int(not torch.equal(a, b)) for a, b in zip(got, ref))
    except Exception as e:
        print("rep", rep, "failed:", e)
        bad += 100
print("mismatches/failures:", bad, "mode", os.environ.get("FFB_GRAPH_CAPTURE_MODE"))
