"""Time ffb_small_svd (the flip-flop's Jacobi SVD) on R_t-like inputs per l and
check it against LAPACK: python tools/jacobi_bench.py [l ...] (run under gpurun;
FFB_JACOBI_WIDE=1 selects the 16-column cluster kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01982_b200 import dense, workloads  # noqa: E402

for l in [int(x) for x in sys.argv[1:]] or [60, 144, 272, 420, 512]:
    g = np.random.default_rng(l)
    U0, _ = np.linalg.qr(g.standard_normal((l, l)))
    V0, _ = np.linalg.qr(g.standard_normal((l, l)))
    s0 = workloads.spectrum("cfg2" if l == 272 else "cfg5", l)
    R = np.linalg.qr((U0 * s0) @ V0.T, mode="r")
    Rd = torch.from_numpy(np.asfortranarray(R)).cuda()
    for _ in range(2):
        U, sig, V, sw = dense.small_svd(Rd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        U, sig, V, sw = dense.small_svd(Rd)
    e1.record()
    torch.cuda.synchronize()
    want = np.linalg.svd(R, compute_uv=False)
    err = np.max(np.abs(sig.cpu().numpy() - want) / want)
    Uh, Vh = U.cpu().numpy(), V.cpu().numpy()
    rec = np.abs((Uh * sig.cpu().numpy()) @ Vh.T - R).max()
    orth = max(np.abs(Uh.T @ Uh - np.eye(l)).max(), np.abs(Vh.T @ Vh - np.eye(l)).max())
    print(f"l={l} {e0.elapsed_time(e1) / 5:.3f} ms sweeps={sw} sigma_rel={err:.1e} recon={rec:.1e} orth={orth:.1e}",
          flush=True)
