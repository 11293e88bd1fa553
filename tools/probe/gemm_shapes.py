"""Time ffb_gemm (beta = 1, as in the panel trailing updates) per tile config on
the short-K / skinny shapes of the cfg2 launch list.  Run under gpurun."""
import ctypes as C
import os
import subprocess
import sys

SHAPES = {  # name: (M, N, K, a_kc, b_kc)
    "trail_8192x208x64": (8192, 208, 64, 0, 1),
    "trail_8192x272x64": (8192, 272, 64, 0, 1),
    "trail_8000x16x64": (8000, 16, 64, 0, 1),
    "hhW_64x208x8192": (64, 208, 8192, 1, 1),
    "T12_64x64x8128": (64, 64, 8128, 1, 1),
    "T12_192x64x8000": (192, 64, 8000, 1, 1),
    "W2_64x208x64": (64, 208, 64, 1, 1),
}


def run_one():
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    from paper_1803_01982_b200 import _capi
    lib = _capi.load()
    ctx = _capi.context(0)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    for name, (M, N, K, akc, bkc) in SHAPES.items():
        A = torch.randn(M * K, dtype=torch.float64, device="cuda")
        B = torch.randn(K * N, dtype=torch.float64, device="cuda")
        Cm = torch.zeros(M * N, dtype=torch.float64, device="cuda")
        lda = K if akc else M
        ldb = K if bkc else N

        def go():
            rc = lib.ffb_gemm(ctx, C.c_void_p(st.cuda_stream), M, N, K, -1.0, C.c_void_p(A.data_ptr()),
                              lda, akc, C.c_void_p(B.data_ptr()), ldb, bkc, 1.0,
                              C.c_void_p(Cm.data_ptr()), M, C.c_void_p(ws.data_ptr()), ws.numel())
            assert rc == 0
        for _ in range(3):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            go()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 20 * 1000.0
    return res


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        r = run_one()
        print(" ".join(f"{k}={v:.1f}us" for k, v in r.items()))
    else:
        for cfg in ["auto", "0", "1", "3", "6", "7"]:
            env = dict(os.environ)
            if cfg != "auto":
                env["FFB_GEMM_CFG"] = cfg
            out = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
            print(f"cfg={cfg}: {out.stdout.strip() or out.stderr[-300:]}")
