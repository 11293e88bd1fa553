"""Time ffb_gemm on the hot-path GEMM shapes per tile config (FFB_GEMM_CFG) vs cuBLAS.

usage: python tools/gemm_bench.py [cfg ...]   (run under gpurun; env FFB_GEMM_SK=0 disables stream-K)
"""
import ctypes as C
import os
import subprocess
import sys

SHAPES = {  # name: (M, N, K, a_kc, b_kc)
    "cfg2_WT": (64, 8192, 8192, 1, 1),
    "cfg2_sketch": (80, 8192, 8192, 1, 1),
    "cfg2_K13": (8192, 272, 8192, 0, 1),
    "cfg2_Qform": (8192, 272, 272, 0, 1),
    "cfg2_WT16": (16, 8192, 7936, 1, 1),
    "cfg2_Pupd": (8192, 64, 192, 0, 1),
    "tiny_80x64x64": (80, 64, 64, 0, 1),
    "tiny_64x64x64": (64, 64, 64, 0, 1),
    "tiny_192x64x192": (192, 64, 192, 0, 1),
    "tiny_64x8192x64": (64, 8192, 64, 1, 1),
    "cfg3_WT": (64, 5000, 20000, 1, 1),
    "cfg3_K13": (20000, 420, 5000, 0, 1),
    "cfg5_WT": (32, 2048, 4096, 1, 1),
    "cfg5_K13": (4096, 144, 2048, 0, 1),
    "cfg4_K13": (400, 50, 160000, 0, 1),
    "cfg4_WT": (32, 160000, 400, 1, 1),
    "cfg4_sketch": (42, 160000, 400, 1, 1),
}


def run_one(cfg):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1803_01982_b200 import _capi
    lib = _capi.load()
    ctx = _capi.context(0)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    out = {}
    for name, (M, N, K, akc, bkc) in SHAPES.items():
        A = torch.randn(M * K, dtype=torch.float64, device="cuda")
        B = torch.randn(K * N, dtype=torch.float64, device="cuda")
        Cm = torch.zeros(M * N, dtype=torch.float64, device="cuda")
        lda = K if akc else M
        ldb = K if bkc else N

        def go():
            rc = lib.ffb_gemm(ctx, C.c_void_p(st.cuda_stream), M, N, K, 1.0, C.c_void_p(A.data_ptr()),
                              lda, akc, C.c_void_p(B.data_ptr()), ldb, bkc, 0.0,
                              C.c_void_p(Cm.data_ptr()), M, C.c_void_p(ws.data_ptr()), ws.numel())
            assert rc == 0
        for _ in range(3):
            go()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            go()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[name] = 2.0 * M * N * K / ms / 1e9 if 2.0 * M * N * K > 1e9 else -1000.0 * ms  # <0: us
    return out


def cublas():
    import torch
    out = {}
    for name, (M, N, K, akc, bkc) in SHAPES.items():
        A = torch.randn(M, K, dtype=torch.float64, device="cuda")
        B = torch.randn(K, N, dtype=torch.float64, device="cuda")
        for _ in range(3):
            A @ B
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            A @ B
        e1.record()
        torch.cuda.synchronize()
        out[name] = 2.0 * M * N * K / (e0.elapsed_time(e1) / 10) / 1e9
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        r = run_one(None)
        print(" ".join(f"{k}={v:.1f}" for k, v in r.items()))
        sys.exit(0)
    cfgs = sys.argv[1:] or ["auto", "0", "1", "2", "3", "4", "5", "6", "7", "8", "9"]
    print("cublas:", " ".join(f"{k}={v:.1f}" for k, v in cublas().items()), flush=True)
    for c in cfgs:
        env = dict(os.environ)
        if c != "auto":
            env["FFB_GEMM_CFG"] = c
        r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
        print(f"cfg {c}:", (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
