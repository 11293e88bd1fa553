"""Device dense helpers over the C ABI: the FP64 DMMA GEMM (``ffb_gemm``) on
torch CUDA views of any 2-D layout, plus the deterministic sum of squares.

Layout rule of ``ffb_gemm`` (include/ffb200.h): an operand is either
column-major (``*_kc = 0`` for A / ``1`` for B) or row-major (the other
flag), with its leading dimension; C is column-major.  torch views with unit
stride in one dimension map onto one of the two without a copy.
"""
from __future__ import annotations

import ctypes as C
import threading

from . import _capi

_tls = threading.local()
_WS_BYTES = (65536 * 4) + (32 << 20)   # stream-K counters + split-K partials


def _ws(torch, dev, stream):
    """Split-K scratch per (thread, device, stream): ffb_gemm is asynchronous and
    writes its partials without a sync, so two streams must never share one."""
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    key = (dev.index, stream)
    buf = cache.get(key)
    if buf is None:
        buf = torch.empty(_WS_BYTES, dtype=torch.uint8, device=dev)
        cache[key] = buf
    return buf


def _layout(t, rows, cols):
    """('col'|'row', ld) for a 2-D view, or None when neither stride is 1."""
    s0, s1 = t.stride()
    if rows <= 1 and cols <= 1:
        return "col", max(rows, 1)
    if s0 == 1 or rows == 1:
        ld = s1 if cols > 1 else max(rows, 1)
        if ld >= max(rows, 1):
            return "col", ld
    if s1 == 1 or cols == 1:
        ld = s0 if rows > 1 else max(cols, 1)
        if ld >= max(cols, 1):
            return "row", ld
    return None


def colmajor(torch, rows, cols, dev):
    return torch.empty((cols, rows), dtype=torch.float64, device=dev).t()


def gemm(A, B, out=None, alpha=1.0, beta=0.0):
    """out = alpha * A @ B + beta * out on the engine's DMMA GEMM (no cuBLAS).

    A (M x K) and B (K x N) are float64 CUDA views of any unit-stride layout;
    out (M x N) is column-major (allocated when None)."""
    import torch

    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError(f"gemm shape mismatch {tuple(A.shape)} @ {tuple(B.shape)}")
    dev = A.device
    la = _layout(A, M, K)
    if la is None:
        A = A.contiguous()
        la = _layout(A, M, K)
    lb = _layout(B, K, N)
    if lb is None:
        B = B.contiguous()
        lb = _layout(B, K, N)
    if out is None:
        out = colmajor(torch, M, N, dev)
        beta = 0.0
    lc = _layout(out, M, N)
    if lc is None or lc[0] != "col":
        raise ValueError("gemm output must be column-major")
    if M == 0 or N == 0:
        return out
    if K == 0:
        out.mul_(beta)
        return out
    lib = _capi.load()
    ctx = _capi.context(dev.index)
    a_kc = 1 if la[0] == "row" else 0      # row-major A: A(i,k) = A[k + i*lda]
    b_kc = 1 if lb[0] == "col" else 0      # col-major B: B(k,j) = B[k + j*ldb]
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = _ws(torch, dev, stream)
        rc = lib.ffb_gemm(ctx, C.c_void_p(stream), M, N, K, float(alpha), C.c_void_p(A.data_ptr()),
                          la[1], a_kc, C.c_void_p(B.data_ptr()), lb[1], b_kc, float(beta),
                          C.c_void_p(out.data_ptr()), lc[1], C.c_void_p(ws.data_ptr()), ws.numel())
    if rc != _capi.FFB_OK:
        raise RuntimeError(f"ffb_gemm failed ({rc}): {_capi.last_error(ctx)}")
    return out


def sumsq(x):
    """Deterministic sum of squares of a contiguous float64 CUDA tensor (ffb_sumsq)."""
    import torch

    x = x.contiguous()
    lib = _capi.load()
    part = torch.empty(lib.ffb_svt_partials(), dtype=torch.float64, device=x.device)
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
        stream = torch.cuda.current_stream(x.device).cuda_stream
        rc = lib.ffb_sumsq(C.c_void_p(stream), C.c_void_p(x.data_ptr()), x.numel(),
                           C.c_void_p(part.data_ptr()), C.c_void_p(out.data_ptr()))
    if rc != _capi.FFB_OK:
        raise RuntimeError(f"ffb_sumsq failed ({rc})")
    return out


def spectral_norm(M, tol=1e-15, max_iter=5000, seed=1234):
    """||M||_2 by power iteration on M^T M with the engine GEMM (the reference
    takes numpy.linalg.svd(M)[0], nuclear.py:116,161).  Stops when the estimate
    changes by < tol relatively for 3 consecutive steps."""
    import numpy as np
    import torch

    m, n = M.shape
    g = np.random.default_rng(seed)
    v = torch.as_tensor(g.standard_normal((n, 1)), device=M.device)
    v = v / torch.linalg.vector_norm(v)
    prev, calm = 0.0, 0
    est = 0.0
    for _ in range(max_iter):
        u = gemm(M, v)
        w = gemm(M.t(), u)
        nw = float(torch.linalg.vector_norm(w))
        if nw == 0.0:
            return 0.0
        est = nw ** 0.5
        v = w / nw
        calm = calm + 1 if abs(est - prev) <= tol * est else 0
        if calm >= 3:
            break
        prev = est
    return est


def small_svd(M):
    """(U, sig, V) of a square float64 CUDA matrix via the engine's one-sided
    block Jacobi (ffb_small_svd): the device replacement for the dgesdd of the
    flip-flop tail (ffsrqr/svd.py:79).  sig descending; M = U diag(sig) V^T."""
    import torch

    from .errors import DimensionError, NumericalError

    l, l2 = M.shape
    if l != l2:
        raise DimensionError("small_svd expects a square matrix")
    dev = M.device
    if not (M.stride(0) == 1 and M.stride(1) >= l):
        M = M.t().contiguous().t()
    lib = _capi.load()
    ctx = _capi.context(dev.index)
    nb = C.c_size_t()
    if lib.ffb_small_svd_workspace_query(l, C.byref(nb)) != _capi.FFB_OK:
        raise DimensionError("invalid size")
    ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    U = colmajor(torch, l, l, dev)
    V = colmajor(torch, l, l, dev)
    sig = torch.empty(l, dtype=torch.float64, device=dev)
    sw = C.c_int32(0)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = lib.ffb_small_svd(ctx, C.c_void_p(stream), C.c_void_p(M.data_ptr()), l, M.stride(1),
                               C.c_void_p(sig.data_ptr()), C.c_void_p(U.data_ptr()), l,
                               C.c_void_p(V.data_ptr()), l, C.c_void_p(ws.data_ptr()), ws.numel(),
                               C.byref(sw))
    if rc == _capi.FFB_ERR_NUMERICAL:
        raise NumericalError(_capi.last_error(ctx))
    if rc != _capi.FFB_OK:
        raise RuntimeError(f"ffb_small_svd failed ({rc}): {_capi.last_error(ctx)}")
    return U, sig, V, int(sw.value)
