"""Drop-in host entry points over the sm_100a engine (C ABI, include/ffb200.h).

Mirrors the reference's Python API for the hot path:

* ``flip_flop_srqr(A, k, l=None, b=32, p=5, epsilon=0.5, g=2.0, d=None, seed=0)``
  — ffsrqr/svd.py:43-98 (same clamp of b, p for small m, same defaults, same
  result type ``ApproxSvd`` with ``meta["srqr"]``/``["params"]``/``["method"]``)
* ``srqr(A, params)`` — ffsrqr/srqr.py:174-210 (``SrqrResult``)
* ``trqrcp(A, params)`` — ffsrqr/sketch.py:150-161 (``PartialFactorization``)
* ``rsisvd(A, k, p=5, q=2, seed=0)`` — ffsrqr/svd.py:101-133, the paper's
  randomized subspace-iteration baseline, on the same device kernels

Inputs may be numpy arrays (results come back as numpy, like the reference)
or CUDA float64 torch tensors (results stay on the device).  Errors are the
reference's exception classes.  Differences, all documented in DESIGN.md:
``meta["srqr"].fact.R`` is the true SRQR R (the reference overwrites it
through a NumPy view, svd.py:67-68) and ``meta["diag_L"]`` exposes the
partial-LQ diagonal explicitly.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _capi, flops, rng
from .errors import (CertificationError, DimensionError, EngineUnavailable, NonFiniteInputError,
                     NumericalError, SingularTrailingBlockError)
from .results import (ApproxSvd, PartialFactorization, SketchParams, SrqrCertificate, SrqrResult,
                      WYFactor)

_tls = threading.local()


def _torch():
    try:
        import torch
    except ImportError as e:  # pragma: no cover
        raise EngineUnavailable("torch is required for device memory") from e
    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return torch


def _device(device):
    torch = _torch()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise EngineUnavailable("the B200 engine runs on CUDA devices only")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def _colmajor(torch, rows, cols, device, dtype=None):
    dtype = dtype or torch.float64
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


import os as _os

_STAGE_CHUNK = int(_os.environ.get("FFB_STAGE_CHUNK_MB", "32")) << 20   # bytes per pinned slot
_STAGE_SLOTS = 4
_stage_pool = None
_stage_pool_lock = threading.Lock()


def _copy_pool():
    global _stage_pool
    with _stage_pool_lock:
        if _stage_pool is None:
            import os
            from concurrent.futures import ThreadPoolExecutor

            nw = int(os.environ.get("FFB_STAGE_WORKERS", "0")) or max(2, min(8, (os.cpu_count() or 4) // 2))
            _stage_pool = ThreadPoolExecutor(max_workers=nw,
                                             thread_name_prefix="ffb-h2d")
        return _stage_pool


def _upload_bytes(torch, a, device):
    """Contiguous numpy array -> 1-D float64 CUDA tensor of the same bytes.

    Pageable numpy memory goes through the driver's bounce buffers at ~11 GB/s.
    Instead, a ring of pinned slots per thread is filled by parallel host copies
    (numpy releases the GIL) while the previous slots' DMA runs on the current
    stream, at up to PCIe rate."""
    nbytes = a.nbytes
    dst = torch.empty(nbytes // 8, dtype=torch.float64, device=device)
    if nbytes < 2 * _STAGE_CHUNK:
        dst.copy_(torch.from_numpy(a.reshape(-1)))
        return dst
    st = torch.cuda.current_stream(device)
    _, slots, events, used = _stage_ring(torch, dst.device)
    src = a.reshape(-1)
    pool = _copy_pool()
    nw = pool._max_workers
    per = _STAGE_CHUNK // 8
    for i, off in enumerate(range(0, src.size, per)):
        j = i % _STAGE_SLOTS
        cnt = min(per, src.size - off)
        if used[j]:
            events[j].synchronize()          # the slot's previous DMA has drained
        hv = slots[j].numpy()
        part = (cnt + nw - 1) // nw
        futs = [pool.submit(np.copyto, hv[q:min(cnt, q + part)], src[off + q:off + min(cnt, q + part)])
                for q in range(0, cnt, part)]
        for f in futs:
            f.result()
        dst[off:off + cnt].copy_(slots[j][:cnt], non_blocking=True)
        events[j].record(st)
        used[j] = True
    return dst


def _stage_ring(torch, device):
    ring = getattr(_tls, "stage", None)
    if ring is None or ring[0] != device:
        ring = _tls.stage = (
            device,
            [torch.empty(_STAGE_CHUNK // 8, dtype=torch.float64, pin_memory=True) for _ in range(_STAGE_SLOTS)],
            [torch.cuda.Event() for _ in range(_STAGE_SLOTS)],
            [False] * _STAGE_SLOTS)
    return ring


def _download(torch, x):
    """CUDA float64 tensor -> numpy array of the same shape and strides kind,
    through the pinned ring (the mirror of _upload_bytes)."""
    if x.numel() * 8 < 2 * _STAGE_CHUNK or x.dtype != torch.float64:
        return _download_many(torch, [x])[0]
    if x.is_contiguous():
        flat, finish = x.reshape(-1), (lambda a: a.reshape(tuple(x.shape)))
    elif x.dim() == 2 and x.t().is_contiguous():
        flat, finish = x.t().reshape(-1), (lambda a: a.reshape(tuple(x.shape[::-1])).T)
    else:
        return x.detach().cpu().numpy()
    st = torch.cuda.current_stream(x.device)
    _, slots, events, used = _stage_ring(torch, x.device)
    out = np.empty(flat.numel())
    pool = _copy_pool()
    nw = pool._max_workers
    per = _STAGE_CHUNK // 8
    offs = list(range(0, flat.numel(), per))

    def issue(i):
        j = i % _STAGE_SLOTS
        if used[j]:
            st.wait_event(events[j])
        cnt = min(per, flat.numel() - offs[i])
        slots[j][:cnt].copy_(flat[offs[i]:offs[i] + cnt], non_blocking=True)
        events[j].record(st)
        used[j] = True

    for i in range(min(_STAGE_SLOTS, len(offs))):
        issue(i)
    for i, off in enumerate(offs):
        j = i % _STAGE_SLOTS
        cnt = min(per, flat.numel() - off)
        events[j].synchronize()
        hv = slots[j].numpy()
        part = (cnt + nw - 1) // nw
        futs = [pool.submit(np.copyto, out[off + q:off + min(cnt, q + part)], hv[q:min(cnt, q + part)])
                for q in range(0, cnt, part)]
        for f in futs:
            f.result()
        if i + _STAGE_SLOTS < len(offs):
            issue(i + _STAGE_SLOTS)
    return finish(out)


def _download_many(torch, xs):
    """CUDA tensors -> numpy arrays with ONE stream synchronisation: every tensor
    of 64 KB or more is copied into pinned host memory of the same strides
    (a plain DMA at PCIe rate; `.cpu()` into pageable memory moved the 16.8 MB
    u and v of cfg2 at ~2.5 GB/s, 16 ms per call) and returned as the numpy view
    of that pinned block, which goes back to torch's host cache when the array is
    collected.  Small tensors take `.cpu()`."""
    outs, pending = [None] * len(xs), False
    for i, x in enumerate(xs):
        if x is None:
            continue
        x = x.detach()
        dense = x.is_contiguous() or (x.dim() == 2 and x.t().is_contiguous())
        if x.is_cuda and dense and x.numel() * x.element_size() >= (64 << 10):
            p = torch.empty_like(x, device="cpu", pin_memory=True)
            if p.stride() == x.stride():
                p.copy_(x, non_blocking=True)
                outs[i] = p
                pending = True
                continue
        outs[i] = x.cpu()
    if pending:
        torch.cuda.current_stream(next(x.device for x in xs if x is not None and x.is_cuda)).synchronize()
    return [None if o is None else o.numpy() for o in outs]


def _to_device(A, device):
    """(device float64 tensor, is_numpy_input, layout, ld): A in HBM in the
    caller's storage order.  Column-major (F-ordered numpy, torch views with unit
    row stride) runs as FFB_LAYOUT_COL, row-major (C-ordered numpy, contiguous
    torch) as FFB_LAYOUT_ROW — read in place by the engine, never transposed."""
    torch = _torch()
    if isinstance(A, torch.Tensor):
        if A.dim() != 2:
            raise DimensionError("expected a 2-D matrix")
        A = A.to(device=device, dtype=torch.float64)
        m, n = A.shape
        if A.stride(0) == 1 and A.stride(1) >= max(m, 1):
            return A, False, _capi.FFB_LAYOUT_COL, A.stride(1)
        if A.stride(1) == 1 and A.stride(0) >= max(n, 1):
            return A, False, _capi.FFB_LAYOUT_ROW, A.stride(0)
        A = A.contiguous()
        return A, False, _capi.FFB_LAYOUT_ROW, max(n, 1)
    a = np.asarray(A, dtype=float)
    if a.ndim != 2:
        raise DimensionError("expected a 2-D matrix")
    m, n = a.shape
    if a.flags.f_contiguous and not a.flags.c_contiguous:
        t = _upload_bytes(torch, a.T, device).view(n, m)     # (n, m) row-major == A column-major
        return t.t(), True, _capi.FFB_LAYOUT_COL, max(m, 1)
    t = _upload_bytes(torch, np.ascontiguousarray(a), device).view(m, n)
    return t, True, _capi.FFB_LAYOUT_ROW, max(n, 1)


def _workspace(torch, device, nbytes):
    """Engine workspace per (thread, device, stream): the engine writes it
    asynchronously, so work queued on two streams must not share one."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(int(nbytes * 1.1) + 4096, dtype=torch.uint8, device=device)
        cache[key] = buf
    return buf


_omega_cache = {}
_omega_lock = threading.Lock()
_OMEGA_CACHE_MAX = 256              # entries
_OMEGA_CACHE_BYTES = 1 << 30        # and bytes of device memory


_omega_inflight = {}


def _omega(torch, dev, s, m, seed):
    """Device copy of Omega = gaussian(s, m, seed, 0) (ffsrqr/sketch.py:108).

    Omega depends only on (seed, s, m), so repeated factorizations with the same
    seed (IALM/SVT iterations, HOSVD modes of equal size, benchmarks) reuse it.
    A key another thread is generating right now is waited for, not redone."""
    key = (dev.index, int(s), int(m), int(seed) & 0xFFFFFFFFFFFFFFFF)
    while True:
        with _omega_lock:
            om = _omega_cache.get(key)
            if om is not None:
                return om
            ev = _omega_inflight.get(key)
            if ev is None:
                ev = _omega_inflight[key] = threading.Event()
                break
        ev.wait()
    try:
        om = torch.from_numpy(rng.gaussian(s, m, seed, rng.STREAM_SKETCH)).to(dev)
        with _omega_lock:
            while _omega_cache and (len(_omega_cache) >= _OMEGA_CACHE_MAX or
                                    sum(v.numel() * 8 for v in _omega_cache.values()) + om.numel() * 8
                                    > _OMEGA_CACHE_BYTES):
                _omega_cache.pop(next(iter(_omega_cache)))
            _omega_cache[key] = om
    finally:
        with _omega_lock:
            _omega_inflight.pop(key, None)
        ev.set()
    return om


_prefetch_pool = None


def prefetch_omega_async(keys, device=None, threads=8):
    """Start generating Omega for (s, m, seed) keys on background host threads
    (in order) and return at once; a factorization that needs one of them waits
    for it.  Overlaps the host RNG of a batch with the device work of its first
    problems."""
    global _prefetch_pool
    import torch
    from concurrent.futures import ThreadPoolExecutor

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with _omega_lock:
        if _prefetch_pool is None or _prefetch_pool._max_workers < threads:
            _prefetch_pool = ThreadPoolExecutor(max_workers=max(1, threads), thread_name_prefix="ffb-omega")
        pool = _prefetch_pool

    def gen(k):
        with torch.cuda.device(dev):
            return _omega(torch, dev, k[0], k[1], k[2])
    return [pool.submit(gen, k) for k in keys]


def clear_omega_cache():
    """Drop every cached sketch matrix (the next call regenerates its Omega)."""
    with _omega_lock:
        _omega_cache.clear()
        _rs_omega_cache.clear()


def prefetch_omega(keys, device=None, threads=8):
    """Generate and cache Omega for many (s, m, seed) on host threads in parallel
    (numpy's Philox releases the GIL), e.g. before a batch of independent problems."""
    import torch
    from concurrent.futures import ThreadPoolExecutor

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        list(ex.map(lambda k: _omega(torch, dev, k[0], k[1], k[2]), keys))


@_capi.GAUSS_CB
def _gauss_cb(user, seed, stream, rows, cols, out):
    try:
        arr = np.ctypeslib.as_array(out, shape=(int(rows) * int(cols),))
        arr[:] = rng.gaussian(int(rows), int(cols), int(seed), int(stream)).ravel()
        return 0
    except Exception:  # pragma: no cover - surfaced as FFB_ERR_ARGUMENT
        return 1


def run(A, params: SketchParams, mode, device=None, trace_gaps=False):
    """Run one factorization mode through the C ABI; returns a dict of outputs."""
    torch = _torch()
    dev = _device(device if device is not None else (A.device if isinstance(A, torch.Tensor) and A.is_cuda else None))
    with torch.cuda.device(dev):
        if not (isinstance(A, torch.Tensor) and A.is_cuda) and len(getattr(A, "shape", ())) == 2:
            # host input: generate Omega on a host thread while A uploads
            m0, n0 = A.shape
            p0 = params.resolve(m0, n0)
            prefetch_omega_async([(p0.b + p0.p, m0, p0.seed)], device=dev, threads=2)
        Ad, is_np, layout, lda = _to_device(A, dev)
        m, n = Ad.shape
        prm = params.resolve(m, n)
        if mode != _capi.FFB_MODE_TRQRCP and prm.l + 1 > min(m, n):
            raise DimensionError(f"srqr needs l+1 <= min(m,n); got l={prm.l}, min={min(m, n)}")
        if prm.b + prm.p > 512:
            raise DimensionError("the B200 engine supports sketch sizes b + p <= 512")
        lib = _capi.load()
        ctx = _capi.context(dev.index)
        cp = _capi.Params(prm.k, prm.l, prm.b, prm.p, prm.d, prm.epsilon, prm.g,
                          int(prm.seed) & 0xFFFFFFFFFFFFFFFF)
        nbytes = C.c_size_t()
        rc = lib.ffb_workspace_query(m, n, C.byref(cp), mode, C.byref(nbytes))
        if rc != _capi.FFB_OK:
            raise DimensionError("invalid dimensions for the engine")
        ws = _workspace(torch, dev, nbytes.value)
        s = prm.b + prm.p
        omega = _omega(torch, dev, s, m, prm.seed)
        l, k = prm.l, prm.k
        out = {}
        res = _capi.Result()
        if mode == _capi.FFB_MODE_FLIPFLOP:
            out["u"] = _colmajor(torch, m, k, dev)
            out["s"] = torch.empty(k, dtype=torch.float64, device=dev)
            out["v"] = _colmajor(torch, n, k, dev)
            out["diag_L"] = torch.empty(l, dtype=torch.float64, device=dev)
            out["sv_all"] = torch.empty(l, dtype=torch.float64, device=dev)
            res.u, res.ldu = out["u"].data_ptr(), m
            res.s = out["s"].data_ptr()
            res.v, res.ldv = out["v"].data_ptr(), n
            res.diag_L = out["diag_L"].data_ptr()
            res.sv_all = out["sv_all"].data_ptr()
        out["perm"] = torch.empty(n, dtype=torch.int64, device=dev)
        res.perm = out["perm"].data_ptr()
        out["R"] = _colmajor(torch, l, n, dev)
        res.R, res.ldr = out["R"].data_ptr(), l
        if trace_gaps:
            # top-2 relative gap of every sketch pivot step (near-tie certification)
            out["pivot_gap"] = torch.empty(l, dtype=torch.float64, device=dev)
            res.pivot_gap = out["pivot_gap"].data_ptr()
        if mode == _capi.FFB_MODE_TRQRCP:
            out["Y"] = _colmajor(torch, m, l, dev)
            out["T"] = _colmajor(torch, l, l, dev)
            out["B"] = _colmajor(torch, s, n, dev)
            res.Y, res.ldy = out["Y"].data_ptr(), m
            res.T, res.ldt = out["T"].data_ptr(), l
            res.B, res.ldb = out["B"].data_ptr(), s
        else:
            out["Q"] = _colmajor(torch, m, l + 1, dev)
            out["rtilde"] = _colmajor(torch, l + 1, l + 1, dev)
            res.Q, res.ldq = out["Q"].data_ptr(), m
            res.rtilde = out["rtilde"].data_ptr()
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = lib.ffb_run(ctx, C.c_void_p(stream), mode, C.c_void_p(Ad.data_ptr()), m, n,
                         lda, layout, C.byref(cp), C.c_void_p(omega.data_ptr()), _gauss_cb, None,
                         C.c_void_p(ws.data_ptr()), ws.numel(), C.byref(res))
        out.update(alpha=res.alpha, g1=res.g1, g2=res.g2, tau=res.tau_bound,
                   tau_hat=res.tau_hat_bound, r22=res.r22, swaps=int(res.swaps),
                   flops=int(res.flops), kernels=int(res.kernels),
                   status_bits=int(res.status_bits), svd_sweeps=int(res.svd_sweeps),
                   i_offs=[int(res.i_off_trace[i]) for i in range(min(int(res.swaps), 64))],
                   is_numpy=is_np, params=prm, m=m, n=n)
        if rc == _capi.FFB_OK:
            return out
        msg = _capi.last_error(ctx)
        if rc == _capi.FFB_ERR_DIMENSION:
            raise DimensionError(msg)
        if rc == _capi.FFB_ERR_SINGULAR_TRAILING:
            raise SingularTrailingBlockError(msg)
        if rc == _capi.FFB_ERR_CERTIFICATION:
            raise CertificationError(msg, result=_srqr_result(out))
        if rc == _capi.FFB_ERR_NUMERICAL:
            if out["status_bits"] & 1:          # kStNonFinite: NaN / Inf in A or a factor
                raise NonFiniteInputError(msg)
            raise NumericalError(msg)
        raise RuntimeError(f"ffb_run failed ({rc}): {msg}")


def _conv(x, as_np):
    if not as_np:
        return x
    return _download(_torch(), x)


def _srqr_result(out):
    np_ = out["is_numpy"]
    prm = out["params"]
    l = prm.l
    Q = out["Q"]
    # numpy callers get numpy R / Q / R-tilde on first access (results._HostOnAccess)
    fact = PartialFactorization(R=out["R"], perm=_conv(out["perm"], np_), k=l, q_dense=Q[:, :l])
    fact._host = np_
    cert = SrqrCertificate(alpha=abs(out["alpha"]), g1=out["g1"], g2=out["g2"],
                           swaps=out["swaps"], tau_bound=out["tau"],
                           tau_hat_bound=out["tau_hat"])
    res = SrqrResult(fact=fact, cert=cert, r22_norm_estimate=out["r22"], rtilde=out["rtilde"], q_ext=Q)
    res._host = np_
    return res


def flip_flop_srqr(A, k, l=None, b=32, p=5, epsilon=0.5, g=2.0, d=None, seed=0, device=None,
                   trace_gaps=False):
    """Rank-k approximate SVD via spectrum-revealing QR plus a flipped QR
    (ffsrqr/svd.py:43-98), on the B200 engine."""
    shape = tuple(A.shape)
    if len(shape) != 2:
        raise DimensionError("expected a 2-D matrix")
    m, n = shape
    if b + p > m:                       # svd.py:53-55
        b = max(1, m - p)
        p = m - b
    params = SketchParams(k=k, l=l, b=b, p=p, epsilon=epsilon, g=g, d=d, seed=seed)
    out = run(A, params, _capi.FFB_MODE_FLIPFLOP, device=device, trace_gaps=trace_gaps)
    np_ = out["is_numpy"]
    res = _srqr_result(out)
    prm = out["params"]
    # the reference's own tally (ffsrqr/flops.py), replayed from the run's shapes
    # and swap trace; the flops the device executed are meta["device_flops"]
    fc = flops.flip_flop_count(out["m"], out["n"], prm.k, prm.l, prm.b, prm.p, prm.d,
                               out["swaps"], out["i_offs"], out["alpha"] == 0.0)
    meta = {"srqr": res, "params": out["params"], "method": "flip_flop_srqr",
            "device_flops": out["flops"],
            "diag_L": _conv(out["diag_L"], np_), "sv_all": _conv(out["sv_all"], np_),
            "pivot_gap": _conv(out["pivot_gap"], np_) if "pivot_gap" in out else None,
            "engine": "ffb200-sm100a",
            "kernels": out["kernels"], "i_offs": out["i_offs"],
            "svd_sweeps": out["svd_sweeps"],
            # exact zero on an R11 diagonal: the sketch update used a zero inverse row
            # where the reference takes lstsq (sketch.py:75-83); only the order of
            # rank-deficient noise columns can differ
            "zero_pivot": bool(out["status_bits"] & 8)}
    if np_:
        u, sv, v = _download_many(_torch(), [out["u"], out["s"], out["v"]])   # one synchronisation
    else:
        u, sv, v = out["u"], out["s"], out["v"]
    return ApproxSvd(u=u, s=sv, v=v, flop_count=fc, meta=meta)


def srqr(A, params: SketchParams, device=None):
    """Spectrum-revealing QR to params.l steps (ffsrqr/srqr.py:174-210)."""
    out = run(A, params, _capi.FFB_MODE_SRQR, device=device)
    return _srqr_result(out)


def trqrcp(A, params: SketchParams, device=None):
    """Truncated randomized QRCP (ffsrqr/sketch.py:150-161)."""
    out = run(A, params, _capi.FFB_MODE_TRQRCP, device=device, trace_gaps=True)
    np_ = out["is_numpy"]
    prm = out["params"]
    fact = PartialFactorization(R=_conv(out["R"], np_), perm=_conv(out["perm"], np_), k=prm.l,
                                wy=WYFactor(_conv(out["Y"], np_), _conv(out["T"], np_)))
    fact.sketch = _conv(out["B"], np_)
    fact.pivot_gap = _conv(out["pivot_gap"], np_) if "pivot_gap" in out else None
    return fact


_rs_omega_cache = {}


def rsisvd(A, k, p=5, q=2, seed=0, device=None):
    """Randomized subspace-iteration SVD baseline (ffsrqr/svd.py:101-133) on the
    B200 engine: Omega = gaussian(n, r, seed, 2_000_000) from the reference RNG,
    then ffb_rsisvd (GEMMs on FP64 DMMA, Householder panel QRs, Jacobi SVD)."""
    torch = _torch()
    shape = tuple(A.shape)
    if len(shape) != 2:
        raise DimensionError("expected a 2-D matrix")
    m, n = shape
    if not 1 <= k <= min(m, n):
        raise DimensionError(f"rsisvd needs 1 <= k <= min(m,n); got k={k}")
    if p < 0 or q < 0:
        raise DimensionError("rsisvd needs p >= 0 and q >= 0")
    r = min(k + p, min(m, n))
    dev = _device(device if device is not None else (A.device if isinstance(A, torch.Tensor) and A.is_cuda else None))
    with torch.cuda.device(dev):
        Ad, is_np, layout, lda = _to_device(A, dev)
        lib = _capi.load()
        ctx = _capi.context(dev.index)
        nbytes = C.c_size_t()
        rc = lib.ffb_rsisvd_workspace_query(m, n, k, r, C.byref(nbytes))
        if rc != _capi.FFB_OK:
            raise DimensionError("invalid dimensions for the engine")
        ws = _workspace(torch, dev, nbytes.value)
        key = (dev.index, n, r, int(seed) & 0xFFFFFFFFFFFFFFFF)
        with _omega_lock:
            om = _rs_omega_cache.get(key)
        if om is None:
            om = torch.from_numpy(rng.gaussian(n, r, seed, rng.STREAM_RSISVD)).to(dev)
            with _omega_lock:
                if len(_rs_omega_cache) > 64:
                    _rs_omega_cache.clear()
                _rs_omega_cache[key] = om
        u = _colmajor(torch, m, k, dev)
        s = torch.empty(k, dtype=torch.float64, device=dev)
        v = _colmajor(torch, n, k, dev)
        fl = C.c_int64(0)
        sw = C.c_int32(0)
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = lib.ffb_rsisvd(ctx, C.c_void_p(stream), C.c_void_p(Ad.data_ptr()), m, n, lda, layout,
                            k, r, q, C.c_void_p(om.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(),
                            C.c_void_p(u.data_ptr()), m, C.c_void_p(s.data_ptr()),
                            C.c_void_p(v.data_ptr()), n, C.byref(fl), C.byref(sw))
        if rc != _capi.FFB_OK:
            msg = _capi.last_error(ctx)
            if rc == _capi.FFB_ERR_DIMENSION:
                raise DimensionError(msg)
            if rc == _capi.FFB_ERR_NUMERICAL:
                raise NumericalError(msg)
            raise RuntimeError(f"ffb_rsisvd failed ({rc}): {msg}")
        meta = {"method": "rsisvd", "q": q, "p": p, "engine": "ffb200-sm100a",
                "svd_sweeps": int(sw.value), "device_flops": int(fl.value)}
        return ApproxSvd(u=_conv(u, is_np), s=_conv(s, is_np), v=_conv(v, is_np),
                         flop_count=flops.rsisvd_count(m, n, k, r, q), meta=meta)
