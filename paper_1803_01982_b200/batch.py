"""Batched and multi-GPU drivers (BASELINE configs 4 and 5).

One GPU: independent factorizations run concurrently on several CUDA streams,
one host thread and one workspace per stream (the C ABI releases the GIL, so
host threads overlap).  Several GPUs (one process per GPU, torchrun): problems
are partitioned contiguously — rank r takes [n*r/W, n*(r+1)/W) — and each rank
factorizes its share with no data-path collective; the only communication is
an NCCL gather of fixed-size result slots to rank 0.
"""
from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

from . import _capi


def partition(n_problems, world, rank):
    """Contiguous share of rank `rank`: range(lo, hi)."""
    lo = (n_problems * rank) // world
    hi = (n_problems * (rank + 1)) // world
    return range(lo, hi)


_pools = {}
_pools_lock = threading.Lock()


def _pool(dev, n_streams):
    """Persistent (streams, host threads) per device and width: the engine keeps
    its workspace and pinned staging per host thread, so reusing the threads keeps
    cudaMalloc / cudaMallocHost (both synchronising) out of every later batch."""
    import torch

    key = (dev.index, n_streams)
    with _pools_lock:
        ent = _pools.get(key)
        if ent is None:
            streams = [torch.cuda.Stream(device=dev) for _ in range(n_streams)]
            ent = (streams, ThreadPoolExecutor(max_workers=n_streams), threading.Lock(),
                   list(range(n_streams)))
            _pools[key] = ent
        return ent


def sm_budget(dev, n_streams):
    """SMs per in-flight problem when `n_streams` problems share the device."""
    import torch

    import os

    if n_streams <= 1:
        return 0
    env = os.environ.get("FFB_SM_BUDGET")
    if env is not None:            # explicit per-problem SM budget (0 = whole device)
        return max(0, int(env))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    return max(8, sms // n_streams)


def run_streams(problems, solve, n_streams=4, device=None, budget="auto"):
    """Run `solve(problem)` for every problem on `n_streams` CUDA streams.

    `solve` is called inside `torch.cuda.stream(s)`; results keep input order.
    budget: SMs each problem's grid-synchronised kernels may use
    (ffb_set_thread_sm_budget); "auto" = SMs / n_streams, 0 = the whole device.
    """
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    streams, ex, lock, free = _pool(dev, max(1, n_streams))
    nb = sm_budget(dev, n_streams) if budget == "auto" else int(budget)
    lib = _capi.load()

    def _one(p):
        with lock:
            sid = free.pop()
        lib.ffb_set_thread_sm_budget(nb)
        try:
            with torch.cuda.device(dev), torch.cuda.stream(streams[sid]):
                out = solve(p)
                streams[sid].synchronize()
                return out
        finally:
            with lock:
                free.append(sid)

    return list(ex.map(_one, problems))


def run_host_pipeline(host_inputs, solve, n_streams=3, prefetch=2, device=None, budget="auto"):
    """Host-resident inputs -> `solve(i, device_tensor)` on `n_streams` compute streams,
    with every upload issued ahead by one copy thread on its own stream.

    With uploads inside each call (``run_streams``), a stream's next upload waits
    for its previous factorization, so the copy engine idles whenever all streams
    compute.  Here the copy engine runs back to back, at most
    ``n_streams + prefetch`` inputs resident on the device at a time.  Inputs
    should be pinned CPU tensors (any strides; the device copy keeps them).
    Results keep input order.  budget: as in run_streams.
    """
    import queue

    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    streams, ex, lock, free = _pool(dev, max(1, n_streams))
    nb = sm_budget(dev, n_streams) if budget == "auto" else int(budget)
    lib = _capi.load()
    key = (dev.index, "copy")
    with _pools_lock:
        if key not in _pools:
            _pools[key] = torch.cuda.Stream(device=dev)
        cst = _pools[key]
    q = queue.Queue(maxsize=max(1, n_streams + prefetch))
    err = []

    def _uploader():
        try:
            with torch.cuda.device(dev), torch.cuda.stream(cst):
                for i, h in enumerate(host_inputs):
                    d = torch.empty_strided(tuple(h.shape), tuple(h.stride()), dtype=h.dtype, device=dev)
                    d.copy_(h, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cst)
                    q.put((i, d, ev))
        except BaseException as e:   # surfaced by the consumers
            err.append(e)
            q.put(None)

    up = threading.Thread(target=_uploader, name="ffb-uploader", daemon=True)
    up.start()

    def _one(_):
        item = q.get()
        if item is None:
            q.put(None)
            raise RuntimeError("upload failed") from (err[0] if err else None)
        i, d, ev = item
        with lock:
            sid = free.pop()
        lib.ffb_set_thread_sm_budget(nb)
        try:
            s_ = streams[sid]
            with torch.cuda.device(dev), torch.cuda.stream(s_):
                s_.wait_event(ev)
                d.record_stream(s_)
                out = solve(i, d)
                s_.synchronize()
                return i, out
        finally:
            with lock:
                free.append(sid)

    res = list(ex.map(_one, range(len(host_inputs))))
    up.join()
    if err:
        raise err[0]
    res.sort(key=lambda t: t[0])
    return [r for _, r in res]


def gather_slots(local_slots, n_problems, slot_shape, rank, world, device, dtype=None):
    """Gather fixed-size per-problem result slots to rank 0.

    local_slots: tensor (len(partition(...)), *slot_shape) on `device`.
    Returns the (n_problems, *slot_shape) tensor on rank 0, None elsewhere.
    Uses torch.distributed.gather (NCCL over NVLink on GPUs, gloo on CPU).
    """
    import torch
    import torch.distributed as dist

    dtype = dtype or local_slots.dtype
    shares = [len(partition(n_problems, world, r)) for r in range(world)]
    pad = max(shares)
    buf = torch.zeros((pad,) + tuple(slot_shape), dtype=dtype, device=device)
    buf[: local_slots.shape[0]] = local_slots
    if world == 1:
        return buf[: shares[0]]
    if dist.get_backend() == "nccl":
        # NCCL has no gather: all_gather into a flat buffer (rank 0 keeps it)
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf)
    else:
        out = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, out, dst=0)
    if rank != 0:
        return None
    return torch.cat([o[:s] for o, s in zip(out, shares)], dim=0)


def flip_flop_batch(make_problem, n_problems, k, l, b, p, seed_of=lambda i: i, n_streams=4,
                    gather=("u", "s"), solve=None):
    """Factorize `n_problems` independent matrices across all ranks.

    make_problem(i) -> device matrix for problem i (generated where it is used;
    A never crosses GPUs).  Returns (results_local, gathered) where gathered maps
    each name in `gather` to the stacked (n_problems, ...) tensor on rank 0.
    """
    import torch
    import torch.distributed as dist

    from .engine import flip_flop_srqr

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    mine = list(partition(n_problems, world, rank))
    solve = solve or (lambda i: flip_flop_srqr(make_problem(i), k, l=l, b=b, p=p, seed=seed_of(i)))
    results = run_streams(mine, solve, n_streams=n_streams) if torch.cuda.is_available() else [solve(i) for i in mine]
    gathered = {}
    for name in gather:
        parts = [getattr(r, name) for r in results]
        parts = [x if isinstance(x, torch.Tensor) else torch.as_tensor(x) for x in parts]
        dev = parts[0].device if parts else (torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
        local = torch.stack(parts) if parts else torch.zeros((0,))
        shape = tuple(local.shape[1:])
        gathered[name] = gather_slots(local, n_problems, shape, rank, world, dev)
    return results, gathered


class NativeBatch:
    """Many independent flip-flop factorizations through one ``ffb_run_batched``
    call: C++ worker threads (the GIL is released for the whole batch), one
    stream, workspace and set of output buffers per problem, allocated once and
    reused by every ``run``.  Replaces the reference's Python loop over
    independent problems (ffsrqr/tensor.py:112-115) without per-problem host work.

    problems: list of CUDA float64 matrices (column- or row-major), all with the
    same k, l, b, p.  seeds: per-problem seed (Omega and g2 streams).
    """

    def __init__(self, problems, k, l, b, p, seeds, d=None, g=2.0, device=None, threads=8):
        import ctypes as C

        import torch

        from . import engine
        from .results import SketchParams

        self.torch = torch
        self.lib = _capi.load()
        dev = torch.device(device) if device is not None else problems[0].device
        self.dev = dev
        self.ctx = _capi.context(dev.index)
        self.threads = max(1, int(threads))
        self.seeds = [int(s) for s in seeds]
        n_prob = len(problems)
        self.items = (_capi.BatchItem * n_prob)()
        self.results = [_capi.Result() for _ in range(n_prob)]
        self.out = []
        self.keep = []
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(n_prob)]
        self.prm = []
        for i, A in enumerate(problems):
            Ad, _, layout, lda = engine._to_device(A, dev)
            m, n = Ad.shape
            sp = SketchParams(k=k, l=l, b=b, p=p, d=d, g=g, seed=self.seeds[i]).resolve(m, n)
            prm = _capi.Params(sp.k, sp.l, sp.b, sp.p, sp.d, sp.epsilon, sp.g,
                               int(sp.seed) & 0xFFFFFFFFFFFFFFFF)
            nb = C.c_size_t()
            rc = self.lib.ffb_workspace_query(m, n, C.byref(prm), _capi.FFB_MODE_FLIPFLOP, C.byref(nb))
            if rc != _capi.FFB_OK:
                from .errors import DimensionError

                raise DimensionError("invalid dimensions for the engine")
            ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
            o = {"u": torch.empty((sp.k, m), dtype=torch.float64, device=dev).t(),
                 "s": torch.empty(sp.k, dtype=torch.float64, device=dev),
                 "v": torch.empty((sp.k, n), dtype=torch.float64, device=dev).t(),
                 "perm": torch.empty(n, dtype=torch.int64, device=dev)}
            res = self.results[i]
            res.u, res.ldu = o["u"].data_ptr(), m
            res.s = o["s"].data_ptr()
            res.v, res.ldv = o["v"].data_ptr(), n
            res.perm = o["perm"].data_ptr()
            it = self.items[i]
            it.stream, it.mode, it.A, it.m, it.n, it.lda = (self.streams[i].cuda_stream, _capi.FFB_MODE_FLIPFLOP,
                                                            Ad.data_ptr(), m, n, lda)
            it.a_layout = layout
            it.prm, it.workspace, it.workspace_bytes = prm, ws.data_ptr(), ws.numel()
            it.out = C.pointer(res)
            self.out.append(o)
            self.keep.append((Ad, ws))
            self.prm.append(sp)

    def run(self, fresh_omega=False, chunk=16, on_chunk=None, omega_threads=8):
        """Factorize every problem; returns the list of output dicts (device
        tensors u, s, v, perm, plus the certificate scalars).

        fresh_omega: regenerate every problem's Omega on host threads (as each
        reference call does) — in problem order, overlapped with the device
        work of the earlier chunks.  The problems run in chunks of `chunk`
        through ffb_run_batched; on_chunk(lo, hi) is called after each chunk
        (e.g. to start gathering its results while the next chunk computes)."""
        import ctypes as C

        from . import engine

        torch = self.torch
        n = len(self.items)
        keys = [(sp.b + sp.p, self.items[i].m, sp.seed) for i, sp in enumerate(self.prm)]
        if fresh_omega:
            engine.clear_omega_cache()
        futs = engine.prefetch_omega_async(keys, device=self.dev, threads=omega_threads)
        torch.cuda.current_stream(self.dev).synchronize()
        size = C.sizeof(_capi.BatchItem)
        base = C.addressof(self.items)
        self._oms = []
        for lo in range(0, n, max(1, chunk)):
            hi = min(n, lo + max(1, chunk))
            for i in range(lo, hi):
                om = futs[i].result()
                self.items[i].omega = om.data_ptr()
                self._oms.append(om)
            part = (_capi.BatchItem * (hi - lo)).from_address(base + lo * size)
            rc = self.lib.ffb_run_batched(self.ctx, part, hi - lo, self.threads, engine._gauss_cb, None)
            if rc != _capi.FFB_OK:
                raise RuntimeError(f"ffb_run_batched failed ({rc}): {_capi.last_error(self.ctx)}")
            for i in range(lo, hi):
                r = self.results[i]
                self.out[i].update(alpha=r.alpha, g1=r.g1, g2=r.g2, swaps=int(r.swaps), tau=r.tau_bound,
                                   tau_hat=r.tau_hat_bound, r22=r.r22)
            if on_chunk is not None:
                on_chunk(lo, hi)
        return self.out
