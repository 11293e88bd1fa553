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
