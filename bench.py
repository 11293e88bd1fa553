#!/usr/bin/env python
"""Benchmark: rank-k Flip-Flop SRQR factorizations/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl ours|reference]

Default workload = BASELINE.json configs[1] ("cfg2"): one 8192x8192 float64
matrix, k=256, p=16, b=64 (working rank l = k+p = 272), Haar
singular vectors and sigma_i = 10^(-8(i-1)/8191), generated on the device from
a fixed seed (synthetic; no dataset involved).  A step = one full
flip_flop_srqr factorization of the device-resident matrix through the engine
(sketch, TRQRCP, SRQR certificate, partial LQ, A*Qhat, small SVD, back-map).
A (537 MB) exceeds the 126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun, one rank per GPU): every rank factorizes its own matrix
(seed = rank) — weak scaling, no collective on the data path; the per-step
time is the max over ranks (NCCL all-reduce of CUDA-event times).

--impl reference: times the CPU oracle port of the reference algorithm
(oracle/, numpy + OpenBLAS on all host cores) on the same workload, rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.0   # measured DMMA peak on this pool's B200 (profiles/r01_fp64_peak.md)
METRIC = "flip_flop_srqr_factorizations_per_s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def ready(self, timeout=10.0):
        """Block until nvidia-smi delivers its first sample (its start-up can
        outlast a short timed region); returns the index the region starts at."""
        t0 = time.time()
        while self.proc is not None and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.01)
        return len(self.samples)

    def stop(self, since=0):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0 = time.time()   # a region shorter than the 50 ms period: take the next sample
        while len(self.samples) <= since and time.time() - t0 < 1.0:
            time.sleep(0.005)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        region = self.samples[since:]
        sm = [float(s[0]) for s in region if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in region if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in region:
            for i, nm in enumerate(names):
                if len(s) > 3 + i and s[3 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(region)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_workload(name, seed, device):
    from paper_1803_01982_b200 import workloads

    cfg = workloads.CONFIGS[name]
    if name == "cfg4":
        A = workloads.torch_tensor_unfoldings(seed=seed, device=device)[0]
    else:
        A = workloads.torch_matrix(name, seed=seed, device=device)
    return cfg, A


def k13_traffic(workload):
    """DRAM bytes per launch of the roofline kernel from the committed ncu capture
    (profiles/*_k13_ncu.json, `ncu --set full`), or None."""
    import glob

    best, src = None, None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_k13_ncu.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        if d.get("workload") == workload:
            best, src = d, os.path.relpath(path, ROOT)
    if best is None:
        return None, None
    return best["dram_bytes_read"] + best["dram_bytes_write"], src


def run_batched(args):
    """cfg4 / cfg5: independent problems partitioned contiguously over the ranks
    (paper_1803_01982_b200.batch.partition); each rank factorizes its share, then
    the singular values and certificates are gathered to rank 0 (the only
    collective).  Strong scaling: the total number of problems is fixed."""
    import torch
    import torch.distributed as dist

    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import batch, workloads

    ws, rank, local = dist_init()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = workloads.CONFIGS[args.workload]
    mine = list(batch.partition(cfg.batch, ws, rank))
    if args.workload == "cfg4":
        unf = workloads.torch_tensor_unfoldings(seed=0, device=dev)
        probs = {i: unf[i] for i in mine}
        seed_of = lambda i: 0
    else:
        probs = {i: workloads.torch_matrix("cfg5", seed=i, device=dev) for i in mine}
        seed_of = lambda i: i
    m, n = cfg.m, cfg.n
    if args.streams <= 0:
        args.streams = 8 if args.workload == "cfg5" else 1
    # Omega for every local problem, generated on host threads (the reference RNG)
    # before the warm-up; SVT iterations reuse a fixed seed, so steady state
    # sees cached sketches
    from paper_1803_01982_b200 import engine
    engine.prefetch_omega([(cfg.b + cfg.p, m, seed_of(i)) for i in mine], device=dev,
                          threads=min(16, len(os.sched_getaffinity(0))))

    def solve(i):
        return ffb.flip_flop_srqr(probs[i], cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=seed_of(i))

    def step():
        if args.streams > 1:
            res = batch.run_streams(mine, solve, n_streams=args.streams, device=dev)
        else:
            res = [solve(i) for i in mine]
        local_s = torch.stack([r.s for r in res]) if res else torch.zeros((0, cfg.k), dtype=torch.float64, device=dev)
        return batch.gather_slots(local_s, cfg.batch, (cfg.k,), rank, ws, dev)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    i0 = clocks.ready()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        gathered = step()
    e1.record(st)
    torch.cuda.synchronize()
    clk = clocks.stop(i0)
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        flop_alg = ffb.flip_flop_flop_formula(m, n, cfg.l, cfg.b, cfg.p) * cfg.batch
        achieved = flop_alg / (ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": cfg.batch * 1000.0 / ms, "unit": "factorizations/s",
            "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Haar factors / Tucker tensor, BASELINE spectra, device-generated)",
            "config": {"workload": args.workload, "m": m, "n": n, "k": cfg.k, "p": cfg.p, "b": cfg.b,
                       "l": cfg.l, "batch": cfg.batch,
                       "parallelism": f"partitioned x{ws} (contiguous), {args.streams} streams/GPU, "
                                      "NCCL gather of s to rank 0",
                       "l2_flush": "per-problem A %d MB, batch >> L2" % (m * n * 8 // 2**20)},
            "step_roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                              "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                              "flop_alg": flop_alg},
            "clocks": clk,
            "gathered": list(gathered.shape) if gathered is not None else None,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_oracle_sample(A_host, cfg, budget_s=30.0):
    """Time the CPU oracle (reference algorithm port) on the same matrix."""
    import oracle

    t0 = time.perf_counter()
    oracle.flip_flop(A_host, cfg.k, l=cfg.l, b=cfg.b, p=cfg.p, seed=0)
    t = time.perf_counter() - t0
    return t


def run_reference(args):
    ws, rank, local = dist_init()
    if rank != 0:
        return 0
    import torch

    from paper_1803_01982_b200 import workloads

    cfg = workloads.CONFIGS[args.workload]
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    _, A = make_workload(args.workload, 0, dev)
    A_host = np.asfortranarray(A.cpu().numpy())
    del A
    cores = len(os.sched_getaffinity(0))
    warm = min(args.warmup, 1)
    times = []
    for _ in range(warm):
        cpu_oracle_sample(A_host, cfg)
    t_start = time.perf_counter()
    for i in range(max(1, args.steps)):
        times.append(cpu_oracle_sample(A_host, cfg))
        if time.perf_counter() - t_start > args.ref_budget_s:
            break
    t = sum(times) / len(times)
    v = 1.0 / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "factorizations/s",
        "n_gpus": ws, "steps": len(times), "warmup": warm, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Haar factors, BASELINE spectrum)",
        "config": {"workload": args.workload, "m": cfg.m, "n": cfg.n, "k": cfg.k, "p": cfg.p,
                   "b": cfg.b, "l": cfg.l},
        "cpu_baseline": {"value": v, "unit": "factorizations/s", "cores": cores, "kind": "port",
                         "sample": f"{len(times)} full {args.workload} factorization(s) by the "
                                   "numpy oracle port (oracle/ffsrqr_oracle.py), OpenBLAS threads=all"},
        "e2e": {"value": v, "unit": "factorizations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    ap.add_argument("--streams", type=int, default=0,
                    help="batched workloads: problems in flight per GPU (CUDA streams); "
                         "0 = default (cfg5: 8, cfg4: 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload in ("cfg4", "cfg5"):
        return run_batched(args)

    import torch
    import torch.distributed as dist

    import paper_1803_01982_b200 as ffb
    from paper_1803_01982_b200 import _capi, engine

    ws, rank, local = dist_init()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, A = make_workload(args.workload, rank, dev)
    m, n = A.shape
    k, l, b, p = cfg.k, cfg.l, cfg.b, cfg.p
    flop_alg = ffb.flip_flop_flop_formula(m, n, l, b, p)

    def step():
        return ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, seed=0)

    for _ in range(max(args.warmup, 3)):
        ap_ = step()
    torch.cuda.synchronize()
    kernels = ap_.meta["kernels"]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    i0 = clocks.ready()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        ap_ = step()
    e1.record(st)
    torch.cuda.synchronize()
    clk = clocks.stop(i0)
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ws * 1000.0 / ms

    # dominant kernel live timing: the A*Qhat GEMM (K13, m x l x n), same shape as in the step
    lib = _capi.load()
    import ctypes as C

    Yh = torch.randn(n, l, dtype=torch.float64, device=dev).t().contiguous().t()
    out = torch.empty((l, m), dtype=torch.float64, device=dev).t()
    wsb = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    ctx = _capi.context(local)
    def kgemm():
        lib.ffb_gemm(ctx, C.c_void_p(st.cuda_stream), m, l, n, 1.0, C.c_void_p(A.data_ptr()),
                     A.stride(1), 0, C.c_void_p(Yh.data_ptr()), n, 1, 0.0,
                     C.c_void_p(out.data_ptr()), m, C.c_void_p(wsb.data_ptr()), wsb.numel())
    for _ in range(3):
        kgemm()
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(st)
    for _ in range(5):
        kgemm()
    g1.record(st)
    torch.cuda.synchronize()
    gms = g0.elapsed_time(g1) / 5
    g_tflops = 2.0 * m * n * l / (gms * 1e-3) / 1e12

    # e2e through the public API with host buffers (pinned), H2D + D2H in the timed region
    A_host = None
    e2e = None
    if rank == 0 or ws > 1:
        A_host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        A_host.copy_(A.t())
        A_host_cm = A_host.t()            # column-major (m, n) host view
        # pinned host destinations of the step's result (u, s, v, perm)
        u_h = torch.empty((k, m), dtype=torch.float64, pin_memory=True).t()
        v_h = torch.empty((k, n), dtype=torch.float64, pin_memory=True).t()
        s_h = torch.empty(k, dtype=torch.float64, pin_memory=True)
        p_h = torch.empty(n, dtype=torch.int64, pin_memory=True)

        def e2e_step():
            r = ffb.flip_flop_srqr(A_host_cm, k, l=l, b=b, p=p, seed=0)
            u_h.copy_(r.u, non_blocking=True)
            v_h.copy_(r.v, non_blocking=True)
            s_h.copy_(r.s, non_blocking=True)
            p_h.copy_(r.meta["srqr"].fact.perm, non_blocking=True)
            st.synchronize()
            return r
        r = e2e_step()
        torch.cuda.synchronize()
        es = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(st)
        for _ in range(es):
            r = e2e_step()
        x1.record(st)
        torch.cuda.synchronize()
        ems = x0.elapsed_time(x1) / es
        h2d = m * n * 8                    # A; Omega is cached on the device per (seed, s, m)
        d2h = (m + n) * k * 8 + k * 8 + n * 8   # u, v, s, perm
        # the same calls pipelined through the public batch driver
        # (batch.run_host_pipeline): one copy thread uploads every step's A from
        # pinned host memory back to back on its own stream, three compute streams
        # factorize; every step still uploads its own A and reads back its own
        # u, s, v, perm into pinned host memory
        from paper_1803_01982_b200 import batch

        npipe = 12
        outs = [(torch.empty((k, m), dtype=torch.float64, pin_memory=True).t(),
                 torch.empty((k, n), dtype=torch.float64, pin_memory=True).t(),
                 torch.empty(k, dtype=torch.float64, pin_memory=True),
                 torch.empty(n, dtype=torch.int64, pin_memory=True)) for _ in range(npipe)]

        def piped(i, A_dev):
            r = ffb.flip_flop_srqr(A_dev, k, l=l, b=b, p=p, seed=0)
            uo, vo, so, po = outs[i]
            uo.copy_(r.u, non_blocking=True)
            vo.copy_(r.v, non_blocking=True)
            so.copy_(r.s, non_blocking=True)
            po.copy_(r.meta["srqr"].fact.perm, non_blocking=True)
            return i

        batch.run_host_pipeline([A_host_cm] * 8, piped, n_streams=3, device=dev)   # warm-up
        torch.cuda.synchronize()
        y0, y1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        y0.record(st)
        batch.run_host_pipeline([A_host_cm] * npipe, piped, n_streams=3, device=dev)
        torch.cuda.synchronize()
        y1.record(st)
        torch.cuda.synchronize()
        pms = y0.elapsed_time(y1) / npipe
        e2e = {"value": 1000.0 / pms * (ws if ws > 1 else 1), "unit": "factorizations/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": pms,
               "path": "paper_1803_01982_b200.flip_flop_srqr on pinned host tensors, "
                       f"{npipe} calls: uploads on a copy stream, 3 compute streams "
                       "(batch.run_host_pipeline)",
               "serial": {"value": 1000.0 / ems * (ws if ws > 1 else 1), "ms_per_step": ems,
                          "path": "one paper_1803_01982_b200.flip_flop_srqr call at a time"}}

    # capacity: independent factorizations of the resident matrix in flight on 3
    # streams (the latency-bound stages leave SMs idle); reported beside `value`,
    # which stays one factorization at a time
    conc = None
    if rank == 0 or ws > 1:
        from paper_1803_01982_b200 import batch as _batch

        def cstep(i):
            return ffb.flip_flop_srqr(A, k, l=l, b=b, p=p, seed=0).s

        _batch.run_streams(list(range(3)), cstep, n_streams=3, device=dev)
        torch.cuda.synchronize()
        z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nconc = 12
        z0.record(st)
        _batch.run_streams(list(range(nconc)), cstep, n_streams=3, device=dev)
        torch.cuda.synchronize()
        z1.record(st)
        torch.cuda.synchronize()
        cms = z0.elapsed_time(z1) / nconc
        conc = {"value": 1000.0 / cms * ws, "unit": "factorizations/s", "ms_per_factorization": cms,
                "streams": 3, "factorizations": nconc}

    # the paper's competitor on the same device kernels: RSISVD,
    # rank k, oversampling p, q = 2 power steps (ffsrqr/svd.py:101-133)
    rsi = None
    if rank == 0 and ws == 1:
        def rs_step():
            return ffb.rsisvd(A, k, p=p, q=2, seed=0)
        rs = rs_step()
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrs = max(1, min(args.steps, 5))
        r0.record(st)
        for _ in range(nrs):
            rs = rs_step()
        r1.record(st)
        torch.cuda.synchronize()
        rms = r0.elapsed_time(r1) / nrs
        rsi = {"value": 1000.0 / rms, "unit": "factorizations/s", "ms_per_step": rms,
               "config": f"k={k}, p={p}, q=2", "path": "paper_1803_01982_b200.rsisvd",
               "sigma_k_rel_vs_flipflop": float(abs(rs.s[-1] - ap_.s[-1]) / ap_.s[-1])}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        A_np = A_host.t().numpy() if A_host is not None else A.cpu().numpy()
        A_np = np.asfortranarray(A_np)
        t_cpu = cpu_oracle_sample(A_np, cfg)
        cpu = {"value": 1.0 / t_cpu, "unit": "factorizations/s",
               "cores": len(os.sched_getaffinity(0)), "kind": "port",
               "sample": f"1 full {args.workload} factorization by the numpy oracle port "
                         f"(oracle/ffsrqr_oracle.py) on the same matrix, {t_cpu:.2f} s"}

    if rank == 0:
        achieved = flop_alg / (ms * 1e-3) / 1e12
        traffic, traffic_src = k13_traffic(args.workload)
        line = {
            "metric": METRIC, "value": value, "unit": "factorizations/s", "n_gpus": ws,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Haar factors, BASELINE spectrum, device-generated)",
            "config": {"workload": args.workload, "m": m, "n": n, "k": k, "p": p, "b": b, "l": l,
                       "l2_flush": "input 537 MB > 126 MB L2" if m * n * 8 > 126e6 else "none",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single"},
            "achieved_tflops": achieved,
            "step_roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                              "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                              "flop_alg": flop_alg,
                              "peak_source": "measured DMMA peak, profiles/r01_fp64_peak.md"},
            "roofline": {"bound": "tensor", "kernel": "K13 A*Qhat DMMA GEMM (m x l x n)",
                         "achieved": g_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": g_tflops / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "algorithmic_bytes": 8 * (m * n + n * l + m * l),
                         "ms_per_launch": gms,
                         "peak_source": "measured DMMA peak (MEASURED_PEAKS.json has no FP64)"},
            "gpu_launches": kernels * args.steps,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "rsisvd_same_device": rsi,
            "concurrent": conc,
            "certificate": {"swaps": ap_.meta["srqr"].cert.swaps, "g2": ap_.meta["srqr"].cert.g2},
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
