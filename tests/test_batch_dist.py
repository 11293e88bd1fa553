"""Multi-process (gloo, world_size 2, CPU) coverage of the batched driver's
host logic: contiguous partitioning and the fixed-slot gather to rank 0.  The
GPU compute is replaced by an injected solver; on a GPU box the same code path
runs with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_01982_b200 import batch


def test_partition_is_contiguous_and_complete():
    for n in (1, 3, 7, 64):
        for world in (1, 2, 3, 4, 8):
            got = [list(batch.partition(n, world, r)) for r in range(world)]
            assert sum(got, []) == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1


class _Fake:
    def __init__(self, i, m, k):
        g = np.random.default_rng(i)
        self.u = torch.from_numpy(g.standard_normal((m, k)))
        self.s = torch.arange(k, dtype=torch.float64) + i


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results, gathered = batch.flip_flop_batch(
            make_problem=None, n_problems=n, k=3, l=4, b=2, p=1,
            solve=lambda i: _Fake(i, 5, 3), gather=("u", "s"))
        if rank == 0:
            torch.save({k: v.clone() for k, v in gathered.items()}, out)
        else:
            assert gathered["u"] is None
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [3, 8])
def test_two_rank_gather_matches_single_rank(tmp_path, n):
    out = str(tmp_path / "g.pt")
    mp.spawn(_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
    got = torch.load(out)
    for i in range(n):
        ref = _Fake(i, 5, 3)
        assert torch.equal(got["u"][i], ref.u)
        assert torch.equal(got["s"][i], ref.s)
