"""bench.py's multi-GPU plumbing on CPU: `--gpus 2` without a torchrun
environment re-launches itself with two ranks (gloo in --dry mode), partitions
the batched problems contiguously and gathers every problem's result slot to
rank 0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,slot", [("cfg5", ["u", "s", "v", "perm", "cert"]),
                                           ("cfg4", ["u", "s", "perm", "cert"])])
def test_bench_spawns_ranks_and_gathers(workload, slot):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload",
                          workload, "--dry", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = lines[0]
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong" and rec["dry"]
    assert rec["gather"]["complete"] and rec["gather"]["slot"] == slot
    assert rec["config"]["parallelism"] == "partitioned x2 (contiguous)"
