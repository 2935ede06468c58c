"""CPU: the N>1 host path with world_size 2 over gloo.

Streams shard with no data-path collective; the only
cross-rank traffic is the timing barrier and the max-over-ranks reduction.
"""
import json
import os
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_05488_b200.sharding import max_over_ranks, shard_streams, weak_shard
from tests import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_streams_partition():
    for total in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            ids = []
            for r in range(world):
                sh = shard_streams(total, r, world)
                ids += sh.stream_ids
                assert abs(sh.count - total / world) < 1
            assert ids == list(range(total))
    assert weak_shard(16, 3, 4).stream_ids == list(range(48, 64))
    assert shard_streams(64, 1, 8).seed(0) == 1008


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = shard_streams(64, rank, world)
    ids = [None] * world
    dist.all_gather_object(ids, sh.stream_ids)
    m = max_over_ranks(10.0 + rank)
    dist.barrier()
    if rank == 0:
        q.put((ids, m))
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_max():
    port = 29500 + os.getpid() % 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, m = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ids[0] == list(range(32)) and ids[1] == list(range(32, 64))
    assert m == 11.0


@pytest.mark.skipif(not os.path.exists(oracle.REF_BENCH), reason="oracle/_ref not built")
def test_reference_arm_under_torchrun_two_ranks():
    """bench.py --impl reference launched like the driver does for N=2: rank 0
    alone runs the CPU reference and prints exactly one JSON line."""
    port = 28500 + os.getpid() % 1000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
           "2", "--steps", "2", "--warmup", "1", "--height", "48", "--width", "64", "--objects", "1",
           "--object-size", "8", "--cpu-budget", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
