"""GPU: the N>1 path with two ranks sharing one B200 (the driver's scaling runs
use one GPU per rank; this box has one). Streams are independent CBNetworks
(network.hpp:139-141), so a rank's share of the global stream ids
must give exactly what one process running all of them gives."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1808_05488_b200 import cbi
from paper_1808_05488_b200.sharding import shard_streams

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOTAL, H, W, T = 5, 96, 128, 5


def _frames(global_ids):
    return np.stack([cbi.from_pnm8(cbi.to_pnm8(cbi.gen_synthetic(cbi.SyntheticConfig(
        H, W, 3, T, 3, 12, 3, 2, 0.0, 1000 + g)))) for g in global_ids], axis=1)  # [T][S][C][H][W]


def _run(global_ids):
    spec = cbi.make_seg_spec(1, H, W)
    net = cbi.convert_to_cb(spec, [0.05] * 5, n_streams=len(global_ids))
    fr = _frames(global_ids)
    for t in range(T):
        net.enqueue(np.ascontiguousarray(fr[t]))
    net.synchronize()
    outs = [net.node_output(len(net.nodes()) - 1, s) for s in range(len(global_ids))]
    return outs, net.counts()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = shard_streams(TOTAL, rank, world)
    outs, counts = _run(sh.stream_ids)
    got = [None] * world
    dist.all_gather_object(got, (sh.stream_ids, [o.tobytes() for o in outs], counts.tolist()))
    if rank == 0:
        q.put(got)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_equal_one_rank(gpu):
    port = 27500 + os.getpid() % 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one, one_counts = _run(list(range(TOTAL)))
    seen = []
    for ids, outs, counts in got:
        counts = np.asarray(counts)
        for k, g in enumerate(ids):
            seen.append(g)
            o = np.frombuffer(outs[k], np.float32).reshape(one[g].shape)
            assert np.array_equal(o, one[g]), f"global stream {g}"
            assert np.array_equal(counts[:, k], one_counts[:, g]), f"global stream {g}"
    assert sorted(seen) == list(range(TOTAL))


def test_bench_two_ranks_strong_scaling_config(gpu):
    """bench.py --config cfg5 (strong scaling: a fixed stream total sharded over the
    ranks) under torchrun with 2 ranks on this one GPU: rank 0 prints one line
    whose value covers all the streams."""
    port = 26500 + os.getpid() % 1000
    env = dict(os.environ, BENCH_DEVICE_MOD="1", BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
           "cfg5", "--streams", "6", "--height", "136", "--width", "240", "--steps", "3", "--warmup", "3",
           "--no-e2e", "--sweep-steps", "0", "--dense-steps", "2", "--profile-steps", "1", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["total_streams"] == 6 and d["config"]["baseline_config"] == "cfg5"
    assert d["value"] > 0 and d["gpu_launches"] > 0
