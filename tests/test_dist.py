"""CPU, world_size 2 over gloo: the N>1 bench plumbing (replicas only).

The hot path does not shard (BASELINE north_star is single-GPU; SURVEY.md
§8e): bench.py --gpus N runs N independent replicas, barriers around the
timed region and reports the MAX step time over ranks, with whole-job
throughput = (sum of replica work) / that time. This checks the collective
helpers those numbers come from."""
import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import bench

    d = bench.Dist()
    d.barrier()
    t = 10.0 + rank  # rank-dependent "elapsed ms"
    out[rank] = (d.max(t), d.sum(1.0), d.world, d.rank)
    d.barrier()
    d.close()


@pytest.mark.timeout(120)
def test_dist_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        mx, total, w, rank = out[r]
        assert mx == 11.0 and total == 2.0 and w == 2 and rank == r
