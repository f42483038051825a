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


def _slab_worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch.distributed as dist

    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams
    from paper_2205_03354_b200.grid import make_periodic_grid
    from paper_2205_03354_b200.slab import SlabCahnHilliard, numpy_slab_step

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, h = 12, 1.0 / 12
    p = CahnHilliardParams.from_epsilon(0.05)
    g = make_periodic_grid(3, n, h)
    c0 = 0.05 * np.random.default_rng(3).uniform(-1, 1, n ** 3)
    s = SlabCahnHilliard(g, p, step_fn=numpy_slab_step(n, n, n // world, h, p))
    s.scatter(c0)
    s.step(1e-7, 5)
    out[rank] = s.local_field()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_slab_exchange_gloo_matches_single_domain():
    # the z-slab halo exchange (ring, two planes each way) over gloo with 2
    # ranks reproduces the single-domain run of the same numpy step
    import numpy as np

    sys.path.insert(0, str(ROOT))
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams
    from paper_2205_03354_b200.grid import make_periodic_grid
    from paper_2205_03354_b200.slab import SlabCahnHilliard, numpy_slab_step

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.concatenate([out[r] for r in range(world)])
    n, h = 12, 1.0 / 12
    p = CahnHilliardParams.from_epsilon(0.05)
    one = SlabCahnHilliard(make_periodic_grid(3, n, h), p, step_fn=numpy_slab_step(n, n, n, h, p))
    one.scatter(0.05 * np.random.default_rng(3).uniform(-1, 1, n ** 3))
    one.step(1e-7, 5)
    assert np.array_equal(got, one.local_field())


def test_numpy_slab_step_matches_oracle(orc):
    # the CPU step used by the exchange test is the CH step (oracle, 1e-10)
    import numpy as np

    sys.path.insert(0, str(ROOT))
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams
    from paper_2205_03354_b200.grid import make_periodic_grid
    from paper_2205_03354_b200.slab import SlabCahnHilliard, numpy_slab_step

    n, h = 12, 1.0 / 12
    p = CahnHilliardParams.from_epsilon(0.05)
    c0 = 0.05 * np.random.default_rng(3).uniform(-1, 1, n ** 3)
    one = SlabCahnHilliard(make_periodic_grid(3, n, h), p, step_fn=numpy_slab_step(n, n, n, h, p))
    one.scatter(c0)
    one.step(1e-7, 5)
    ref = orc.ch_explicit(3, n, h, p, 1e-7, 5, c0)
    assert np.linalg.norm(one.local_field() - ref) <= 1e-10 * np.linalg.norm(ref)
