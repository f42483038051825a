"""The slab step (sk_ch_explicit_slab: z wrap replaced by ghost planes) on one
GPU: with a single rank the halo exchange is the periodic self-copy, and the
result is bit-identical to the single-domain kernel (same loads, same order)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams, CahnHilliardState
from paper_2205_03354_b200.grid import BoundaryKind, GridSpec
from paper_2205_03354_b200.slab import SlabCahnHilliard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,formulation", [((64, 64, 32), "factored"), ((70, 40, 12), "factored"),
                                              ((64, 32, 16), "composed")])
def test_slab_single_rank_equals_single_domain(dims, formulation):
    p = CahnHilliardParams.from_epsilon(0.02, formulation)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    c0 = 0.05 * np.random.default_rng(11).uniform(-1, 1, g.unknown_count())
    s = SlabCahnHilliard(g, p)
    s.scatter(c0)
    s.step(dt, 20)
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, 20)
    assert np.array_equal(s.local_field(), st.c)


def _cuda_slab_worker(rank, world, port, dims, steps, out, overlapped=False):
    import os
    import sys

    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import numpy as np
    import torch.distributed as dist

    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams
    from paper_2205_03354_b200.grid import BoundaryKind, GridSpec
    from paper_2205_03354_b200.slab import SlabCahnHilliard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    s = SlabCahnHilliard(g, p)  # the CUDA slab step (sk_ch_explicit_slab) on cuda:0
    s.scatter(0.05 * np.random.default_rng(11).uniform(-1, 1, g.unknown_count()))
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    if overlapped:
        s.step_overlapped(dt, steps)
    else:
        s.step(dt, steps)
    out[rank] = s.local_field()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("overlapped", [False, True])
def test_slab_two_cuda_ranks_equal_single_domain(overlapped):
    # two ranks (processes) each run the CUDA slab step on its half of the z
    # planes — both on the one GPU here, independent kernels, the halo planes
    # exchanged over gloo through host memory — and reproduce the
    # single-domain kernel bit for bit
    import socket

    import torch.multiprocessing as mp

    def free_port():
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        return port

    dims, steps, world = (64, 64, 32), 12, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_cuda_slab_worker, args=(world, free_port(), dims, steps, out, overlapped), nprocs=world, join=True)
    got = np.concatenate([out[r] for r in range(world)])
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    st = CahnHilliardState(g, 0.05 * np.random.default_rng(11).uniform(-1, 1, g.unknown_count()))
    CahnHilliardExplicit(g, p).step(st, 0.2 * h ** 4 / (144 * p.kappa), steps)
    assert np.array_equal(got, st.c)


def test_slab_overlapped_single_rank_equals_single_domain():
    # the boundary / interior split on one rank (periodic self-exchange)
    dims = (64, 64, 32)
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    c0 = 0.05 * np.random.default_rng(12).uniform(-1, 1, g.unknown_count())
    s = SlabCahnHilliard(g, p)
    s.scatter(c0)
    s.step_overlapped(dt, 15)
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, 15)
    assert np.array_equal(s.local_field(), st.c)


@pytest.mark.parametrize("dims", [(64, 64, 32), (70, 40, 12), (64, 32, 8)])
def test_peer_slab_single_rank_equals_single_domain(dims):
    # halo exchange fused into the step's stores (sk_ch_explicit_slab_peer):
    # with one rank the "neighbours" are this rank's own ghost planes
    from paper_2205_03354_b200.slab import PeerSlabCahnHilliard

    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    c0 = 0.05 * np.random.default_rng(13).uniform(-1, 1, g.unknown_count())
    s = PeerSlabCahnHilliard(g, p)
    s.scatter(c0)
    s.step(dt, 17)
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, 17)
    assert np.array_equal(s.local_field(), st.c)


def _peer_slab_worker(rank, world, port, dims, steps, out):
    import os
    import sys

    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import numpy as np
    import torch.distributed as dist

    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams
    from paper_2205_03354_b200.grid import BoundaryKind, GridSpec
    from paper_2205_03354_b200.slab import PeerSlabCahnHilliard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    s = PeerSlabCahnHilliard(g, p)  # IPC mappings of the neighbours' buffers (same GPU here)
    s.scatter(0.05 * np.random.default_rng(14).uniform(-1, 1, g.unknown_count()))
    s.step(0.2 * h ** 4 / (144 * p.kappa), steps)
    out[rank] = s.local_field()
    s.close()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_peer_slab_cuda_ranks_equal_single_domain(world):
    # `world` processes, each stepping its slab with the fused halo stores
    # into its neighbours' ghost planes through CUDA IPC mappings (on the one
    # GPU here: independent kernels, ordered by stream sync + a gloo barrier
    # per step; across GPUs the same stores go over NVLink): bit-identical
    # to the single-domain kernel
    import socket

    import torch.multiprocessing as mp

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    dims, steps = (64, 64, 32), 9
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_peer_slab_worker, args=(world, port, dims, steps, out), nprocs=world, join=True)
    got = np.concatenate([out[r] for r in range(world)])
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    st = CahnHilliardState(g, 0.05 * np.random.default_rng(14).uniform(-1, 1, g.unknown_count()))
    CahnHilliardExplicit(g, p).step(st, 0.2 * h ** 4 / (144 * p.kappa), steps)
    assert np.array_equal(got, st.c)
