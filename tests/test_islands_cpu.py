"""Host-side logic of the multi-GPU island model, world_size 2 over gloo (CPU)."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_01288_b200.scheduler import gather_elites, island_seeds, migration_sources


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    I, E, km = 3, 2, 64
    groups = torch.full((I, E, km), rank * 100, dtype=torch.int16)
    groups[:, :, 0] = torch.arange(I, dtype=torch.int16)[:, None] + rank * I
    costs = torch.arange(I * E, dtype=torch.float64).view(I, E) + 1000 * rank
    gr, co = gather_elites(groups, costs)
    src = migration_sources(rank, world, I)
    # every island receives the previous global island's elites
    recv = [int(gr[s, 0, 0]) for s in src]
    out[rank] = (tuple(gr.shape), tuple(co.shape), recv, float(co[src[0], 0]))
    # max-over-ranks timing reduction used by bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert float(t) == world
    dist.destroy_process_group()


def test_gather_and_ring_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][0] == (6, 2, 64) and out[0][1] == (6, 2)
    assert out[0][2] == [5, 0, 1]   # rank 0 islands 0,1,2 <- global 5,0,1
    assert out[1][2] == [2, 3, 4]   # rank 1 islands 3,4,5 <- global 2,3,4
    assert out[0][3] == 1000.0 + 4  # island 0 gets island 5 (rank 1, local 2) elite 0


def test_island_seeds_partition_the_spawned_streams():
    a = island_seeds(7, 4, offset=0) + island_seeds(7, 4, offset=4)
    b = island_seeds(7, 8)
    assert [x.bit_generator.state for x in a] == [x.bit_generator.state for x in b]


def test_gather_is_identity_without_process_group():
    g = torch.zeros((2, 1, 8), dtype=torch.int16)
    c = torch.zeros((2, 1), dtype=torch.float64)
    gr, co = gather_elites(g, c)
    assert gr is g and co is c


def test_shard_bounds_contiguous_cover():
    from paper_2206_01288_b200 import shard_bounds
    for P in (0, 1, 7, 8, 9, 1000, 1 << 20):
        for G in (1, 2, 3, 4, 8):
            b = shard_bounds(P, G)
            assert len(b) == G and b[0][0] == 0 and b[-1][1] == P
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        shard_bounds(4, 0)


def _shard_worker(rank, world, port, out):
    """Each rank prices its contiguous shard of one global population; an
    all-gather restores the input order (the multi-GPU batch seam, SURVEY.md
    §8(e), replacing scheduler.py:537-542's map).  The 'price' here is a
    host stand-in; the GPU path is tested in test_gpu_costmodel.py."""
    import numpy as np

    from paper_2206_01288_b200 import shard_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = 1001
    pop = np.random.default_rng(0).integers(0, 64, size=(P, 8, 8)).astype(np.int16)
    bounds = shard_bounds(P, world)
    lo, hi = bounds[rank]
    mine = torch.from_numpy(pop[lo:hi].reshape(hi - lo, -1).sum(axis=1).astype(np.float64))
    # all_gather needs equal sizes: pad to the largest shard
    width = max(h - l for l, h in bounds)
    pad = torch.full((width,), float("nan"), dtype=torch.float64)
    pad[: hi - lo] = mine
    got = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(got, pad)
    full = torch.cat([got[r][: h - l] for r, (l, h) in enumerate(bounds)])
    out[rank] = bool(np.array_equal(full.numpy(), pop.reshape(P, -1).sum(axis=1).astype(np.float64)))
    dist.destroy_process_group()


def test_sharded_population_gather_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] and out[1]
