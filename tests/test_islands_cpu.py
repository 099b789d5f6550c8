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
