"""Multi-rank plumbing of bench.py on CPU (gloo, world_size 2): the batched
workload (C5) is partitioned into disjoint contiguous problem ranges that
cover every problem exactly once, each rank builds its own inputs with the
reference generators, and the max-over-ranks reduction used for timing works.
No data-path collective exists (problems are independent)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import bench
    P = 10
    lo, hi = rank * P // world, (rank + 1) * P // world
    gen = bench.ProductGen()
    # first problem of this rank: C5 generator with the rank's seed offset
    coords = gen.gen_jitter(16, 0.5, 0.2, bench.SEED + lo, 2)
    t = torch.tensor([float(lo), float(hi), float(coords.sum())], dtype=torch.float64)
    gathered = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, t)
    m = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put(([g.tolist() for g in gathered], float(m.item())))
    dist.destroy_process_group()


def test_problem_partition_and_max_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got, mx = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [(int(a), int(b)) for a, b, _ in got]
    assert ranges == [(0, 5), (5, 10)]
    assert mx == 2.0
    # each rank generated a different problem (different seeds)
    assert got[0][2] != got[1][2]
