"""CPU: the multi-GPU partitioning with 2 ranks over gloo (the N>1 path of
bench.py, minus the GPU): ranks own disjoint unit sets that cover every unit,
and timing is max-reduced over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_02750_b200.sharding import gather_outputs, max_over_ranks, partition_units


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shapes, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for batch, heads in shapes:
            mine = partition_units(batch, heads, world, rank)
            gathered = [None] * world
            dist.all_gather_object(gathered, mine)
            if rank == 0:
                flat = [u for part in gathered for u in part]
                out.put((batch, heads, len(flat), len(set(flat)),
                         sorted(flat) == sorted((b, h) for b in range(batch) for h in range(heads))))
        t = max_over_ranks(1.0 + rank)
        if rank == 0:
            out.put(("max", t))
        # optional output all-gather: each rank's outputs carry its unit ids
        batch, heads = 5, 3  # uneven shards (batch-major: 2 and 3 sequences)
        mine = partition_units(batch, heads, world, rank)
        counts = [len(partition_units(batch, heads, world, r)) for r in range(world)]
        local = torch.tensor([[b * heads + h, rank] for b, h in mine], dtype=torch.float32)
        full = gather_outputs(local, counts)
        if rank == 0:
            out.put(("gather", full[:, 0].tolist(), full[:, 1].tolist(), counts))
    finally:
        dist.destroy_process_group()


def test_partition_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    shapes = [(64, 32), (1, 32), (16, 32), (3, 8), (128, 8)]
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shapes, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(len(shapes) + 2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in results[:-2]:
        batch, heads, n, n_unique, covers = r
        assert n == n_unique == batch * heads and covers, r
    assert results[-2] == ("max", 2.0)
    tag, ids, owners, counts = results[-1]
    assert tag == "gather" and ids == list(range(15)), ids
    assert owners == [0.0] * counts[0] + [1.0] * counts[1]


@pytest.mark.parametrize("batch,heads,world", [(64, 32, 8), (1, 32, 8), (16, 32, 8), (5, 3, 4)])
def test_partition_balanced(batch, heads, world):
    sizes = [len(partition_units(batch, heads, world, r)) for r in range(world)]
    assert sum(sizes) == batch * heads
    assert max(sizes) - min(sizes) <= max(heads, 1)
