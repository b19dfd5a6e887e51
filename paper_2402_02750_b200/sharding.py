"""Unit partitioning across GPUs.

A unit is one (batch element, kv-head) cache of a layer; units never exchange
data on the decode path (reference attention.cpp:26-100 touches one state),
so ranks own disjoint unit sets and run with no collective.

* batch-major contiguous blocks when batch >= world: a sequence's heads stay on
  one GPU, as in data-parallel serving;
* head-major when batch < world (e.g. config 1: 32 heads of one sequence).

`max_over_ranks` is the only cross-rank operation bench.py performs (timing).
"""
from __future__ import annotations


def partition_units(batch: int, heads: int, world: int, rank: int):
    """Returns the sorted list of (batch, head) units owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    units = []
    if batch >= world:
        lo = batch * rank // world
        hi = batch * (rank + 1) // world
        for b in range(lo, hi):
            units.extend((b, h) for h in range(heads))
    else:
        flat = [(b, h) for h in range(heads) for b in range(batch)]  # head-major
        n = len(flat)
        units = sorted(flat[n * rank // world: n * (rank + 1) // world])
    return units


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over the default process group (or itself)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
