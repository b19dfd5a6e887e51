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


def gather_outputs(out_local, n_local_per_rank):
    """Optional all-gather of the per-rank decode outputs (the only
    collective the decode path may have; NCCL over NVLink on GPUs, gloo on CPU).

    out_local: [n_local, ...] tensor of this rank's units (in partition order);
    n_local_per_rank: unit count of every rank.  Returns [sum(n), ...] in rank
    order, i.e. the global unit order of `partition_units`.  Uneven shards are
    padded to the largest one for the collective and trimmed afterwards.
    """
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return out_local
    world = dist.get_world_size()
    m = max(n_local_per_rank)
    tail = tuple(out_local.shape[1:])
    pad = out_local.new_zeros((m,) + tail)
    pad[: out_local.shape[0]] = out_local
    if dist.get_backend() == "nccl":
        buf = out_local.new_empty((world * m,) + tail)
        dist.all_gather_into_tensor(buf, pad)
        parts = [buf[r * m: r * m + n] for r, n in enumerate(n_local_per_rank)]
    else:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        parts = [b[:n] for b, n in zip(bufs, n_local_per_rank)]
    return torch.cat(parts)
