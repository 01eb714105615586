"""Multi-GPU group sharding (north star: "groups shard naturally across the 8 GPUs ... a single NCCL all-gather over
NVLink assembles the pruned cache").

Every rank prefills and prunes the contiguous block of groups GroupPlan.plan(..., world).shard(rank) gives it and
writes the pruned rows at their GLOBAL cache offsets (cache row offsets are a pure function of (rho, N_g),
prefill.cpp:235-238, so no exchange is needed before the collective).  The one data-path collective is the
all-gather of the pruned K/V/origin segments; NCCL's all-gather needs equal counts, the per-rank segments are ragged
(225 groups over 8 ranks), so it is issued as one broadcast per source rank directly into that rank's slice of the
replicated cache (no padding, no compaction copy), grouped so NCCL overlaps them.
Works on any torch.distributed backend (gloo for the CPU tests, nccl on the GPU box).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .prefill import GroupPlan


def segment_bounds(plan: GroupPlan, world: int) -> list[tuple[int, int]]:
    """Global cache rows [begin, end) owned by each rank."""
    rb = plan.rank_begin
    if len(rb) != world + 1:
        raise ValueError("plan was built for a different world size")
    return [(int(plan.row_off[rb[r]]), int(plan.row_off[rb[r + 1]])) for r in range(world)]


def allgather_cache(tensors: list[torch.Tensor], bounds: list[tuple[int, int]], unit: list[int], group=None,
                    async_op: bool = False):
    """Replicate each rank's pruned segment into every rank's full cache.

    tensors[i] is a flat cache buffer whose row r occupies [r*unit[i], (r+1)*unit[i]); on entry each rank has filled
    its own rows bounds[rank]; on return (or after the returned work handles complete) every rank holds all rows.
    """
    world = len(bounds)
    if world == 1:
        return []
    works = []
    for t, u in zip(tensors, unit):
        for src, (b, e) in enumerate(bounds):
            if e > b:
                works.append(dist.broadcast(t[b * u:e * u], src=src, group=group, async_op=True))
    if async_op:
        return works
    for w in works:
        w.wait()
    return []
