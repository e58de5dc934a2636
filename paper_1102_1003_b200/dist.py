"""Multi-GPU plumbing: one process per GPU, the pair triangle dealt across ranks by the
library's planner (batmap_pair_supports_part), compacted triples gathered to one rank over
torch.distributed (NCCL over NVLink on a B200 box) and merged by the library's device sort.

This is the only exchange the method has: every pair's count is independent
(P:60), so no collective touches the data path before the final gather.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gather_triples(local: torch.Tensor, dst: int = 0, group=None):
    """Gather every rank's [K_r, 3] int32 triples to rank `dst` (concatenated in rank order).

    Returns the concatenation on `dst` and None elsewhere.  Works with any backend that
    supports all_gather and gather (NCCL, gloo).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(max(counts), 1)
    pad = torch.zeros((mx, 3), dtype=local.dtype, device=local.device)
    if local.shape[0]:
        pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def pair_supports_distributed(coll, items=None, threshold: int = 1, dst: int = 0, group=None):
    """This rank's share of the pairs (batmap_pair_supports_part), gathered and sorted on `dst`."""
    from .batmap import sort_triples

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    local = coll.pair_supports(items, threshold, part=rank, n_parts=world)
    allp = gather_triples(local, dst=dst, group=group)
    if allp is None:
        return None
    return sort_triples(allp)
