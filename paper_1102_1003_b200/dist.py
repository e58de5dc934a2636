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


def _all_gather_flat(t, group=None):
    """Concatenation of every rank's equal-sized 1-D tensor `t` (rank order)."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    src = t.cpu()  # gloo (tests): host staging
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    return torch.cat(parts).to(t.device)


def build_distributed(offsets, tids, n_transactions: int, group=None, **kw):
    """Sharded build: every rank builds the BatMaps of its share of each width
    class (batmap_build_shard), the shares and failure records are all-gathered over the process
    group (NCCL over NVLink on a B200 box), and batmap_shard_import completes every rank's handle.
    Returns a Collection equivalent to a whole build on every rank."""
    from .batmap import Collection

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    c = Collection(offsets, tids, n_transactions, part=rank, n_parts=world, **kw)
    if world == 1:  # a one-part build is the whole build: nothing to exchange
        return c
    stride_w = max(c.shard_sizes(p)[0] for p in range(world))
    nf = torch.tensor([c.shard_sizes(rank)[1]], dtype=torch.int64, device=offsets.device)
    counts = _all_gather_flat(nf, group)
    n_fails = [int(x) for x in counts.tolist()]
    stride_f = max(max(n_fails), 1)
    words = torch.empty(max(stride_w, 1), dtype=torch.int32, device=offsets.device)
    fails = torch.empty(stride_f, dtype=torch.int64, device=offsets.device)
    c.shard_export(words, fails)
    c.shard_import(_all_gather_flat(words, group), words.numel(), _all_gather_flat(fails, group), n_fails, stride_f)
    return c


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


def mine_distributed(offsets, tids, n_transactions: int, threshold: int = 1, dst: int = 0, group=None,
                     device=None, **kw):
    """End to end from host buffers at N ranks (the multi-GPU counterpart of mine_host): every rank
    copies the vertical CSR (pinned host memory preferred) to its GPU, runs the sharded build and
    its share of the pairs, and `dst` receives the gathered, sorted triples as a host int32
    [K, 3] array (None on the other ranks)."""
    import numpy as np

    from .batmap import sort_triples

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    off_d = torch.as_tensor(offsets).to(dev, non_blocking=True)
    tids_d = torch.as_tensor(tids).to(dev, non_blocking=True)
    c = build_distributed(off_d, tids_d, n_transactions, group=group, **kw)
    try:
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        local = c.pair_supports(None, threshold, part=rank, n_parts=world)
        if dist.get_backend(group) != "nccl":
            local = local.cpu()  # gloo (tests): host staging
        allp = gather_triples(local, dst=dst, group=group)
        if allp is None:
            return None
        return np.asarray(sort_triples(allp.to(dev)).cpu())
    finally:
        c.close()
