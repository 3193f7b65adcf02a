"""Dictionary sharding across GPUs.

Every (query, word) pair is independent, so the dictionary is split into
contiguous input-order id ranges, one per GPU; each GPU scans the full query
batch against its shard and reports word ids rebased by the shard's first id.
Because shard g owns ids below shard g+1, the oracle's (query asc, word asc)
order is the per-query concatenation of shard rows: a gather, not a sort.
There is no data-path collective.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of shard `rank` of `world` over n ids (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return n * rank // world, n * (rank + 1) // world


def merge_csr(parts) -> tuple[np.ndarray, np.ndarray]:
    """Concatenate per-shard CSRs [(offsets, ids), ...] (shard order) row by row."""
    if not parts:
        raise ValueError("no shards")
    nq = len(parts[0][0]) - 1
    counts = np.zeros(nq, dtype=np.uint64)
    for off, _ in parts:
        if len(off) - 1 != nq:
            raise ValueError("shards disagree on the number of queries")
        counts += np.diff(off.astype(np.uint64))
    offsets = np.zeros(nq + 1, dtype=np.uint64)
    offsets[1:] = np.cumsum(counts)
    ids = np.zeros(int(offsets[-1]), dtype=np.uint32)
    cursor = offsets[:-1].copy()
    for off, sid in parts:
        lens = np.diff(off.astype(np.int64))
        if not len(sid):
            continue
        # destination of every element of this shard's rows
        row_of = np.repeat(np.arange(nq), lens)
        within = np.arange(len(sid), dtype=np.int64) - np.repeat(off[:-1].astype(np.int64), lens)
        ids[(cursor[row_of].astype(np.int64) + within)] = sid
        cursor += lens.astype(np.uint64)
    return offsets, ids


def gather_csr(offsets: np.ndarray, ids: np.ndarray, group=None, dst: int = 0):
    """Gather every rank's CSR to `dst` (torch.distributed, any backend) and
    merge there; other ranks get None."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    objs = [None] * world if rank == dst else None
    dist.gather_object((offsets, ids), objs, dst=dst, group=group)
    if rank != dst:
        return None
    return merge_csr(objs)
