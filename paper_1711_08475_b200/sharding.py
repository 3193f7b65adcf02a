"""Dictionary sharding across GPUs.

Every (query, word) pair is independent, so the dictionary is split into
contiguous input-order id ranges, one per GPU; each GPU scans the full query
batch against its shard and reports word ids rebased by the shard's first id.
Because shard g owns ids below shard g+1, the oracle's (query asc, word asc)
order is the per-query concatenation of shard rows: a gather, not a sort.

Two deployments:

* one process drives several GPUs: ``GpuFingerprintedDictionary(words,
  scheme, devices=(0, 1, ...))``; libfpg.so scans the shards concurrently and
  gathers their rows on the host (fpg_batch_download);
* one process per GPU (torch.distributed, NCCL over NVLink/NVSwitch): each
  rank holds ``GpuFingerprintedDictionary(shard, scheme, id_base=lo)`` and
  ``query_batch_distributed`` gathers the ranks' device-resident CSRs to one
  rank over NCCL point-to-point, merges them there with a CUDA kernel
  (fpg_csr_merge_device) and copies the merged CSR to the host once.  The
  only collective traffic is the result gather itself.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of shard `rank` of `world` over n ids (sizes differ by <= 1);
    the same split as libfpg.so's assign_ranges."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return n * rank // world, n * (rank + 1) // world


def shard_of(blob: np.ndarray, offs: np.ndarray, lo: int, hi: int) -> tuple[np.ndarray, np.ndarray]:
    """Words [lo, hi) of a packed (blob, offsets) collection, offsets rebased."""
    a, b = int(offs[lo]), int(offs[hi])
    return blob[a:b], (offs[lo:hi + 1] - offs[lo]).astype(np.uint64)


def merge_csr(parts) -> tuple[np.ndarray, np.ndarray]:
    """Concatenate per-shard host CSRs [(offsets, ids), ...] (shard order) row
    by row.  Host form of fpg_csr_merge_device, for CSRs already on the host
    (e.g. a gloo process group)."""
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
    """Gather every rank's host CSR to `dst` (torch.distributed, any backend)
    and merge there; other ranks get None."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    objs = [None] * world if rank == dst else None
    dist.gather_object((offsets, ids), objs, dst=dst, group=group)
    if rank != dst:
        return None
    return merge_csr(objs)


def gather_rows(offsets, ids, dst: int = 0, group=None):
    """Point-to-point gather of per-rank CSR tensors to rank `dst`.

    offsets: int64 tensor [nq + 1] (uint64 bits), ids: int32 tensor (uint32
    bits), both on this rank's communication device (CUDA for NCCL, CPU for
    gloo).  Totals are exchanged first (all_gather), then every rank sends
    its rows to `dst` (isend / irecv: NVLink peer copies under NCCL).
    Returns the list of (offsets, ids) per rank at `dst` (its own tensors in
    its slot), None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = offsets.device
    tot = torch.tensor([ids.numel()], dtype=torch.int64, device=dev)
    tots = [torch.empty_like(tot) for _ in range(world)]
    dist.all_gather(tots, tot, group=group)
    gdst = dst if group is None else dist.get_global_rank(group, dst)
    if rank != dst:
        reqs = [dist.isend(offsets, gdst, group=group)]
        if ids.numel():
            reqs.append(dist.isend(ids, gdst, group=group))
        for r in reqs:
            r.wait()
        return None
    parts, reqs = [], []
    for r in range(world):
        if r == rank:
            parts.append((offsets, ids))
            continue
        src = r if group is None else dist.get_global_rank(group, r)
        o = torch.empty_like(offsets)
        i = torch.empty(int(tots[r].item()), dtype=ids.dtype, device=dev)
        reqs.append(dist.irecv(o, src, group=group))
        if i.numel():
            reqs.append(dist.irecv(i, src, group=group))
        parts.append((o, i))
    for q in reqs:
        q.wait()
    return parts


class _DevArray:
    """__cuda_array_interface__ over a device pointer owned by libfpg.so."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_tensors(csr: dict):
    """(offsets int64, ids int32) torch views of Batch.device_csr(): no copy."""
    import torch

    dev = torch.device("cuda", csr["device"])
    nq, total = csr["nq"], csr["total"]
    off = torch.as_tensor(_DevArray(csr["offsets"], nq + 1, "<i8"), device=dev)
    ids = (torch.as_tensor(_DevArray(csr["ids"], total, "<i4"), device=dev) if total
           else torch.empty(0, dtype=torch.int32, device=dev))
    return off, ids


def merge_device(parts, nq: int, device: int):
    """Merged (offsets, ids) device tensors of per-rank CSR tensors on
    `device`, by fpg_csr_merge_device on torch's current stream."""
    import torch

    from .fingerprints import csr_merge_device

    dev = torch.device("cuda", device)
    total = sum(int(i.numel()) for _, i in parts)
    out_off = torch.empty(nq + 1, dtype=torch.int64, device=dev)
    out_ids = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    ptrs = [(o.data_ptr(), i.data_ptr() if i.numel() else 0) for o, i in parts]
    csr_merge_device(device, ptrs, nq, out_off.data_ptr(), out_ids.data_ptr(),
                     torch.cuda.current_stream(dev).cuda_stream)
    return out_off, out_ids[:total]


def query_batch_distributed(batch, opt, want_stats: bool = False, dst: int = 0, group=None,
                            host_out=None):
    """Runs the uploaded query batch on this rank's shard, gathers every
    rank's CSR to rank `dst` over the process group (device to device) and
    merges it there on the GPU.  Rank `dst` returns (offsets, ids) as host
    numpy arrays (copied into `host_out` = (pinned int64, pinned int32 torch
    tensors) when given and large enough); other ranks return None."""
    import torch
    import torch.distributed as dist

    batch.run(opt, want_stats=want_stats)
    csr = batch.device_csr(0)
    off, ids = device_tensors(csr)
    torch.cuda.set_device(csr["device"])
    # libfpg's run synchronised its own stream before returning: the tensors are ready
    parts = gather_rows(off, ids, dst=dst, group=group)
    if dist.get_rank(group) != dst:
        return None
    m_off, m_ids = merge_device(parts, csr["nq"], csr["device"])
    if host_out is not None and host_out[0].numel() >= m_off.numel() and host_out[1].numel() >= m_ids.numel():
        h_off, h_ids = host_out[0][: m_off.numel()], host_out[1][: m_ids.numel()]
        h_off.copy_(m_off, non_blocking=True)
        h_ids.copy_(m_ids, non_blocking=True)
    else:
        h_off, h_ids = m_off.cpu(), m_ids.cpu()
    torch.cuda.current_stream().synchronize()
    return h_off.numpy().view(np.uint64), h_ids.numpy().view(np.uint32)
