"""The N>1 path on CPU: world_size 2 over gloo.  Each rank owns a contiguous
shard of the dictionary (generated in place from the shared seeded stream),
scans the full query batch against it with word ids rebased by the shard
start, and rank 0 gathers + merges the per-shard CSRs.  The merged result
must equal one scan over the whole dictionary.  The per-rank scan here is the
oracle (this container has no GPU); on a B200 the same host logic wraps
libfpg.so (bench.py / GpuFingerprintedDictionary(id_base=...))."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N_WORDS, N_QUERIES = 6000, 120


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, oscheme
    from paper_1711_08475_b200.corpus import generate_dictionary, generate_queries, make_scheme
    from paper_1711_08475_b200.sharding import gather_csr, shard_bounds

    lo, hi = shard_bounds(N_WORDS, world, rank)
    blob, offs = generate_dictionary(2, n=hi - lo, first=lo)
    base_blob, base_offs = generate_dictionary(2, n=N_WORDS)  # letters over the WHOLE dictionary
    qb, qo = generate_queries(2, base_blob, base_offs, nq=N_QUERIES)
    s = make_scheme(base_blob, 2, 16)
    osch = oscheme(2, s.letters().symbols(), 16, 2, 3)
    off, ids, _ = Oracle().query_batch(blob, offs, qb, qo, osch, 1, 1, True, True, threads=2)
    ids = ids + np.uint32(lo)  # rebase to global ids
    merged = gather_csr(off, ids)
    # the point-to-point tensor gather of query_batch_distributed (NCCL on a
    # GPU box; CPU tensors over gloo here), merged with the host merge
    import torch

    from paper_1711_08475_b200.sharding import gather_rows, merge_csr

    parts = gather_rows(torch.from_numpy(off.view(np.int64)), torch.from_numpy(ids.view(np.int32)))
    if rank == 0:
        m2 = merge_csr([(o.numpy().view(np.uint64), i.numpy().view(np.uint32)) for o, i in parts])
        assert np.array_equal(m2[0], merged[0]) and np.array_equal(m2[1], merged[1])
        np.savez(out_path, off=merged[0], ids=merged[1])
    else:
        assert parts is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_shard_gather_equals_single_scan(tmp_path, world):
    out = str(tmp_path / "merged.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)

    from oracle.oracle import Oracle, oscheme
    from paper_1711_08475_b200.corpus import generate_dictionary, generate_queries, make_scheme

    blob, offs = generate_dictionary(2, n=N_WORDS)
    qb, qo = generate_queries(2, blob, offs, nq=N_QUERIES)
    s = make_scheme(blob, 2, 16)
    off, ids, _ = Oracle().query_batch(blob, offs, qb, qo, oscheme(2, s.letters().symbols(), 16, 2, 3), 1, 1,
                                       True, True, threads=2)
    assert np.array_equal(got["off"], off)
    assert np.array_equal(got["ids"], ids)
    assert len(ids) > 0
