"""N>1 path on CPU: world_size-2 gloo group exercising the query sharding and
the max-over-ranks timing reduction bench.py uses (one process per GPU over
NCCL on the B200 box).  Runs the restatement oracle per shard so the merged
per-rank results can be checked against a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_00855_b200.shard import Group, shard_range


def test_shard_ranges_partition():
    for count in (0, 1, 7, 10, 10000, 10001):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(count, world, r) for r in range(world)]
            got = [i for lo, hi in spans for i in range(lo, hi)]
            assert got == list(range(count))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_00855_b200 import _abi as A, synth
        from oracle.refpy import OracleLib
        g = Group(world)
        p = A.synth_params(docs=400, dense_dim=8, learned_vocab=500, learned_nnz=8,
                           statistical_vocab=500, statistical_nnz=6, seed=4)
        c, kg, _ = synth.generate_corpus(p, 1)
        q = synth.synth_queries(p, 37, beam_width=24)
        lo, hi = shard_range(q.count, world, rank)
        oracle = OracleLib()
        ix = oracle.index_build(oracle.store(c, kg), degree=6, knn_k=10, seed=3)
        g.barrier()
        res = oracle.batch_query(ix, q.subset(np.arange(lo, hi)))
        elapsed = 0.5 + rank  # stand-in for the per-rank device time
        out[rank] = (lo, hi, res.doc_id[:, :10].tolist(), g.max(elapsed), g.sum(hi - lo),
                     g.bcast(123.0 if rank == 0 else -1.0))
        g.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_query_sharding_matches_single_process(oracle):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_2511_00855_b200 import _abi as A, synth
    p = A.synth_params(docs=400, dense_dim=8, learned_vocab=500, learned_nnz=8,
                       statistical_vocab=500, statistical_nnz=6, seed=4)
    c, kg, _ = synth.generate_corpus(p, 1)
    q = synth.synth_queries(p, 37, beam_width=24)
    ix = oracle.index_build(oracle.store(c, kg), degree=6, knn_k=10, seed=3)
    full = oracle.batch_query(ix, q).doc_id[:, :10].tolist()
    merged = out[0][2] + out[1][2]
    assert out[0][:2] == (0, 19) and out[1][:2] == (19, 37)
    assert merged == full
    assert out[0][3] == out[1][3] == 1.5          # max over ranks
    assert out[0][4] == out[1][4] == 37           # queries across ranks
    assert out[0][5] == out[1][5] == 123.0        # beam broadcast from rank 0


# ------------------------------------------------ vertex-range sharded build
def test_vertex_ranges_partition():
    from paper_2511_00855_b200.shard import vertex_ranges
    for n in (1, 7, 33, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = vertex_ranges(n, world)
            assert [i for lo, hi in spans for i in range(lo, hi)] == list(range(n))


def _knn_worker(rank, world, port, out):
    """One rank of the sharded NN-Descent (fg_index_build_sharded's scheme):
    the full snapshot is replicated, each rank computes its vertex range, one
    all-gather of the {ids, scores, fresh} rows and an all-reduce of the
    replaced count per pass (gloo here, NCCL on the GPUs)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_00855_b200 import _abi as A, synth
        from paper_2511_00855_b200.shard import vertex_ranges
        from oracle.refpy import OracleLib
        p = A.synth_params(docs=300, dense_dim=8, learned_vocab=400, learned_nnz=8,
                           statistical_vocab=400, statistical_nnz=6, seed=9)
        c, kg, _ = synth.generate_corpus(p, 1)
        o = OracleLib()
        st = o.store(c, kg)
        k, n = 12, c.n
        ids, sc, fr = o.knn_init(st, n, k, 42)
        lo, hi = vertex_ranges(n, world)[rank]
        cn = (n + world - 1) // world
        passes = 0
        for _ in range(10):
            nids, nsc, nfr, ch = o.knn_iterate_range(st, ids, sc, fr, lo, hi)
            full = []
            for arr in (nids, nsc, nfr):  # all-gather of the owned rows (padded equal slices)
                a = arr.view(np.int32) if arr.dtype == np.uint32 else arr  # (gloo has no uint32)
                mine = torch.zeros((cn, k), dtype=torch.from_numpy(a[:1]).dtype)
                mine[:hi - lo] = torch.from_numpy(a[lo:hi])
                parts = [torch.zeros_like(mine) for _ in range(world)]
                dist.all_gather(parts, mine)
                full.append(torch.cat(parts)[:n].numpy().view(arr.dtype))
            ids, sc, fr = full
            t = torch.tensor([ch], dtype=torch.int64)
            dist.all_reduce(t)
            passes += 1
            if int(t.item()) / (n * k) < 0.01:
                break
        out[rank] = (ids.tolist(), sc.tolist(), passes)
    finally:
        dist.destroy_process_group()


def test_two_rank_vertex_range_knn_matches_single_process(oracle):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_knn_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_2511_00855_b200 import _abi as A, synth
    p = A.synth_params(docs=300, dense_dim=8, learned_vocab=400, learned_nnz=8,
                       statistical_vocab=400, statistical_nnz=6, seed=9)
    c, kg, _ = synth.generate_corpus(p, 1)
    st = oracle.store(c, kg)
    ids, sc, fr = oracle.knn_build(st, c.n, 12, max_iterations=10, seed=42)
    assert out[0][0] == out[1][0] == ids.tolist()                  # identical on every rank
    assert np.array_equal(np.array(out[0][1]).view(np.uint64), sc.view(np.uint64))  # bitwise scores
    assert out[0][2] == out[1][2] > 1                              # same convergence decision
