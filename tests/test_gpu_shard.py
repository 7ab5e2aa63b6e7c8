"""Vertex-range sharded construction (fg_index_build_sharded).

On one GPU the G ranks' ranges run in this process (sim_ranks = G: every
rank writes its slice of the same buffers, which is what the NCCL all-gather
produces on G GPUs).  The index must be identical to the unsharded build and
to the unmodified reference for every G — the NN-Descent passes are
double-buffered (knn_graph.cpp:91,141-144) and the refinery is per node."""
import os

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def corpus3k():
    p = A.synth_params(docs=3001, dense_dim=64, learned_vocab=5000, learned_nnz=24,
                       statistical_vocab=5000, statistical_nnz=16, entity_vocab=400,
                       kg_triplets=1500, chains=10, answers_per_chain=4, seed=13)
    c, kg, _ = synth.generate_corpus(p, 0)
    return p, c, kg, fg.DeviceCorpus(c)


def same_index(a, b):
    for key in ("semantic", "norm_order", "logical_ptr", "logical"):
        assert np.array_equal(a[key], b[key]), key
    assert np.array_equal(a["keyword"].ptr, b["keyword"].ptr)
    assert np.array_equal(a["keyword"].idx, b["keyword"].idx)


BUILD = dict(degree=16, knn_k=32, knn_iterations=10, seed=42, logical_cap=16)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_sharded_build_equals_single(corpus3k, G):
    p, c, kg, dc = corpus3k
    want = fg.build_hybrid_index(dc, kg, **BUILD).export()
    got = fg.build_hybrid_index_sharded(dc, kg, sim_ranks=G, **BUILD).export()
    same_index(got, want)


def test_sharded_build_equals_reference(corpus3k, ref):
    p, c, kg, dc = corpus3k
    got = fg.build_hybrid_index_sharded(dc, kg, sim_ranks=4, **BUILD).export()
    rix = ref.index_build(ref.store(c, kg), threads=os.cpu_count() or 1, **BUILD)
    same_index(got, ref.index_export(rix, c.n))


def test_single_rank_communicator(corpus3k):
    """fg_comm_* with one rank: NCCL loads, the build runs through the comm path."""
    p, c, kg, dc = corpus3k
    comm = fg.Comm(1, 0, fg.Comm.unique_id(), 0)
    got = fg.build_hybrid_index_sharded(dc, kg, comm=comm, **BUILD).export()
    comm.close()
    same_index(got, fg.build_hybrid_index(dc, kg, **BUILD).export())


# ------------------------------------------------ real ranks, one GPU
def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def _shard_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = A.synth_params(docs=3001, dense_dim=64, learned_vocab=5000, learned_nnz=24,
                           statistical_vocab=5000, statistical_nnz=16, entity_vocab=400,
                           kg_triplets=1500, chains=10, answers_per_chain=4, seed=13)
        c, kg, _ = synth.generate_corpus(p, 0)
        dc = fg.DeviceCorpus(c, device=0)
        comm = fg.HostComm(world, rank, 0)
        ix = fg.build_hybrid_index_sharded(dc, kg, comm=comm, **BUILD)
        g = ix.export()
        out[rank] = (g["semantic"].tobytes(), g["keyword"].idx.tobytes(), g["norm_order"].tobytes())
        ix.close()
        comm.close()
        dc.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_process_sharded_build(corpus3k, world):
    """`world` real ranks (processes), each its own CUDA context on GPU 0 and
    its own vertex range, exchanging each pass's lists through the host
    communicator (gloo): every rank ends with the single-process index."""
    import torch.multiprocessing as mp
    p, c, kg, dc = corpus3k
    want = fg.build_hybrid_index(dc, kg, **BUILD).export()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        sem, kw, no = out[r]
        assert sem == want["semantic"].tobytes(), r
        assert kw == want["keyword"].idx.tobytes(), r
        assert no == want["norm_order"].tobytes(), r
