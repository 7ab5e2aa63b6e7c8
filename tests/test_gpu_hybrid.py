"""The certified-approximate kernel for entity-context and required-keyword
batches (csrc/search_hybrid.cu; search.cpp:141-280) against the UNMODIFIED
reference's batch_query on the same index, at the C4 row shape: dense d=768,
learned vocab 30,522 nnz 120, statistical vocab 831,592 nnz 40 (hash
lookups), KG logical edges, degree 32 / knn_k 64.

The index is built on the GPU (its parity is test_gpu_bench_shape.py's and
test_gpu_parity.py's subject) and handed to the reference through
index_create, so the reference only searches.  Every query's hit ids, score
bits, hit count, warnings and `expanded` must be identical.
"""
import os

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def c4(ref):
    p = A.synth_params(docs=16000, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30522,
                       learned_nnz=120, statistical_vocab=831592, statistical_nnz=40, entity_vocab=3000,
                       entity_rate=0.3, max_entities_per_doc=2, kg_triplets=16000, relation_vocab=8, chains=48,
                       answers_per_chain=10, seed=7)
    c, kg, chains = synth.generate_corpus(p, 0)
    dev = fg.DeviceCorpus(c)
    gix = fg.build_hybrid_index(dev, kg, degree=32, knn_k=64, seed=42, logical_cap=64)
    rix = ref.index_create(ref.store(c, kg), gix.export(), 64)
    yield dict(p=p, c=c, kg=kg, chains=chains, dev=dev, gix=gix, rix=rix)
    gix.close()
    dev.close()


def same(g, r):
    assert np.array_equal(g.hit_count, r.hit_count)
    for i in range(g.count):
        assert g.error(i) == r.error(i), i
        h = int(g.hit_count[i])
        assert np.array_equal(g.doc_id[i, :h], r.doc_id[i, :h]), i
        assert np.array_equal(g.score[i, :h].view(np.uint64), r.score[i, :h].view(np.uint64)), i
    assert np.array_equal(g.warnings, r.warnings)
    assert np.array_equal(g.expanded, r.expanded)


def chain_queries(chains, went, beam=128, hops=2):
    dense = np.stack([ch.query_dense for ch in chains])
    learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
    stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains], [ch.query_statistical[1] for ch in chains])
    w = np.tile(np.array([[1, 1, 1, went]], np.float32), (len(chains), 1))
    ents = A.CSR.from_rows([[ch.e0] for ch in chains])
    return A.Queries(dense, learned, stat, w, k=10, beam_width=beam, max_entity_hops=hops, entities=ents)


def keyword_queries(p, count, beam, seed):
    q = synth.synth_queries(p, count, beam_width=beam)
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(q.count):
        si, _ = q.statistical.row(i)
        rows.append(sorted(set(rng.choice(si, size=1 + i % 3, replace=False).tolist())))
    q.required = A.CSR.from_rows(rows)
    return q


@pytest.mark.parametrize("went,hops", [(100.0, 2), (0.5, 2), (100.0, 1), (100.0, 3)])
def test_chain_queries_identical(c4, ref, went, hops):
    q = chain_queries(c4["chains"], went, hops=hops)
    g = fg.batch_query(c4["gix"], q)
    assert c4["gix"].last_search_kernel() == "search_hybrid_kernel"
    same(g, ref.batch_query(c4["rix"], q, threads=THREADS))


@pytest.mark.parametrize("conj", [True, False])
def test_keyword_queries_identical(c4, ref, conj):
    q = keyword_queries(c4["p"], 96, 256, seed=3)
    g = fg.batch_query(c4["gix"], q, conjunctive=conj)
    assert c4["gix"].last_search_kernel() == "search_hybrid_kernel"
    same(g, ref.batch_query(c4["rix"], q, conjunctive=conj, threads=THREADS))


def test_mixed_batch_identical(c4, ref):
    """Entities + required keywords in one query, next to plain and
    keyword-only queries and an entity query whose entity is unknown
    (entity-fallback warning)."""
    chains = c4["chains"][:16]
    q = chain_queries(chains, 100.0, beam=192)
    rng = np.random.default_rng(9)
    rows = []
    for i in range(q.count):
        si, _ = q.statistical.row(i)
        rows.append(sorted(rng.choice(si, size=1, replace=False).tolist()) if i % 2 else [])
    q.required = A.CSR.from_rows(rows)
    ents = [[ch.e0] for ch in chains]
    ents[3] = [10 ** 7]                   # unknown entity -> norm seeds + warning
    ents[5] = []                          # entity weight without entities -> entities-required
    q.entities = A.CSR.from_rows(ents)
    q.weights[7, 3] = 0.0                 # entities but no entity weight: plain seeds
    g = fg.batch_query(c4["gix"], q)
    same(g, ref.batch_query(c4["rix"], q, threads=THREADS))


def test_forced_exact_resolution(c4, ref, monkeypatch):
    """eps x 1e9: almost every comparison is resolved by the exact chain."""
    monkeypatch.setenv("FGB_EPS_SCALE", "1e9")
    q = chain_queries(c4["chains"][:24], 100.0)
    same(fg.batch_query(c4["gix"], q), ref.batch_query(c4["rix"], q, threads=THREADS))
    q = keyword_queries(c4["p"], 32, 128, seed=5)
    same(fg.batch_query(c4["gix"], q), ref.batch_query(c4["rix"], q, threads=THREADS))


def test_deleted_nodes_identical(c4, ref):
    """Deleted nodes route through cand but never reach top-k or the twin pool."""
    c, kg = c4["c"], c4["kg"]
    flags = np.zeros(c.n, np.uint8)
    flags[np.random.default_rng(4).choice(c.n, 1600, replace=False)] = 1
    for ch in c4["chains"][:8]:
        flags[ch.answer_docs[:3].astype(np.int64)] = 1
    graph = c4["gix"].export()
    cd = A.Corpus(c.dense, c.learned, c.statistical, c.keywords, c.entities, c.doc_id, flags, c.learned_dim,
                  c.statistical_dim)
    dev2 = fg.DeviceCorpus(cd)
    gix2 = fg.HybridIndex.from_graph(dev2, graph, kg)
    rix2 = ref.index_create(ref.store(cd, kg), graph, 64)
    q = chain_queries(c4["chains"], 100.0)
    same(fg.batch_query(gix2, q), ref.batch_query(rix2, q, threads=THREADS))
    q = keyword_queries(c4["p"], 48, 192, seed=11)
    same(fg.batch_query(gix2, q), ref.batch_query(rix2, q, threads=THREADS))
    gix2.close()
    dev2.close()


def test_overflow_reruns_identical(c4, ref, monkeypatch):
    """2-slot initial twin pools / context tables: most queries overflow and
    re-run alone with 4x tables; results unchanged."""
    monkeypatch.setenv("FGB_SEARCH_SCRATCH0", "2")
    q = chain_queries(c4["chains"][:16], 100.0)
    g = fg.batch_query(c4["gix"], q)
    assert c4["gix"].last_search_stats()[1] >= 2
    same(g, ref.batch_query(c4["rix"], q, threads=THREADS))
    q = keyword_queries(c4["p"], 24, 256, seed=13)
    same(fg.batch_query(c4["gix"], q), ref.batch_query(c4["rix"], q, threads=THREADS))


@pytest.mark.parametrize("variant", ["hash", "cuckoo-fallback", "cuckoo-fallback+overflow"])
def test_lookup_variants_identical(c4, ref, monkeypatch, variant):
    """Cuckoo query tables are the default; the filter + hash lookups
    (FGB_SEARCH_CUCKOO=0) and the re-run after a failed cuckoo build (test
    hook: every even query fails; with overflowing scratch as well) agree."""
    if variant == "hash":
        monkeypatch.setenv("FGB_SEARCH_CUCKOO", "0")
    else:
        monkeypatch.setenv("FGB_SEARCH_PREFETCH", str(5 | 0x100))
    if variant.endswith("overflow"):
        monkeypatch.setenv("FGB_SEARCH_SCRATCH0", "2")
    q = chain_queries(c4["chains"][:16], 100.0)
    g = fg.batch_query(c4["gix"], q)
    assert c4["gix"].last_search_kernel() == "search_hybrid_kernel"
    if variant != "hash":
        assert c4["gix"].last_search_stats()[1] >= 2
    same(g, ref.batch_query(c4["rix"], q, threads=THREADS))
    q = keyword_queries(c4["p"], 24, 256, seed=13)
    same(fg.batch_query(c4["gix"], q), ref.batch_query(c4["rix"], q, threads=THREADS))
