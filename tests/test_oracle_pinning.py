"""CPU: pin the restatement oracle (oracle/fg_oracle.cpp) to the UNMODIFIED
reference (oracle/_ref) — every stage bit for bit — and pin the product's
host-side generator to the reference's generate_corpus.  No GPU needed."""
import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A, synth


def corpus_of(**kw):
    p = A.synth_params(**kw)
    return (p,) + synth.generate_corpus(p, 0)


def bits(x):
    return np.asarray(x).view(np.uint64 if np.asarray(x).dtype == np.float64 else np.uint32)


@pytest.mark.parametrize("kw", [
    dict(docs=400, dense_dim=16),
    dict(docs=900, dense_dim=24, entity_vocab=80, kg_triplets=200, chains=4, answers_per_chain=3),
    dict(docs=1500, dense_dim=128, learned_vocab=30000, learned_nnz=64, statistical_vocab=30000,
         statistical_nnz=64, seed=7),
    dict(docs=200, dense_dim=8, learned_vocab=10, learned_nnz=20, statistical_vocab=0,
         statistical_nnz=40),
])
def test_generator_matches_reference(ref, kw):
    p = A.synth_params(**kw)
    c1, g1, ch1 = synth.generate_corpus(p, 4)
    c2, g2, nch = ref.generate_corpus(p)
    assert np.array_equal(bits(c1.dense), bits(c2.dense))
    for f in ("learned", "statistical"):
        a, b = getattr(c1, f), getattr(c2, f)
        assert np.array_equal(a.ptr, b.ptr) and np.array_equal(a.idx, b.idx)
        assert np.array_equal(bits(a.val), bits(b.val))
    for f in ("keywords", "entities"):
        a, b = getattr(c1, f), getattr(c2, f)
        assert np.array_equal(a.ptr, b.ptr) and np.array_equal(a.idx, b.idx)
    assert np.array_equal(g1.source, g2.source) and np.array_equal(g1.target, g2.target)
    assert np.array_equal(g1.relation, g2.relation)
    assert (c1.learned_dim, c1.statistical_dim, len(ch1)) == (c2.learned_dim, c2.statistical_dim, nch)
    q1 = synth.synth_queries(p, 25)
    d, li, lv, si, sv, w = ref.synth_queries(p, 25)
    assert np.array_equal(bits(q1.dense), bits(d)) and np.array_equal(q1.learned.idx, li)
    assert np.array_equal(bits(q1.learned.val), bits(lv)) and np.array_equal(q1.statistical.idx, si)
    assert np.array_equal(bits(q1.statistical.val), bits(sv)) and np.array_equal(bits(q1.weights), bits(w))


@pytest.fixture(scope="module")
def case():
    return corpus_of(docs=700, dense_dim=16, learned_vocab=1500, learned_nnz=14,
                     statistical_vocab=1500, statistical_nnz=10, entity_vocab=150,
                     kg_triplets=500, chains=8, answers_per_chain=4, seed=11)


def test_scores_pinned(ref, oracle, case):
    p, c, kg, chains = case
    rs, os_ = ref.store(c, kg), oracle.store(c, kg)
    assert np.array_equal(bits(ref.sqnorm(rs, c.n)), bits(oracle.sqnorm(os_, c.n)))
    q = synth.synth_queries(p, 5)
    q.weights[1, 0] = 0
    q.weights[2, 2] = 0
    ids = np.arange(c.n, dtype=np.uint32)
    for i in range(q.count):
        assert np.array_equal(bits(ref.batch_scores(rs, q, i, ids)), bits(oracle.batch_scores(os_, q, i, ids)))
        r, o = ref.build_query_vector(q, i), oracle.build_query_vector(q, i)
        assert all(np.array_equal(bits(x), bits(y)) for x, y in zip(r[:3], o[:3])) and r[3] == o[3]


def test_knn_and_refine_pinned(ref, oracle, case):
    p, c, kg, chains = case
    rs, os_ = ref.store(c, kg), oracle.store(c, kg)
    r0, o0 = ref.knn_init(rs, c.n, 12, 5), oracle.knn_init(os_, c.n, 12, 5)
    for x, y in zip(r0, o0):
        assert np.array_equal(x, y)
    cur = r0
    for _ in range(2):
        r1, o1 = ref.knn_iterate(rs, *cur), oracle.knn_iterate(os_, *cur)
        for x, y in zip(r1, o1):
            assert np.array_equal(np.asarray(x), np.asarray(y))
        cur = r1[:3]
    lists = ref.knn_build(rs, c.n, 12, seed=5)
    assert all(np.array_equal(x, y) for x, y in zip(lists, oracle.knn_build(os_, c.n, 12, seed=5)))
    for per in (False, True):
        rsem, rkw, rt = ref.refine(rs, *lists, degree=6, per_neighbour=per, trace=True)
        osem, okw, ot = oracle.refine(os_, *lists, degree=6, per_neighbour=per, trace=True)
        assert np.array_equal(rsem, osem)
        assert all(np.array_equal(a, b) for a, b in zip(rkw, okw))
        for key in ("ordered_ids", "detours", "kept_count"):
            assert np.array_equal(rt[key], ot[key])


def _same(g, r, expanded=True):
    assert np.array_equal(g.hit_count, r.hit_count)
    for i in range(g.count):
        assert g.error(i) == r.error(i)
        h = int(g.hit_count[i])
        assert np.array_equal(g.doc_id[i, :h], r.doc_id[i, :h])
        assert np.array_equal(bits(g.score[i, :h]), bits(r.score[i, :h]))
    assert np.array_equal(g.warnings, r.warnings)
    if expanded:
        assert np.array_equal(g.expanded, r.expanded)


def test_index_and_search_pinned(ref, oracle, case):
    p, c, kg, chains = case
    rix = ref.index_build(ref.store(c, kg), degree=6, knn_k=12, seed=5, logical_cap=8)
    oix = oracle.index_build(oracle.store(c, kg), degree=6, knn_k=12, seed=5, logical_cap=8)
    rg, og = ref.index_export(rix, c.n), oracle.index_export(oix, c.n)
    for key in ("semantic", "logical_ptr", "logical", "norm_order"):
        assert np.array_equal(rg[key], og[key]), key
    assert np.array_equal(rg["keyword"].idx, og["keyword"].idx)
    q = synth.synth_queries(p, 30, beam_width=24)
    _same(oracle.batch_query(oix, q), ref.batch_query(rix, q))
    rows = [q.statistical.row(i)[0][: (i % 3)].tolist() for i in range(q.count)]
    q.required = A.CSR.from_rows(rows)
    for conj in (True, False):
        _same(oracle.batch_query(oix, q, conjunctive=conj), ref.batch_query(rix, q, conjunctive=conj))
    dense = np.stack([ch.query_dense for ch in chains])
    learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
    stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains], [ch.query_statistical[1] for ch in chains])
    for went in (100.0, 0.0):
        w = np.tile(np.array([[1, 1, 1, went]], np.float32), (len(chains), 1))
        qe = A.Queries(dense, learned, stat, w, k=10, beam_width=32,
                       entities=A.CSR.from_rows([[ch.e0] for ch in chains]))
        _same(oracle.batch_query(oix, qe), ref.batch_query(rix, qe))
    _same(oracle.brute_force(oracle.store(c, kg), q), ref.brute_force(ref.store(c, kg), q), False)
