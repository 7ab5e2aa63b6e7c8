"""Golden vectors made by the UNMODIFIED reference (tests/golden/make_golden.py)
checked against (a) the CPU restatement oracle — no GPU, runs everywhere —
and (b) the GPU path through the C-ABI (-m gpu).  Comparisons are bitwise.
"""
import os

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden_small.npz"))
PARAMS = dict(docs=600, dense_dim=16, learned_vocab=1200, learned_nnz=12, statistical_vocab=1200,
              statistical_nnz=10, entity_vocab=120, kg_triplets=400, chains=6,
              answers_per_chain=3, seed=21)
BUILD = dict(degree=6, knn_k=12, knn_iterations=10, seed=5, logical_cap=8)


def u64(x):
    return np.asarray(x).view(np.uint64)


def corpus():
    c = A.Corpus(G["dense"], A.CSR(G["lptr"], G["lidx"], G["lval"]),
                 A.CSR(G["sptr"], G["sidx"], G["sval"]), None, A.CSR(G["eptr"], G["eidx"]))
    return c, A.KG(G["kg_s"], G["kg_r"], G["kg_t"])


def queries():
    from paper_2511_00855_b200 import synth
    p = A.synth_params(**PARAMS)
    q = synth.synth_queries(p, 24, k=8, beam_width=20)
    rows = [q.statistical.row(i)[0][: i % 3].tolist() if i % 4 == 0 else [] for i in range(24)]
    q.required = A.CSR.from_rows(rows)
    q.k[5] = 0
    return q


def check_results(prefix, r):
    assert np.array_equal(r.hit_count, G[f"{prefix}_count"])
    for i in range(r.count):
        h = int(r.hit_count[i])
        assert np.array_equal(r.doc_id[i, :h], G[f"{prefix}_doc"][i, :h]), i
        assert np.array_equal(u64(r.score[i, :h]), u64(G[f"{prefix}_score"][i, :h])), i
        assert r.error(i) == str(G[f"{prefix}_err"][i])
    assert np.array_equal(r.warnings, G[f"{prefix}_warn"])


def test_generator_reproduces_golden_corpus():
    from paper_2511_00855_b200 import synth
    c, kg, _ = synth.generate_corpus(A.synth_params(**PARAMS), 2)
    assert np.array_equal(c.dense.view(np.uint32), G["dense"].view(np.uint32))
    assert np.array_equal(c.learned.idx, G["lidx"]) and np.array_equal(c.statistical.idx, G["sidx"])
    assert np.array_equal(c.learned.val.view(np.uint32), G["lval"].view(np.uint32))
    assert np.array_equal(kg.source, G["kg_s"]) and np.array_equal(kg.target, G["kg_t"])


def test_oracle_matches_golden(oracle):
    c, kg = corpus()
    st = oracle.store(c, kg)
    assert np.array_equal(u64(oracle.sqnorm(st, c.n)), u64(G["sqnorm"]))
    q = queries()
    ids = np.arange(c.n, dtype=np.uint32)
    assert np.array_equal(u64(oracle.batch_scores(st, q, 0, ids)), u64(G["scores_q0"]))
    i0 = oracle.knn_init(st, c.n, BUILD["knn_k"], BUILD["seed"])
    assert np.array_equal(i0[0], G["init_ids"]) and np.array_equal(u64(i0[1]), u64(G["init_sc"]))
    i1 = oracle.knn_iterate(st, *i0)
    assert np.array_equal(i1[0], G["pass_ids"]) and i1[3] == int(G["pass_changed"])
    kb = oracle.knn_build(st, c.n, BUILD["knn_k"], max_iterations=10, seed=BUILD["seed"])
    assert np.array_equal(kb[0], G["knn_ids"]) and np.array_equal(kb[2], G["knn_fr"])
    sem, kw, tr = oracle.refine(st, *kb, degree=BUILD["degree"], trace=True)
    assert np.array_equal(sem, G["ref_sem"]) and np.array_equal(tr["ordered_ids"], G["ref_ord"])
    assert np.array_equal(tr["detours"], G["ref_det"])
    ix = oracle.index_build(oracle.store(c, kg), **BUILD)
    g = oracle.index_export(ix, c.n)
    assert np.array_equal(g["semantic"], G["ix_sem"]) and np.array_equal(g["logical"], G["ix_lg"])
    assert np.array_equal(g["norm_order"], G["ix_norm"])
    check_results("plain", oracle.batch_query(ix, q))
    check_results("truth", oracle.brute_force(oracle.store(c, kg), q.with_(k=8)))


@pytest.mark.gpu
def test_gpu_matches_golden():
    from paper_2511_00855_b200 import fusegraph as fg
    c, kg = corpus()
    dc = fg.DeviceCorpus(c)
    assert np.array_equal(u64(dc.sqnorm()), u64(G["sqnorm"]))
    q = queries()
    ids = np.arange(c.n, dtype=np.uint32)
    assert np.array_equal(u64(fg.batch_scores(dc, q, 1, ids)), u64(G["scores_q1"]))
    i0 = fg.init_random_graph(dc, BUILD["knn_k"], BUILD["seed"])
    assert np.array_equal(i0[0], G["init_ids"])
    i1 = fg.nn_descent_iterate(dc, *i0)
    assert np.array_equal(i1[0], G["pass_ids"]) and np.array_equal(u64(i1[1]), u64(G["pass_sc"]))
    assert np.array_equal(i1[2], G["pass_fr"]) and i1[3] == int(G["pass_changed"])
    kb = fg.build_knn_graph(dc, k=BUILD["knn_k"], max_iterations=10, seed=BUILD["seed"])
    assert np.array_equal(kb[0], G["knn_ids"]) and np.array_equal(u64(kb[1]), u64(G["knn_sc"]))
    sem, kw, tr = fg.refine_graph(dc, *kb[:3], degree=BUILD["degree"], trace=True)
    assert np.array_equal(sem, G["ref_sem"]) and np.array_equal(tr["detours"], G["ref_det"])
    assert np.array_equal(np.array([len(x) for x in kw]), G["ref_kwc"])
    ix = fg.build_hybrid_index(dc, kg, **BUILD)
    g = ix.export()
    assert np.array_equal(g["semantic"], G["ix_sem"])
    assert np.array_equal(g["keyword"].idx, G["ix_kidx"]) and np.array_equal(g["logical"], G["ix_lg"])
    check_results("plain", fg.batch_query(ix, q))
    check_results("truth", fg.brute_force_topk(dc, q.with_(k=8)))
