"""GPU parity at a realistic size: the configs[0] shape (10K docs, d=128,
learned + statistical nnz 64, vocab 30K) built and searched on the B200 and
by the unmodified reference (all host threads) — identical index, identical
hits, bitwise scores.  Also checks the full-size (bench) invariants that
need no reference: structural validity of a built index."""
import os

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth

pytestmark = pytest.mark.gpu

C1 = dict(docs=10000, dense_dim=128, clusters=20, cluster_spread=0.25, learned_vocab=30000,
          learned_nnz=64, statistical_vocab=30000, statistical_nnz=64, seed=1)


def test_c1_build_and_search_identical_to_reference(ref):
    p = A.synth_params(**C1)
    c, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    gix = fg.build_hybrid_index(dc, kg, degree=32, knn_k=32, knn_iterations=10, seed=42)
    rix = ref.index_build(ref.store(c, kg), degree=32, knn_k=32, knn_iterations=10, seed=42,
                          threads=os.cpu_count() or 1)
    g, r = gix.export(), ref.index_export(rix, c.n)
    assert np.array_equal(g["semantic"], r["semantic"])
    assert np.array_equal(g["keyword"].ptr, r["keyword"].ptr)
    assert np.array_equal(g["keyword"].idx, r["keyword"].idx)
    assert np.array_equal(g["norm_order"], r["norm_order"])
    q = synth.synth_queries(p, 300, beam_width=128)
    gr = fg.batch_query(gix, q)
    rr = ref.batch_query(rix, q, threads=os.cpu_count() or 1)
    assert np.array_equal(gr.hit_count, rr.hit_count)
    assert np.array_equal(gr.doc_id, rr.doc_id)
    assert np.array_equal(gr.score.view(np.uint64), rr.score.view(np.uint64))
    assert np.array_equal(gr.expanded, rr.expanded)
    # recall@10 against exhaustive truth is therefore equal too
    t = fg.brute_force_topk(dc, q)
    rec = np.mean([fg.recall_at_k(gr.ids(i), t.ids(i), 10) for i in range(q.count)])
    assert rec > 0.5


def test_built_index_invariants():
    p = A.synth_params(**dict(C1, docs=20000, seed=3))
    c, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    ix = fg.build_hybrid_index(dc, kg, degree=16, knn_k=32, seed=42)
    g = ix.export()
    sem = g["semantic"]
    n = c.n
    assert sem.shape == (n, 16) and (sem < n).all()
    assert not (sem == np.arange(n)[:, None]).any()                      # no self loops
    assert (np.sort(sem, axis=1)[:, 1:] != np.sort(sem, axis=1)[:, :-1]).all()  # no duplicates
    kp, ki = g["keyword"].ptr, g["keyword"].idx
    for u in range(0, n, 97):                                             # keyword/semantic disjoint
        assert not np.intersect1d(ki[kp[u]:kp[u + 1]], sem[u]).size
    sq = dc.sqnorm()[g["norm_order"]]
    assert (np.diff(sq) <= 0).all()                                       # norm order
