"""insert_batch on the device index (update.cpp:33-197) against
the UNMODIFIED reference's insert_batch on the identical index: every
semantic / keyword / logical list, the norm order and subsequent search
results must be identical; a rejected batch leaves the index untouched."""
import numpy as np
import pytest

from paper_2511_00855_b200 import Error, _abi as A, fusegraph as fg, synth

pytestmark = pytest.mark.gpu


def part(c: A.Corpus, rows) -> A.Corpus:
    rows = np.asarray(rows)
    return A.Corpus(c.dense[rows], c.learned.subset(rows), c.statistical.subset(rows), c.keywords.subset(rows),
                    c.entities.subset(rows), c.doc_id[rows], np.zeros(len(rows), np.uint8), c.learned_dim,
                    c.statistical_dim)


def same(a, b):
    for key in ("semantic", "norm_order", "logical_ptr", "logical"):
        assert np.array_equal(a[key], b[key]), key
    assert np.array_equal(a["keyword"].ptr, b["keyword"].ptr)
    assert np.array_equal(a["keyword"].idx, b["keyword"].idx)


@pytest.fixture(scope="module")
def split(ref):
    p = A.synth_params(docs=1400, dense_dim=48, learned_vocab=3000, learned_nnz=20, statistical_vocab=3000,
                       statistical_nnz=14, entity_vocab=300, kg_triplets=1200, chains=8, answers_per_chain=3,
                       seed=31)
    c, kg, _ = synth.generate_corpus(p, 0)
    return p, c, kg


@pytest.mark.parametrize("batch", [1, 37, 200])
def test_insert_matches_reference(split, ref, batch):
    p, c, kg = split
    n0 = c.n - 200
    base, new = part(c, np.arange(n0)), part(c, np.arange(n0, n0 + batch))
    build = dict(degree=10, knn_k=20, seed=42, logical_cap=16)
    rix = ref.index_build(ref.store(base, kg), **build)
    ref.index_insert(rix, new)
    gix = fg.build_hybrid_index(fg.DeviceCorpus(base), kg, **build)
    gix.insert(new)
    same(gix.export(), ref.index_export(rix, n0 + batch))
    q = synth.synth_queries(p, 40, beam_width=48)
    g, r = fg.batch_query(gix, q, entry_count=40), ref.batch_query(rix, q, entry_count=40)
    assert np.array_equal(g.doc_id, r.doc_id)
    assert np.array_equal(g.score.view(np.uint64), r.score.view(np.uint64))
    assert np.array_equal(g.expanded, r.expanded)


def test_insert_rejects_duplicates_untouched(split):
    p, c, kg = split
    base = part(c, np.arange(600))
    gix = fg.build_hybrid_index(fg.DeviceCorpus(base), kg, degree=10, knn_k=20, seed=42)
    before = gix.export()
    with pytest.raises(Error) as e:
        gix.insert(part(c, np.array([650, 5])))          # doc 5 is already indexed
    assert e.value.code == "duplicate-id"
    with pytest.raises(Error) as e:
        gix.insert(part(c, np.array([650, 650])))        # repeated within the batch
    assert e.value.code == "duplicate-id"
    same(gix.export(), before)
