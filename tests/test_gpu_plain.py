"""GPU parity of the plain-query search kernel (search_plain.cu).

Plain batches (no entity context, no required keywords) run the certified-
approximate kernel: warp-cooperative scores within a rigorous error bound,
every uncertain comparison re-scored with the reference's exact chain, the
final top-k re-scored exactly.  These tests pin it against the UNMODIFIED
reference bit for bit, including with the error bound inflated by 1e9 so that
the exact-resolution paths run on almost every comparison, and on corpora
built of duplicated documents (exact score ties, node-id tie-breaks).
"""
import os

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth

pytestmark = pytest.mark.gpu


class env:
    def __init__(self, **kw):
        self.kw = {k: str(v) for k, v in kw.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kw}
        os.environ.update(self.kw)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def same(g, r):
    assert np.array_equal(g.hit_count, r.hit_count)
    for i in range(g.count):
        h = int(g.hit_count[i])
        assert g.error(i) == r.error(i), i
        assert np.array_equal(g.node[i, :h], r.node[i, :h]), i
        assert np.array_equal(g.doc_id[i, :h], r.doc_id[i, :h]), i
        assert np.array_equal(g.score[i, :h].view(np.uint64), r.score[i, :h].view(np.uint64)), i
    assert np.array_equal(g.expanded, r.expanded)
    assert np.array_equal(g.warnings, r.warnings)


@pytest.fixture(scope="module")
def c2_small(ref):
    """configs[1] row shape (d=768, learned nnz 120, vocab 30,522) at 4K docs."""
    p = A.synth_params(docs=4000, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30522,
                       learned_nnz=120, statistical_vocab=0, statistical_nnz=40, seed=7)
    c, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    gix = fg.build_hybrid_index(dc, kg, degree=16, knn_k=32, seed=42)
    rix = ref.index_create(ref.store(c, kg), gix.export(), 32)
    return p, c, dc, gix, rix


@pytest.mark.parametrize("beam,entry", [(10, 32), (64, 32), (128, 256), (512, 64)])
def test_plain_c2_shape_identical(c2_small, ref, beam, entry):
    p, c, dc, gix, rix = c2_small
    q = synth.synth_queries(p, 48, beam_width=beam)
    g = fg.batch_query(gix, q, entry_count=entry)
    same(g, ref.batch_query(rix, q, entry_count=entry, threads=os.cpu_count() or 1))
    with env(FGB_SEARCH_PLAIN=0):  # the general (sequential-chain) kernel agrees too
        same(fg.batch_query(gix, q, entry_count=entry), g)
    with env(FGB_SEARCH_CUCKOO=0):  # bitmap + rank lookups instead of the cuckoo tables
        same(fg.batch_query(gix, q, entry_count=entry), g)
    with env(FGB_SEARCH_CUCKOO=0, FGB_SEARCH_BITMAP=0):  # filter + hash lookups
        same(fg.batch_query(gix, q, entry_count=entry), g)


def test_plain_c3_shape_identical(ref):
    """configs[2] row shape: learned vocab 30,522 (bitmap-sized) + statistical
    vocab 831,592 (hash-sized); the batch then takes the hash for both paths.
    Per-query simplex weights over the three paths."""
    p = A.synth_params(docs=3000, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30522,
                       learned_nnz=120, statistical_vocab=831592, statistical_nnz=40, seed=8)
    c, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    gix = fg.build_hybrid_index(dc, kg, degree=16, knn_k=32, seed=42)
    rix = ref.index_create(ref.store(c, kg), gix.export(), 32)
    q = synth.synth_queries(p, 48, beam_width=128)
    g = fg.batch_query(gix, q, entry_count=64)
    same(g, ref.batch_query(rix, q, entry_count=64, threads=os.cpu_count() or 1))
    # learned path alone (statistical weight 0): the learned bitmap again
    q.weights[:, 2] = 0.0
    same(fg.batch_query(gix, q, entry_count=64), ref.batch_query(rix, q, entry_count=64,
                                                                  threads=os.cpu_count() or 1))


def test_plain_forced_exact_resolution(c2_small, ref):
    """Error bound x1e9: nearly every comparison is 'uncertain' and resolved
    through the exact chain — results must not change."""
    p, c, dc, gix, rix = c2_small
    q = synth.synth_queries(p, 24, beam_width=96)
    want = ref.batch_query(rix, q, entry_count=64, threads=os.cpu_count() or 1)
    with env(FGB_EPS_SCALE="1e9"):
        same(fg.batch_query(gix, q, entry_count=64), want)
    with env(FGB_EPS_SCALE="1e15"):
        same(fg.batch_query(gix, q, entry_count=64), want)


def test_plain_duplicate_documents_ties(ref):
    """Every document appears 3 times: identical scores everywhere, so order
    is decided by node id through the exact-resolution path."""
    p = A.synth_params(docs=600, dense_dim=64, learned_vocab=2000, learned_nnz=24, statistical_vocab=2000,
                       statistical_nnz=12, seed=11)
    c, kg, _ = synth.generate_corpus(p, 0)
    rep = lambda x: np.concatenate([x, x, x])  # noqa: E731

    def rep_csr(m):
        rows = [m.row(i) for i in range(c.n)] * 3
        return A.CSR.from_rows([r[0] for r in rows], [r[1] for r in rows] if m.val is not None else None)

    n3 = 3 * c.n
    c3 = A.Corpus(rep(c.dense), rep_csr(c.learned), rep_csr(c.statistical), rep_csr(c.keywords),
                  A.CSR.from_rows([[] for _ in range(n3)]), np.arange(n3, dtype=np.uint64),
                  np.zeros(n3, np.uint8), c.learned_dim, c.statistical_dim)
    dc = fg.DeviceCorpus(c3)
    gix = fg.build_hybrid_index(dc, None, degree=8, knn_k=16, seed=42)
    rix = ref.index_create(ref.store(c3, None), gix.export(), 16)
    q = synth.synth_queries(p, 40, beam_width=40)
    same(fg.batch_query(gix, q, entry_count=48), ref.batch_query(rix, q, entry_count=48))


def test_plain_deleted_and_d128(ref):
    p = A.synth_params(docs=3000, dense_dim=128, learned_vocab=30000, learned_nnz=64,
                       statistical_vocab=30000, statistical_nnz=64, seed=2)
    c, kg, _ = synth.generate_corpus(p, 0)
    flags = np.zeros(c.n, np.uint8)
    flags[np.random.default_rng(5).choice(c.n, 400, replace=False)] = 1
    dc0 = fg.DeviceCorpus(c)
    g = fg.build_hybrid_index(dc0, kg, degree=16, knn_k=32, seed=42).export()
    cd = A.Corpus(c.dense, c.learned, c.statistical, c.keywords, c.entities, c.doc_id, flags,
                  c.learned_dim, c.statistical_dim)
    dc = fg.DeviceCorpus(cd)
    gix = fg.HybridIndex.from_graph(dc, g, kg)
    rix = ref.index_create(ref.store(cd, kg), g, 32)
    q = synth.synth_queries(p, 64, beam_width=100)
    same(fg.batch_query(gix, q, entry_count=100), ref.batch_query(rix, q, entry_count=100))


def test_plain_buffer_reuse_and_pinned_inputs(c2_small, ref):
    """batch_query reuses its device/pinned buffers across calls: a large
    batch, then a small one, then an invalid-query batch, then pinned inputs —
    each must match the reference exactly (no stale rows from a prior call)."""
    p, c, dc, gix, rix = c2_small
    big = synth.synth_queries(p, 64, beam_width=64)
    small = big.subset(np.arange(5)).with_(beam_width=32)
    bad = small.with_(k=np.array([10, 0, 10, 10, 10], np.uint32))  # query 1: invalid-k
    thr = os.cpu_count() or 1
    same(fg.batch_query(gix, big, entry_count=32), ref.batch_query(rix, big, entry_count=32, threads=thr))
    same(fg.batch_query(gix, small, entry_count=32), ref.batch_query(rix, small, entry_count=32, threads=thr))
    g = fg.batch_query(gix, bad, entry_count=32)
    same(g, ref.batch_query(rix, bad, entry_count=32, threads=thr))
    assert g.error(1).startswith("invalid-k") and g.hit_count[1] == 0
    same(fg.batch_query(gix, big.pinned(), entry_count=32), ref.batch_query(rix, big, entry_count=32, threads=thr))


def test_plain_hbm_cand_pool_identical(c2_small, ref, monkeypatch):
    """Beams above kGpoolBeam keep the cand pool in HBM instead of shared
    memory (search.cu); forced on here at small beams, results unchanged."""
    monkeypatch.setenv("FGB_SEARCH_GPOOL", "1")
    p, c, dc, gix, rix = c2_small
    for beam in (96, 2100):  # (2100: above the threshold without the override)
        q = synth.synth_queries(p, 32, beam_width=beam)
        same(fg.batch_query(gix, q, entry_count=64), ref.batch_query(rix, q, entry_count=64))
        assert gix.last_search_kernel() == "search_plain_kernel"


@pytest.mark.parametrize("variant", ["cuckoo", "hash", "cuckoo-fallback"])
def test_plain_hash_vocab_lookup_variants(ref, monkeypatch, variant):
    """Batches run two-choice cuckoo tables by default; with a hash-sized
    statistical vocabulary (831,592) the filter + hash layout (FGB_SEARCH_CUCKOO=0)
    and the fallback after a failed cuckoo build (test hook: half the queries
    fail, the batch re-runs with hash lookups) give the same results."""
    if variant == "hash":
        monkeypatch.setenv("FGB_SEARCH_CUCKOO", "0")
    if variant == "cuckoo-fallback":
        monkeypatch.setenv("FGB_SEARCH_PREFETCH", str(5 | 0x100))
    p = A.synth_params(docs=3000, dense_dim=96, learned_vocab=30522, learned_nnz=60, statistical_vocab=831592,
                       statistical_nnz=40, seed=12)
    c, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    gix = fg.build_hybrid_index(dc, kg, degree=16, knn_k=32, seed=42)
    rix = ref.index_create(ref.store(c, kg), gix.export(), 32)
    q = synth.synth_queries(p, 80, beam_width=96)
    same(fg.batch_query(gix, q, entry_count=64), ref.batch_query(rix, q, entry_count=64))
    assert gix.last_search_kernel() == "search_plain_kernel"
