"""ctypes mirror of include/fg_b200.h (the C-ABI), shared by the product
bindings, the oracle bindings and the tests.

Only structure layouts and numpy<->pointer plumbing live here; no compute.
"""
from __future__ import annotations

import ctypes as C
import numpy as np

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)


class SparseView(C.Structure):
    _fields_ = [("ptr", u64p), ("idx", u32p), ("val", f32p)]


class ListView(C.Structure):
    _fields_ = [("ptr", u64p), ("idx", u32p)]


class CorpusView(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("dense_dim", C.c_uint32), ("learned_dim", C.c_uint32),
        ("statistical_dim", C.c_uint32), ("dense", f32p), ("learned", SparseView),
        ("statistical", SparseView), ("keywords", ListView), ("entities", ListView),
        ("doc_id", u64p), ("deleted", u8p),
    ]


class Weights(C.Structure):
    _fields_ = [("dense", C.c_float), ("learned", C.c_float), ("statistical", C.c_float),
                ("entity", C.c_float)]


class QueryView(C.Structure):
    _fields_ = [
        ("count", C.c_uint64), ("dense_dim", C.c_uint32), ("dense", f32p),
        ("learned", SparseView), ("statistical", SparseView), ("weights", C.POINTER(Weights)),
        ("required_keywords", ListView), ("entities", ListView), ("k", u32p),
        ("beam_width", u32p), ("max_entity_hops", u32p),
    ]


class KgView(C.Structure):
    _fields_ = [("count", C.c_uint64), ("source", u32p), ("relation", u32p), ("target", u32p)]


class KnnLists(C.Structure):
    _fields_ = [("n", C.c_uint64), ("k", C.c_uint32), ("ids", u32p), ("scores", f64p),
                ("fresh", u8p)]


class KnnParams(C.Structure):
    _fields_ = [("k", C.c_uint32), ("max_iterations", C.c_uint32), ("convergence", C.c_double),
                ("seed", C.c_uint64)]


class RefineParams(C.Structure):
    _fields_ = [("degree", C.c_uint32), ("per_neighbour_keyword_check", C.c_int)]


class Refined(C.Structure):
    _fields_ = [("semantic", u32p), ("keyword_cap", C.c_uint32), ("keyword", u32p),
                ("keyword_count", u32p)]


class RefineTrace(C.Structure):
    _fields_ = [("ordered_ids", u32p), ("ordered_scores", f64p), ("detours", u32p),
                ("kept", u32p), ("kept_count", u32p)]


class BuildParams(C.Structure):
    _fields_ = [("degree", C.c_uint32), ("knn_k", C.c_uint32), ("knn_iterations", C.c_uint32),
                ("seed", C.c_uint64), ("logical_cap", C.c_uint32),
                ("default_entity_hops", C.c_uint32), ("per_neighbour_keyword_check", C.c_int)]


class GraphView(C.Structure):
    _fields_ = [("degree", C.c_uint32), ("semantic", u32p), ("keyword", ListView),
                ("logical_ptr", u64p), ("logical", u32p), ("norm_order", u32p)]


class SearchOpts(C.Structure):
    _fields_ = [("entry_count", C.c_uint32), ("conjunctive_filter", C.c_int)]


class SearchResults(C.Structure):
    _fields_ = [("hit_stride", C.c_uint32), ("doc_id", u64p), ("node", u32p), ("score", f64p),
                ("hit_count", u32p), ("expanded", u64p), ("scored", u64p), ("warnings", u32p),
                ("errors", C.c_char_p), ("error_stride", C.c_uint32)]


class SynthParams(C.Structure):
    _fields_ = [
        ("docs", C.c_uint32), ("dense_dim", C.c_uint32), ("clusters", C.c_uint32),
        ("cluster_spread", C.c_float), ("learned_vocab", C.c_uint32),
        ("learned_nnz", C.c_uint32), ("statistical_vocab", C.c_uint32),
        ("statistical_nnz", C.c_uint32), ("zipf_exponent", C.c_double),
        ("entity_vocab", C.c_uint32), ("entity_rate", C.c_double),
        ("max_entities_per_doc", C.c_uint32), ("kg_triplets", C.c_uint32),
        ("relation_vocab", C.c_uint32), ("chains", C.c_uint32),
        ("answers_per_chain", C.c_uint32), ("seed", C.c_uint64),
    ]


WARN_ENTITY_FALLBACK = 1
WARN_KEYWORD_SHORTFALL = 2


def ptr(a, t):
    """Pointer of a contiguous numpy array (None -> NULL)."""
    if a is None:
        return C.cast(None, t)
    assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
    return a.ctypes.data_as(t)


def arr(a, dtype):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- containers
class CSR:
    """Row pointer + indices (+ values) — one sparse path or id list."""

    __slots__ = ("ptr", "idx", "val")

    def __init__(self, ptr, idx, val=None):
        self.ptr = arr(ptr, np.uint64)
        self.idx = arr(idx, np.uint32)
        self.val = arr(val, np.float32)

    @staticmethod
    def empty(rows, with_val=True):
        return CSR(np.zeros(rows + 1, np.uint64), np.zeros(0, np.uint32),
                   np.zeros(0, np.float32) if with_val else None)

    @staticmethod
    def from_rows(rows, vals=None):
        lens = [len(r) for r in rows]
        p = np.zeros(len(rows) + 1, np.uint64)
        p[1:] = np.cumsum(lens)
        idx = np.array([x for r in rows for x in r], dtype=np.uint32)
        v = None
        if vals is not None:
            v = np.array([x for r in vals for x in r], dtype=np.float32)
        return CSR(p, idx, v)

    @staticmethod
    def fixed(idx2d, val2d=None):
        idx2d = np.asarray(idx2d)
        n, w = idx2d.shape
        p = np.arange(n + 1, dtype=np.uint64) * np.uint64(w)
        return CSR(p, idx2d.reshape(-1), None if val2d is None else np.asarray(val2d).reshape(-1))

    def row(self, i):
        b, e = int(self.ptr[i]), int(self.ptr[i + 1])
        return (self.idx[b:e], None if self.val is None else self.val[b:e])

    @property
    def rows(self):
        return len(self.ptr) - 1

    def subset(self, rows):
        rows = np.asarray(rows, dtype=np.int64)
        lens = (self.ptr[rows + 1] - self.ptr[rows]).astype(np.int64)
        p = np.zeros(len(rows) + 1, np.uint64)
        p[1:] = np.cumsum(lens)
        take = np.concatenate([np.arange(int(self.ptr[r]), int(self.ptr[r + 1])) for r in rows]) \
            if len(rows) else np.zeros(0, np.int64)
        take = take.astype(np.int64)
        return CSR(p, self.idx[take], None if self.val is None else self.val[take])

    def sparse_view(self):
        return SparseView(ptr(self.ptr, u64p), ptr(self.idx, u32p), ptr(self.val, f32p))

    def list_view(self):
        return ListView(ptr(self.ptr, u64p), ptr(self.idx, u32p))


def null_sparse():
    return SparseView(C.cast(None, u64p), C.cast(None, u32p), C.cast(None, f32p))


def null_list():
    return ListView(C.cast(None, u64p), C.cast(None, u32p))


class InsertParams(C.Structure):
    _fields_ = [("knn_k", C.c_uint32), ("nn_descent_iterations", C.c_uint32), ("threads", C.c_uint32)]


class Corpus:
    """DocumentStore (types.hpp:119-133) as structure-of-arrays."""

    def __init__(self, dense, learned: CSR, statistical: CSR, keywords: CSR | None = None,
                 entities: CSR | None = None, doc_id=None, deleted=None, learned_dim=0,
                 statistical_dim=0):
        self.dense = arr(dense, np.float32)
        assert self.dense.ndim == 2
        self.n, self.dense_dim = self.dense.shape
        self.learned = learned
        self.statistical = statistical
        self.keywords = keywords
        self.entities = entities
        self.doc_id = arr(doc_id, np.uint64)
        self.deleted = arr(deleted, np.uint8)
        self.learned_dim = learned_dim
        self.statistical_dim = statistical_dim

    def view(self) -> CorpusView:
        v = CorpusView()
        v.n = self.n
        v.dense_dim = self.dense_dim
        v.learned_dim = self.learned_dim
        v.statistical_dim = self.statistical_dim
        v.dense = ptr(self.dense, f32p)
        v.learned = self.learned.sparse_view() if self.learned is not None else null_sparse()
        v.statistical = (self.statistical.sparse_view() if self.statistical is not None
                         else null_sparse())
        v.keywords = self.keywords.list_view() if self.keywords is not None else null_list()
        v.entities = self.entities.list_view() if self.entities is not None else null_list()
        v.doc_id = ptr(self.doc_id, u64p)
        v.deleted = ptr(self.deleted, u8p)
        return v

    def keyword_csr(self) -> CSR:
        if self.keywords is not None:
            return self.keywords
        return CSR(self.statistical.ptr, self.statistical.idx)

    def doc_ids(self):
        return self.doc_id if self.doc_id is not None else np.arange(self.n, dtype=np.uint64)


class KG:
    def __init__(self, source=(), relation=(), target=()):
        self.source = np.ascontiguousarray(source, dtype=np.uint32)
        self.relation = np.ascontiguousarray(relation, dtype=np.uint32)
        self.target = np.ascontiguousarray(target, dtype=np.uint32)

    def view(self) -> KgView:
        return KgView(len(self.source), ptr(self.source, u32p), ptr(self.relation, u32p),
                      ptr(self.target, u32p))

    def __len__(self):
        return len(self.source)


class Queries:
    """A batch of QuerySpec (types.hpp:70-78)."""

    def __init__(self, dense, learned: CSR, statistical: CSR, weights, k=10, beam_width=64,
                 max_entity_hops=2, required: CSR | None = None, entities: CSR | None = None):
        self.dense = arr(dense, np.float32)
        self.count, self.dense_dim = self.dense.shape
        self.learned = learned
        self.statistical = statistical
        w = np.asarray(weights, dtype=np.float32).reshape(self.count, -1)
        if w.shape[1] == 3:
            w = np.concatenate([w, np.zeros((self.count, 1), np.float32)], axis=1)
        self.weights = np.ascontiguousarray(w)
        self.k = self._per_query(k)
        self.beam_width = self._per_query(beam_width)
        self.max_entity_hops = self._per_query(max_entity_hops)
        self.required = required
        self.entities = entities

    def _per_query(self, v):
        a = np.asarray(v, dtype=np.uint32)
        if a.ndim == 0:
            a = np.full(self.count, int(a), np.uint32)
        return np.ascontiguousarray(a)

    def with_(self, **kw):
        q = Queries.__new__(Queries)
        q.__dict__.update(self.__dict__)
        for key, v in kw.items():
            if key in ("k", "beam_width", "max_entity_hops"):
                v = q._per_query(v)
            setattr(q, key, v)
        return q

    def subset(self, rows):
        rows = np.asarray(rows, dtype=np.int64)
        return Queries(self.dense[rows], self.learned.subset(rows), self.statistical.subset(rows),
                       self.weights[rows], self.k[rows], self.beam_width[rows],
                       self.max_entity_hops[rows],
                       None if self.required is None else self.required.subset(rows),
                       None if self.entities is None else self.entities.subset(rows))

    def view(self) -> QueryView:
        v = QueryView()
        v.count = self.count
        v.dense_dim = self.dense_dim
        v.dense = ptr(self.dense, f32p)
        v.learned = self.learned.sparse_view() if self.learned is not None else null_sparse()
        v.statistical = (self.statistical.sparse_view() if self.statistical is not None
                         else null_sparse())
        v.weights = self.weights.ctypes.data_as(C.POINTER(Weights))
        v.required_keywords = self.required.list_view() if self.required is not None else null_list()
        v.entities = self.entities.list_view() if self.entities is not None else null_list()
        v.k = ptr(self.k, u32p)
        v.beam_width = ptr(self.beam_width, u32p)
        v.max_entity_hops = ptr(self.max_entity_hops, u32p)
        return v

    def pinned(self) -> "Queries":
        """A copy whose arrays live in page-locked host memory (torch pinned
        tensors), so the library's host->device copies run at full DMA speed."""
        import torch

        owners = []

        def pin(a):
            if a is None:
                return None
            t = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), pin_memory=True)
            owners.append(t)  # the numpy view does not keep the tensor alive
            out = t.numpy()
            out[...] = a
            return out

        def pin_csr(c):
            return None if c is None else CSR(pin(c.ptr), pin(c.idx), pin(c.val))

        q = Queries.__new__(Queries)
        q.__dict__.update(self.__dict__)
        q.dense = pin(self.dense)
        q.learned, q.statistical = pin_csr(self.learned), pin_csr(self.statistical)
        q.required, q.entities = pin_csr(self.required), pin_csr(self.entities)
        q.weights, q.k = pin(self.weights), pin(self.k)
        q.beam_width, q.max_entity_hops = pin(self.beam_width), pin(self.max_entity_hops)
        q._pinned = owners
        return q

    def h2d_bytes(self) -> int:
        """Bytes of the query payload a search call ships to the device."""
        total = self.dense.nbytes + self.weights.nbytes + 3 * 4 * self.count
        for c in (self.learned, self.statistical, self.required, self.entities):
            if c is not None:
                total += c.ptr.nbytes + c.idx.nbytes + (0 if c.val is None else c.val.nbytes)
        return total


class Results:
    """SearchResult rows (search.hpp:31-43) in flat arrays."""

    ERR_STRIDE = 192

    def __init__(self, count, hit_stride):
        self.count = count
        self.hit_stride = max(1, int(hit_stride))
        self.doc_id = np.zeros((count, self.hit_stride), np.uint64)
        self.node = np.zeros((count, self.hit_stride), np.uint32)
        self.score = np.zeros((count, self.hit_stride), np.float64)
        self.hit_count = np.zeros(count, np.uint32)
        self.expanded = np.zeros(count, np.uint64)
        self.scored = np.zeros(count, np.uint64)
        self.warnings = np.zeros(count, np.uint32)
        self._err = C.create_string_buffer(count * self.ERR_STRIDE)

    def struct(self) -> SearchResults:
        return SearchResults(self.hit_stride, ptr(self.doc_id, u64p), ptr(self.node, u32p),
                             ptr(self.score, f64p), ptr(self.hit_count, u32p),
                             ptr(self.expanded, u64p), ptr(self.scored, u64p),
                             ptr(self.warnings, u32p), C.cast(self._err, C.c_char_p),
                             self.ERR_STRIDE)

    def error(self, i) -> str:
        raw = self._err.raw[i * self.ERR_STRIDE:(i + 1) * self.ERR_STRIDE]
        return raw.split(b"\0", 1)[0].decode()

    def hits(self, i):
        h = int(self.hit_count[i])
        return list(zip(self.doc_id[i, :h].tolist(), self.node[i, :h].tolist(),
                        self.score[i, :h].tolist()))

    def ids(self, i):
        return self.doc_id[i, :int(self.hit_count[i])]


def graph_view(g: dict) -> GraphView:
    """fg_graph_view over a dict(degree, semantic, keyword: CSR, logical_ptr,
    logical (E x 4), norm_order); the dict must outlive the view."""
    gv = GraphView()
    gv.degree = g["degree"]
    gv.semantic = ptr(g["semantic"], u32p)
    gv.keyword = g["keyword"].list_view()
    gv.logical_ptr = ptr(g.get("logical_ptr"), u64p)
    gv.logical = ptr(g.get("logical"), u32p)
    gv.norm_order = ptr(g.get("norm_order"), u32p)
    return gv


def knn_struct(ids, scores, fresh):
    n, k = ids.shape
    return KnnLists(n, k, ptr(ids, u32p), ptr(scores, f64p), ptr(fresh, u8p))


def synth_params(**kw) -> SynthParams:
    """SynthParams with the reference defaults (synth.hpp:19-45)."""
    d = dict(docs=1000, dense_dim=16, clusters=20, cluster_spread=0.25, learned_vocab=2000,
             learned_nnz=20, statistical_vocab=2000, statistical_nnz=20, zipf_exponent=1.1,
             entity_vocab=0, entity_rate=0.3, max_entities_per_doc=2, kg_triplets=0,
             relation_vocab=8, chains=0, answers_per_chain=10, seed=1)
    unknown = set(kw) - set(d)
    assert not unknown, unknown
    d.update(kw)
    return SynthParams(**d)
