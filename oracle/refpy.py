"""TEST INFRASTRUCTURE — Python bindings of the two CPU checkers.

  RefLib    -> oracle/_ref/libfgref.so : the UNMODIFIED reference (fusegraph_ref)
  OracleLib -> oracle/liboracle.so     : our CPU restatement (fg_oracle.cpp)

Both expose the same methods, taking the flat containers of
paper_2511_00855_b200._abi, so a test can run the GPU path, the restatement
and the reference on the very same arrays.  Only tests/, smoke() and
bench.py's CPU-baseline / reference arm may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2511_00855_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfgref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")


class CheckerError(RuntimeError):
    def __init__(self, what):
        super().__init__(what)
        self.code = what.split(":", 1)[0]


def build(ref=True):
    """make -C oracle (restatement always; the reference when its sources exist)."""
    targets = ["oracle"] + (["ref"] if ref else [])
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL)


class _Base:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        P = C.POINTER
        p = self.prefix
        sig = {
            "last_error": (C.c_char_p, []),
            "store_create": (C.c_int, [P(A.CorpusView), P(A.KgView), P(C.c_void_p)]),
            "store_free": (None, [C.c_void_p]),
            "store_sqnorm": (C.c_int, [C.c_void_p, A.f64p]),
            "build_query_vector": (C.c_int, [P(A.QueryView), C.c_uint64, A.f32p, A.u32p, A.f32p,
                                             A.u32p, A.f32p, A.f64p]),
            "batch_scores": (C.c_int, [C.c_void_p, P(A.QueryView), C.c_uint64, A.u32p, C.c_uint64,
                                       C.c_uint, A.f64p]),
            "pair_scores": (C.c_int, [C.c_void_p, A.u32p, A.u32p, C.c_uint64, A.f64p]),
            "knn_init": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint, P(A.KnnLists)]),
            "knn_iterate": (C.c_int, [C.c_void_p, P(A.KnnLists), C.c_uint, A.u64p]),
            "knn_iterate_range": (C.c_int, [C.c_void_p, P(A.KnnLists), C.c_uint64, C.c_uint64, A.u64p]),
            "knn_build": (C.c_int, [C.c_void_p, P(A.KnnParams), C.c_uint, P(A.KnnLists)]),
            "refine": (C.c_int, [C.c_void_p, P(A.KnnLists), P(A.RefineParams), C.c_uint,
                                 P(A.Refined), P(A.RefineTrace)]),
            "index_build": (C.c_int, [C.c_void_p, P(A.BuildParams), C.c_uint, P(C.c_void_p)]),
            "index_create": (C.c_int, [C.c_void_p, P(A.GraphView), C.c_uint32, P(C.c_void_p)]),
            "index_free": (None, [C.c_void_p]),
            "index_sizes": (C.c_int, [C.c_void_p, A.u32p, A.u64p, A.u64p]),
            "index_export": (C.c_int, [C.c_void_p, A.u32p, A.u64p, A.u32p, A.u64p, A.u32p,
                                       A.u32p]),
            "index_set_deleted": (C.c_int, [C.c_void_p, A.u8p]),
            "index_serialize": (C.c_int, [C.c_void_p, C.c_char_p, A.u64p]),
            "index_insert": (C.c_int, [C.c_void_p, P(A.CorpusView), C.c_uint32, C.c_uint32]),
            "index_deserialize": (C.c_int, [C.c_char_p, P(C.c_void_p)]),
            "batch_query": (C.c_int, [C.c_void_p, P(A.QueryView), P(A.SearchOpts), C.c_uint,
                                      P(A.SearchResults)]),
            "brute_force": (C.c_int, [C.c_void_p, P(A.QueryView), C.c_uint, P(A.SearchResults)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, p + name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
            setattr(self, "_" + name, fn)

    def _check(self, st):
        if st != 0:
            raise CheckerError(self._last_error().decode())

    # ---------------------------------------------------------------- store
    def store(self, corpus: A.Corpus, kg: A.KG | None = None):
        h = C.c_void_p()
        v = corpus.view()
        kv = kg.view() if kg is not None else A.KG().view()
        self._check(self._store_create(C.byref(v), C.byref(kv), C.byref(h)))
        return _Handle(h, self._store_free)

    def sqnorm(self, store, n):
        out = np.zeros(n, np.float64)
        self._check(self._store_sqnorm(store.h, A.ptr(out, A.f64p)))
        return out

    def build_query_vector(self, q: A.Queries, i: int):
        dense = np.zeros(q.dense_dim, np.float32)
        li, _ = q.learned.row(i)
        si, _ = q.statistical.row(i)
        lv = np.zeros(max(len(li), 1), np.float32)
        sv = np.zeros(max(len(si), 1), np.float32)
        ln, sn, sq = C.c_uint32(), C.c_uint32(), C.c_double()
        v = q.view()
        self._check(self._build_query_vector(C.byref(v), i, A.ptr(dense, A.f32p), C.byref(ln),
                                             A.ptr(lv, A.f32p), C.byref(sn), A.ptr(sv, A.f32p),
                                             C.byref(sq)))
        return dense, lv[:ln.value], sv[:sn.value], sq.value

    def batch_scores(self, store, q: A.Queries, qi: int, ids, threads=1):
        ids = np.ascontiguousarray(ids, np.uint32)
        out = np.zeros(len(ids), np.float64)
        v = q.view()
        self._check(self._batch_scores(store.h, C.byref(v), qi, A.ptr(ids, A.u32p), len(ids),
                                       threads, A.ptr(out, A.f64p)))
        return out

    def pair_scores(self, store, a, b):
        a = np.ascontiguousarray(a, np.uint32)
        b = np.ascontiguousarray(b, np.uint32)
        out = np.zeros(len(a), np.float64)
        self._check(self._pair_scores(store.h, A.ptr(a, A.u32p), A.ptr(b, A.u32p), len(a),
                                      A.ptr(out, A.f64p)))
        return out

    # ---------------------------------------------------------------- knn
    @staticmethod
    def _lists(n, k):
        return (np.zeros((n, k), np.uint32), np.zeros((n, k), np.float64),
                np.zeros((n, k), np.uint8))

    def knn_init(self, store, n, k, seed, threads=1):
        ids, sc, fr = self._lists(n, k)
        s = A.knn_struct(ids, sc, fr)
        self._check(self._knn_init(store.h, k, seed, threads, C.byref(s)))
        return ids, sc, fr

    def knn_iterate(self, store, ids, sc, fr, threads=1):
        ids, sc, fr = ids.copy(), sc.copy(), fr.copy()
        s = A.knn_struct(ids, sc, fr)
        ch = C.c_uint64()
        self._check(self._knn_iterate(store.h, C.byref(s), threads, C.byref(ch)))
        return ids, sc, fr, ch.value

    def knn_iterate_range(self, store, ids, sc, fr, lo, hi):
        """One pass for nodes [lo, hi) only (other rows returned unchanged)."""
        ids, sc, fr = ids.copy(), sc.copy(), fr.copy()
        s = A.knn_struct(ids, sc, fr)
        ch = C.c_uint64()
        self._check(self._knn_iterate_range(store.h, C.byref(s), lo, hi, C.byref(ch)))
        return ids, sc, fr, ch.value

    def knn_build(self, store, n, k, max_iterations=12, convergence=0.01, seed=42, threads=1):
        kk = min(k, n - 1) if n >= 2 else k
        ids, sc, fr = self._lists(n, kk)
        s = A.knn_struct(ids, sc, fr)
        p = A.KnnParams(k, max_iterations, convergence, seed)
        self._check(self._knn_build(store.h, C.byref(p), threads, C.byref(s)))
        return ids, sc, fr

    # ---------------------------------------------------------------- refine
    def refine(self, store, ids, sc, fr, degree, per_neighbour=False, threads=1, trace=False):
        n, k = ids.shape
        sem = np.zeros((n, degree), np.uint32)
        kw = np.zeros((n, k), np.uint32)
        kwc = np.zeros(n, np.uint32)
        out = A.Refined(A.ptr(sem, A.u32p), k, A.ptr(kw, A.u32p), A.ptr(kwc, A.u32p))
        t = None
        tr = None
        if trace:
            t = dict(ordered_ids=np.zeros((n, k), np.uint32),
                     ordered_scores=np.zeros((n, k), np.float64),
                     detours=np.zeros((n, k), np.uint32), kept=np.zeros((n, degree), np.uint32),
                     kept_count=np.zeros(n, np.uint32))
            tr = A.RefineTrace(A.ptr(t["ordered_ids"], A.u32p), A.ptr(t["ordered_scores"], A.f64p),
                               A.ptr(t["detours"], A.u32p), A.ptr(t["kept"], A.u32p),
                               A.ptr(t["kept_count"], A.u32p))
        lists = A.knn_struct(ids, sc, fr)
        p = A.RefineParams(degree, int(per_neighbour))
        self._check(self._refine(store.h, C.byref(lists), C.byref(p), threads, C.byref(out),
                                 C.byref(tr) if tr is not None else None))
        keyword = [kw[u, :kwc[u]].copy() for u in range(n)]
        return sem, keyword, t

    # ---------------------------------------------------------------- index
    def index_build(self, store, degree=32, knn_k=32, knn_iterations=10, seed=42, logical_cap=64,
                    default_entity_hops=2, per_neighbour=False, threads=1):
        """Consumes `store` (the reference moves the DocumentStore in)."""
        h = C.c_void_p()
        p = A.BuildParams(degree, knn_k, knn_iterations, seed, logical_cap, default_entity_hops,
                          int(per_neighbour))
        self._check(self._index_build(store.h, C.byref(p), threads, C.byref(h)))
        return _Handle(h, self._index_free)

    def index_insert(self, ix, docs: A.Corpus, knn_k=0, iterations=10):
        v = docs.view()
        self._check(self._index_insert(ix.h, C.byref(v), knn_k, iterations))

    def index_serialize(self, ix, path: str) -> int:
        nb = C.c_uint64()
        self._check(self._index_serialize(ix.h, path.encode(), C.byref(nb)))
        return nb.value

    def index_deserialize(self, path: str):
        h = C.c_void_p()
        self._check(self._index_deserialize(path.encode(), C.byref(h)))
        return _Handle(h, self._index_free)

    def index_create(self, store, graph: dict, knn_k=0):
        """HybridIndex over the given edge tables (consumes `store`)."""
        h = C.c_void_p()
        gv = graph_view(graph)
        self._check(self._index_create(store.h, C.byref(gv), knn_k, C.byref(h)))
        return _Handle(h, self._index_free)

    def index_export(self, ix, n):
        deg, kt, lt = C.c_uint32(), C.c_uint64(), C.c_uint64()
        self._check(self._index_sizes(ix.h, C.byref(deg), C.byref(kt), C.byref(lt)))
        sem = np.zeros((n, deg.value), np.uint32)
        kp = np.zeros(n + 1, np.uint64)
        ki = np.zeros(kt.value, np.uint32)
        lp = np.zeros(n + 1, np.uint64)
        lg = np.zeros((lt.value, 4), np.uint32)
        no = np.zeros(n, np.uint32)
        self._check(self._index_export(ix.h, A.ptr(sem, A.u32p), A.ptr(kp, A.u64p),
                                       A.ptr(ki, A.u32p), A.ptr(lp, A.u64p), A.ptr(lg, A.u32p),
                                       A.ptr(no, A.u32p)))
        return dict(degree=deg.value, semantic=sem, keyword=A.CSR(kp, ki), logical_ptr=lp,
                    logical=lg, norm_order=no)

    def index_set_deleted(self, ix, flags):
        flags = np.ascontiguousarray(flags, np.uint8)
        self._check(self._index_set_deleted(ix.h, A.ptr(flags, A.u8p)))

    def batch_query(self, ix, q: A.Queries, entry_count=32, conjunctive=True, threads=1):
        res = A.Results(q.count, int(q.k.max()) if q.count else 1)
        rs = res.struct()
        v = q.view()
        o = A.SearchOpts(entry_count, int(conjunctive))
        self._check(self._batch_query(ix.h, C.byref(v), C.byref(o), threads, C.byref(rs)))
        return res

    def brute_force(self, store, q: A.Queries, threads=1):
        res = A.Results(q.count, int(q.k.max()) if q.count else 1)
        rs = res.struct()
        v = q.view()
        self._check(self._brute_force(store.h, C.byref(v), threads, C.byref(rs)))
        return res


class _Handle:
    def __init__(self, h, free):
        self.h = h
        self._free = free

    def close(self):
        if self.h:
            self._free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


graph_view = A.graph_view


class RefLib(_Base):
    prefix = "fgref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.fgref_synth_generate.argtypes = [C.POINTER(A.SynthParams), C.POINTER(C.c_void_p)]
        L.fgref_synth_view.argtypes = [C.c_void_p, C.POINTER(A.CorpusView), C.POINTER(A.KgView),
                                       A.u64p]
        L.fgref_synth_free.argtypes = [C.c_void_p]
        L.fgref_synth_free.restype = None
        L.fgref_synth_queries.argtypes = [C.POINTER(A.SynthParams), C.c_uint64, C.c_uint64,
                                          C.c_int, A.f32p, A.u32p, A.f32p, A.u32p, A.f32p,
                                          C.POINTER(A.Weights)]
        L.fgref_queries_create.argtypes = [C.POINTER(A.QueryView), C.POINTER(C.c_void_p)]
        L.fgref_queries_free.argtypes = [C.c_void_p]
        L.fgref_queries_free.restype = None
        L.fgref_batch_query_prepared.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                 C.POINTER(A.SearchOpts), C.c_uint,
                                                 C.POINTER(A.SearchResults)]
        L.fgref_index_brute_force.argtypes = [C.c_void_p, C.POINTER(A.QueryView), C.c_uint,
                                              C.POINTER(A.SearchResults)]

    def generate_corpus(self, params: A.SynthParams):
        h = C.c_void_p()
        self._check(self.lib.fgref_synth_generate(C.byref(params), C.byref(h)))
        try:
            v, kg, nc = A.CorpusView(), A.KgView(), C.c_uint64()
            self.lib.fgref_synth_view(h, C.byref(v), C.byref(kg), C.byref(nc))
            n, d = v.n, v.dense_dim

            def cp(p, m, dt):
                return np.ctypeslib.as_array(p, shape=(m,)).astype(dt, copy=True) if m else \
                    np.zeros(0, dt)

            def csr(sv, with_val=True):
                pp = cp(sv.ptr, n + 1, np.uint64)
                m = int(pp[-1])
                return A.CSR(pp, cp(sv.idx, m, np.uint32), cp(sv.val, m, np.float32) if with_val
                             else None)

            corpus = A.Corpus(cp(v.dense, n * d, np.float32).reshape(n, d), csr(v.learned),
                              csr(v.statistical), csr(v.keywords, False), csr(v.entities, False),
                              cp(v.doc_id, n, np.uint64), cp(v.deleted, n, np.uint8),
                              v.learned_dim, v.statistical_dim)
            graph = A.KG(cp(kg.source, kg.count, np.uint32), cp(kg.relation, kg.count, np.uint32),
                         cp(kg.target, kg.count, np.uint32))
            return corpus, graph, nc.value
        finally:
            self.lib.fgref_synth_free(h)

    def synth_queries(self, params, count, stream=0x71E5, with_weights=True):
        d = params.dense_dim
        ln = min(params.learned_nnz, params.learned_vocab)
        sn = min(params.statistical_nnz, params.statistical_vocab)
        dense = np.zeros((count, d), np.float32)
        li = np.zeros(count * ln, np.uint32)
        lv = np.zeros(count * ln, np.float32)
        si = np.zeros(count * sn, np.uint32)
        sv = np.zeros(count * sn, np.float32)
        w = np.zeros((count, 4), np.float32)
        self._check(self.lib.fgref_synth_queries(C.byref(params), stream, count, int(with_weights),
                                                 A.ptr(dense, A.f32p), A.ptr(li, A.u32p),
                                                 A.ptr(lv, A.f32p), A.ptr(si, A.u32p),
                                                 A.ptr(sv, A.f32p),
                                                 w.ctypes.data_as(C.POINTER(A.Weights))))
        return dense, li, lv, si, sv, w

    def prepare_queries(self, q: A.Queries):
        h = C.c_void_p()
        v = q.view()
        self._check(self.lib.fgref_queries_create(C.byref(v), C.byref(h)))
        return _Handle(h, self.lib.fgref_queries_free)

    def batch_query_prepared(self, ix, prepared, begin, end, k_max, entry_count=32,
                             conjunctive=True, threads=1):
        res = A.Results(end - begin, k_max)
        rs = res.struct()
        o = A.SearchOpts(entry_count, int(conjunctive))
        self._check(self.lib.fgref_batch_query_prepared(ix.h, prepared.h, begin, end, C.byref(o),
                                                        threads, C.byref(rs)))
        return res

    def index_brute_force(self, ix, q: A.Queries, threads=1):
        res = A.Results(q.count, int(q.k.max()) if q.count else 1)
        rs = res.struct()
        v = q.view()
        self._check(self.lib.fgref_index_brute_force(ix.h, C.byref(v), threads, C.byref(rs)))
        return res


class OracleLib(_Base):
    prefix = "fgo_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)


def ref_available() -> bool:
    return os.path.exists(REF_SO)
